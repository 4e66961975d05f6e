"""Run the C1 frame pipeline a few times (for ncu capture)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2201_05024_b200 as K
F = int(sys.argv[1]) if len(sys.argv) > 1 else 1
rx, pil, tx, _ = K.host_frames(range(F), 6, 16, 685, 3840, "QPSK")
pipe = K.FramePipeline(F, 6, 16, 685, 3840, "QPSK", precision="f32")
pipe.load(rx, pil, tx)
for _ in range(3):
    pipe.launch()
torch.cuda.synchronize()
print("bit errors", int(pipe.bit_err.sum()))
