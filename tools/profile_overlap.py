"""A few graph replays of the overlapped C1 pipeline (for ncu launch lists)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2201_05024_b200 as K
rx, pil, tx, _ = K.host_frames([0], 6, 16, 685, 3840, "QPSK")
p = K.FramePipeline(1, 6, 16, 685, 3840, "QPSK", precision="f32", overlap=True)
p.load(rx, pil, tx)
for _ in range(3):
    p.launch()
torch.cuda.synchronize()
print("bit errors", int(p.bit_err.sum()))
