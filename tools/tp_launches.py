"""One pipeline launch of F C1 frames (for an ncu launch list) plus a
graph-replay timing of the same pipeline (F frames per launch)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_05024_b200 as K
F = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rx, pil, tx, _ = K.host_frames(range(F), 6, 16, 685, 3840, "QPSK")
p = K.FramePipeline(F, 6, 16, 685, 3840, "QPSK", precision="f32", store_est=False)
p.load(rx, pil, tx)
p.launch(); torch.cuda.synchronize()
if reps:
    p.capture(); p.replay(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); p.replay(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    print(f"F={F}: pipeline median {np.median(ts):.1f} us  min {min(ts):.1f} us; status {int(p.status.max())} bit errors {int(p.bit_err.sum())}")
