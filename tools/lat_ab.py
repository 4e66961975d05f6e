"""Single-frame C1 latency: graph-replay p50/p99 over n replays, three rounds."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_05024_b200 as K
rx, pil, tx, _ = K.host_frames(range(64), 6, 16, 685, 3840, "QPSK")
p = K.FramePipeline(1, 6, 16, 685, 3840, "QPSK", precision="f32", store_est=False)
p.load(rx[:1], pil[:1], tx[:1]); p.capture()
for _ in range(300): p.replay()
torch.cuda.synchronize()
for r in range(3):
    ts = []
    for i in range(1000):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); p.replay(); b.record(); ts.append((a, b))
    torch.cuda.synchronize()
    us = np.array([a.elapsed_time(b) * 1e3 for a, b in ts])
    print(f"round {r}: p50 {np.percentile(us, 50):.1f} p99 {np.percentile(us, 99):.1f} us")
