"""Single-frame C1 latency: graph-replay p50/p99 over n replays, three rounds;
'copies' also refreshes the inputs from a device pool before every replay (as
bench.py does), 'fixed' replays one frame."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_05024_b200 as K
mode = sys.argv[1] if len(sys.argv) > 1 else "fixed"
rx, pil, tx, _ = K.host_frames(range(64), 6, 16, 685, 3840, "QPSK")
p = K.FramePipeline(1, 6, 16, 685, 3840, "QPSK", precision="f32", store_est=False,
                    overlap="serial" not in sys.argv)
pool = K.FramePipeline(64, 6, 16, 685, 3840, "QPSK", precision="f32", store_est=False)
pool.load(rx, pil, tx)
f0 = int(mode[5:]) if mode.startswith("fixed") and len(mode) > 5 else 0
p.load(rx[f0:f0 + 1], pil[f0:f0 + 1], tx[f0:f0 + 1]); p.capture()
for _ in range(300): p.replay()
torch.cuda.synchronize()
for r in range(3):
    ts = []
    for i in range(1000):
        if mode.startswith("copies"):
            j = 0 if mode == "copies0" else i % 64
            p.rx.copy_(pool.rx[j:j + 1]); p.pilots.copy_(pool.pilots[j:j + 1]); p.tx.copy_(pool.tx[j:j + 1])
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); p.replay(); b.record(); ts.append((a, b))
    torch.cuda.synchronize()
    us = np.array([a.elapsed_time(b) * 1e3 for a, b in ts])
    print(f"{mode} round {r}: p50 {np.percentile(us, 50):.1f} p99 {np.percentile(us, 99):.1f} us")
