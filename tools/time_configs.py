"""Per-frame latency of the BASELINE configs through FramePipeline (FP32):
C1 (paper), C4 (massive, paper frame and full band), C3 points.
Usage: python tools/time_configs.py [name ...]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_05024_b200 as K

CONF = {
    "C1": dict(K=6, M=16, n_train=685, n_data=3840, scheme="QPSK", W=20),
    "C4": dict(K=16, M=64, n_train=685, n_data=3840, scheme="QAM16", W=20),
    "C4full": dict(K=16, M=64, n_train=6000, n_data=32400, scheme="QAM16", W=20),
    "C3_2048_64": dict(K=6, M=16, n_train=2048, n_data=3840, scheme="QPSK", W=64),
    "C3_8192_128": dict(K=6, M=16, n_train=8192, n_data=3840, scheme="QPSK", W=128),
}
names = sys.argv[1:] or list(CONF)
for name in names:
    c = CONF[name]
    rx, pil, tx, bits = K.host_frames([7], c["K"], c["M"], c["n_train"], c["n_data"], c["scheme"])
    p = K.FramePipeline(1, c["K"], c["M"], c["n_train"], c["n_data"], c["scheme"],
                        cfg=K.ApsmConfig(window=c["W"]), precision="f32")
    p.load(rx, pil, tx)
    p.launch(); torch.cuda.synchronize()
    reps = 20 if c["n_train"] <= 2048 else 3
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); p.launch(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    det = p.launch(time_detect=True); torch.cuda.synchronize()
    be = p.bit_err.cpu().numpy().ravel()
    nbits = c["n_data"] * (2 if c["scheme"] == "QPSK" else 4)
    print(f"{name:12s} K={c['K']:2d} M={c['M']:2d} n_train={c['n_train']:5d} n_data={c['n_data']:5d} "
          f"W={c['W']:3d}: frame {np.median(ts):10.1f} us (min {min(ts):.1f}), detect {det:8.1f} us, "
          f"status {int(p.status.max())}, BER {be.sum() / (nbits * c['K']):.2e}, "
          f"atoms {p.n_active.cpu().numpy().ravel()[:4].tolist()}", flush=True)
