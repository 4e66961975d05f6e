"""Graph-replay latency of the C1 frame pipeline, fused vs overlapped detection."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_05024_b200 as K
rx, pil, tx, _ = K.host_frames([0], 6, 16, 685, 3840, "QPSK")
for ov in (False, True):
    p = K.FramePipeline(1, 6, 16, 685, 3840, "QPSK", precision="f32", overlap=ov)
    p.load(rx, pil, tx); p.capture(); torch.cuda.synchronize()
    ts = []
    for _ in range(300):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); p.replay(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    print("overlap", ov, "graph replay p50 %.1f us p99 %.1f us" % (np.median(ts), np.percentile(ts, 99)), "bit err", int(p.bit_err.sum()))
