"""C3 sweep timing: K1 + K2 per frame (6 users, M=16) for n_train x W, FP32.
Usage: python tools/time_wide.py [n_train,W ...]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_05024_b200 as K
from paper_2201_05024_b200 import _device as dv, _lib
from paper_2201_05024_b200.apsm import qtab_device

pts = [tuple(map(int, a.split(","))) for a in sys.argv[1:]] or \
    [(nt, w) for nt in (685, 2048, 4096, 8192) for w in (20, 64, 128)]
Kk, M, prec = 6, 16, "f32"
for nt, W in pts:
    rx, pil, tx, _ = K.host_frames([1], Kk, M, nt, 16, "QPSK")
    p = K.FramePipeline(1, Kk, M, nt, 16, "QPSK", cfg=K.ApsmConfig(window=W), precision=prec,
                        overlap=False)
    p.load(rx, pil, tx)
    kp = _lib.params(p.cfg.params)
    st = dv.stream()
    gs = p.Np * p.ld
    def gram():
        _lib.check(dv.fn("kapsm_pilot_gram", prec)(dv.ptr(p.rx), p.T * M * 2, 1, nt, M, kp,
                                                   dv.ptr(p.gram), p.ld, gs, st), "gram")
    def train():
        _lib.check(dv.fn("kapsm_train", prec)(
            dv.ptr(p.gram), p.ld, gs, dv.ptr(p.rx), p.T * M * 2, dv.ptr(None), 0, 2 * M,
            dv.ptr(p.pilots), 1, Kk, p.Np, W, float(p.cfg.epsilon), kp, dv.ptr(p.qtab),
            dv.ptr(None), dv.ptr(None), dv.ptr(p.coeff), dv.ptr(p.first_step), dv.ptr(p.theta),
            dv.ptr(p.n_active), dv.ptr(p.status), st), "train")
    res = {}
    for name, fn in (("gram", gram), ("train", train)):
        fn(); torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        res[name] = min(ts)
    st_ = p.status.cpu().numpy()
    print(f"n_train {nt:5d} W {W:3d}: gram {res['gram']:9.1f} us  train {res['train']:10.1f} us "
          f"({res['train'] / p.Np * 1e3:7.1f} ns/step)  atoms {p.n_active.cpu().numpy().ravel().tolist()} "
          f"status {int(st_.max())}", flush=True)
    if os.environ.get("WIDE_CLOCKS"):
        fsv = p.first_step.cpu().numpy()[0, 0, 100:356].reshape(64, 4)
        print("  phase clocks (cumulative from step start: pre-barrier, barrier, update, end):")
        print("  median", np.median(fsv, axis=0).tolist(), " rows 10-14:", fsv[10:15].tolist())
