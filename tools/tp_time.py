"""Time the throughput pipeline's trainer stages (band rows, pilot screen,
one-warp trainer) and the whole pipeline on F C1 frames (default 1024),
CUDA events, median of reps.  usage: python tools/tp_time.py [F] [reps]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2201_05024_b200 as K
from paper_2201_05024_b200.framegen import FrameGenerator
from paper_2201_05024_b200 import _device as dv, _lib

def main():
    F = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    gen = FrameGenerator(F, 6, 16, 685, 3840, "QPSK", slots=1, workers=max(1, (os.cpu_count() or 2) - 1))
    gen.fill(0, list(range(F))).wait()
    p = K.FramePipeline(F, 6, 16, 685, 3840, "QPSK", precision="f32", store_est=False)
    p.rx.copy_(gen.rx[0].view(p.rx.shape))
    p.pilots.copy_(gen.pilots[0].view(p.pilots.shape))
    p.tx.copy_(gen.tx[0].view(p.tx.shape))
    lib = _lib.load()
    c = p.cfg
    st = dv.stream()


    def stage(bits):
        _lib.check(lib.kapsm_internal_train_tp_f32(
            bits, dv.ptr(p.rx), p.T * 16 * 2, dv.ptr(p.pilots), F, 6, 685, 16, c.window,
            float(c.epsilon), _lib.params(c.params), dv.ptr(p.qtab), dv.ptr(p._gram_buf),
            dv.ptr(p.coeff), dv.ptr(p.first_step), dv.ptr(p.theta), dv.ptr(p.n_active),
            dv.ptr(p.status), st), "tp")


    def timed(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        return float(np.median(ts))


    out = {"band": timed(lambda: stage(1)), "pilot_screen": timed(lambda: stage(2)),
           "trainer": timed(lambda: stage(4)), "pipeline": timed(p.launch)}
    r = p.results(check=True)
    print(f"F={F} " + " ".join(f"{k}={v:.0f}us" for k, v in out.items()),
          f"atoms={int(r['n_active'].sum())} bit_err={int(r['bit_err'].sum())}", flush=True)
    gen.close()


if __name__ == "__main__":
    main()
