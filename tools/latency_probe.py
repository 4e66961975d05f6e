"""Quick probe: C1 single-frame pipeline latency (graph replay) + stage times."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_05024_b200 as K
from paper_2201_05024_b200 import _device as dv, _lib

def stage_times(pipe, reps=20):
    c = pipe.cfg; p = _lib.params(c.params); pre = pipe.prec
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t = np.zeros(3)
    for _ in range(reps):
        st = dv.stream()
        ev[0].record()
        _lib.check(dv.fn("kapsm_pilot_gram", pre)(dv.ptr(pipe.rx), pipe.T*pipe.M*2, pipe.F, pipe.n_train, pipe.M, p, dv.ptr(pipe.gram), pipe.ld, pipe.Np*pipe.ld, st), "g")
        ev[1].record()
        _lib.check(dv.fn("kapsm_train", pre)(dv.ptr(pipe.gram), pipe.ld, pipe.Np*pipe.ld, dv.ptr(pipe.rx), pipe.T*pipe.M*2, dv.ptr(None), 0, 2*pipe.M, dv.ptr(pipe.pilots), pipe.F, pipe.K, pipe.Np, c.window, float(c.epsilon), p, dv.ptr(pipe.qtab), dv.ptr(None), dv.ptr(None), dv.ptr(pipe.coeff), dv.ptr(pipe.first_step), dv.ptr(pipe.theta), dv.ptr(pipe.n_active), dv.ptr(pipe.status), st), "t")
        ev[2].record()
        _lib.check(dv.fn("kapsm_detect_frames", pre)(dv.ptr(pipe.rx), pipe.T*pipe.M*2, pipe.F, pipe.K, pipe.n_train, pipe.n_data, pipe.M, dv.ptr(pipe.coeff), dv.ptr(pipe.theta), p, dv.ptr(pipe.points), pipe.n_points, pipe.bps, dv.ptr(pipe.tx), dv.ptr(pipe.est), dv.ptr(pipe.labels), dv.ptr(pipe.bit_err), dv.ptr(pipe.sym_err), st), "d")
        ev[3].record(); ev[3].synchronize()
        t += [ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3])]
    return t / reps * 1e3

for (F, Kn, M, sch) in [(1, 6, 16, "QPSK"), (16, 6, 16, "QPSK"), (148, 6, 16, "QPSK"), (1, 16, 64, "QAM16")]:
    rx, pil, tx, _ = K.host_frames(range(F), Kn, M, 685, 3840, sch)
    pipe = K.FramePipeline(F, Kn, M, 685, 3840, sch, precision="f32")
    pipe.load(rx, pil, tx)
    pipe.launch(); torch.cuda.synchronize()
    st = stage_times(pipe)
    pipe.capture()
    lat = []
    for i in range(50):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); pipe.replay(); e1.record(); e1.synchronize()
        lat.append(e0.elapsed_time(e1) * 1e3)
    lat = np.array(lat[5:])
    r = pipe.results()
    print(f"F={F} K={Kn} M={M} {sch}: graph p50 {np.median(lat):.1f} us p99 {np.percentile(lat,99):.1f} us "
          f"-> {F/np.median(lat)*1e6:.0f} frames/s | gram {st[0]:.1f} train {st[1]:.1f} detect {st[2]:.1f} us | "
          f"bit_err sum {int(r['bit_err'].sum())} status {int(r['status'].max())}", flush=True)
