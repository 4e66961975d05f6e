"""Time the production kernels of the C1 frame pipeline separately (CUDA events,
median of reps): pilot_gram, apsm_train, detect_frames; and the whole graph."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_05024_b200 as K
from paper_2201_05024_b200 import _device as dv, _lib
F = int(sys.argv[1]) if len(sys.argv) > 1 else 1
CFG = {"C1": (6, 16, 685, 3840, "QPSK"), "C4": (16, 64, 685, 3840, "QAM16")}[sys.argv[2] if len(sys.argv) > 2 else "C1"]
reps = 30
rx, pil, tx, _ = K.host_frames(range(F), *CFG)
pipe = K.FramePipeline(F, *CFG, precision="f32", full_workspace=True)
pipe.load(rx, pil, tx)
pipe.launch(); torch.cuda.synchronize()
c = pipe.cfg; p = _lib.params(c.params); st = dv.stream(); gstride = pipe.Np * pipe.ld
def gram():
    _lib.check(dv.fn("kapsm_pilot_gram", "f32")(dv.ptr(pipe.rx), pipe.T * pipe.M * 2, pipe.F, pipe.n_train, pipe.M, p, dv.ptr(pipe.gram), pipe.ld, gstride, st), "g")
def train():
    _lib.check(dv.fn("kapsm_train", "f32")(dv.ptr(pipe.gram), pipe.ld, gstride, dv.ptr(pipe.rx), pipe.T * pipe.M * 2, dv.ptr(None), 0, 2 * pipe.M, dv.ptr(pipe.pilots), pipe.F, pipe.K, pipe.Np, c.window, float(c.epsilon), p, dv.ptr(pipe.qtab), dv.ptr(None), dv.ptr(None), dv.ptr(pipe.coeff), dv.ptr(pipe.first_step), dv.ptr(pipe.theta), dv.ptr(pipe.n_active), dv.ptr(pipe.status), st), "t")
def detect():
    _lib.check(dv.fn("kapsm_detect_frames", "f32")(dv.ptr(pipe.rx), pipe.T * pipe.M * 2, pipe.F, pipe.K, pipe.n_train, pipe.n_data, pipe.M, dv.ptr(pipe.coeff), dv.ptr(pipe.theta), p, dv.ptr(pipe.points), pipe.n_points, pipe.bps, dv.ptr(pipe.tx), dv.ptr(pipe.est), dv.ptr(pipe.labels), dv.ptr(pipe.bit_err), dv.ptr(pipe.sym_err), st), "d")
def whole():
    pipe.launch()
for name, fn in [("pilot_gram", gram), ("apsm_train", train), ("detect_frames", detect), ("pipeline", whole)]:
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"{name:14s} F={F}: median {np.median(ts):8.1f} us  min {min(ts):8.1f} us")
print("status", pipe.status.cpu().numpy().ravel()[:12].tolist(), "bit errors", int(pipe.bit_err.sum()))
# split detection stages
live = torch.zeros((int(_lib.load().kapsm_screen_workspace_bytes(F, pipe.n_train, pipe.n_data)) // 4 + 4,), dtype=torch.int32, device="cuda")
def screen():
    _lib.check(dv.fn("kapsm_detect_screen", "f32")(dv.ptr(pipe.rx), pipe.T * pipe.M * 2, pipe.F, pipe.n_train, pipe.n_data, pipe.M, p, dv.ptr(live), st), "s")
def finish():
    _lib.check(dv.fn("kapsm_detect_finish", "f32")(dv.ptr(pipe.rx), pipe.T * pipe.M * 2, pipe.F, pipe.K, pipe.n_train, pipe.n_data, pipe.M, dv.ptr(pipe.coeff), dv.ptr(pipe.theta), p, dv.ptr(pipe.points), pipe.n_points, pipe.bps, dv.ptr(pipe.tx), dv.ptr(live), dv.ptr(pipe.est), dv.ptr(pipe.labels), dv.ptr(pipe.bit_err), dv.ptr(pipe.sym_err), st), "f")
for name, fn in [("detect_screen", screen), ("detect_finish", finish)]:
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"{name:14s} F={F}: median {np.median(ts):8.1f} us  min {min(ts):8.1f} us")
print("live bits set", int(torch.bitwise_count(live).sum()) if hasattr(torch, "bitwise_count") else "?")
