"""Per-step clock64 profile of the critical warp (frame 0, user 0) at C1."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_05024_b200 as K
from paper_2201_05024_b200 import _device as dv, _lib
lib = _lib.load()
fn = lib.kapsm_internal_train_clock_f32
P, L, I, D = C.c_void_p, C.c_longlong, C.c_int, C.c_double
fn.argtypes = [P, L, L, P, L, P, I, I, I, I, I, D, _lib.KernelParamsC, P, P, P, P, P, P, P, I, P]
rx, pil, tx, _ = K.host_frames([0], 6, 16, 685, 3840, "QPSK")
pipe = K.FramePipeline(1, 6, 16, 685, 3840, "QPSK", precision="f32")
pipe.load(rx, pil, tx); pipe.launch(); torch.cuda.synchronize()
clk = torch.zeros(2 * pipe.Np, dtype=torch.int64, device="cuda")
c = pipe.cfg
for var in [0, 2, 4]:
  for rep in range(3):
    _lib.check(fn(dv.ptr(pipe.gram), pipe.ld, pipe.Np*pipe.ld, dv.ptr(pipe.rx), pipe.T*pipe.M*2, dv.ptr(pipe.pilots), 1, 6, pipe.Np, 2*pipe.M, c.window, float(c.epsilon), _lib.params(c.params), dv.ptr(pipe.qtab), dv.ptr(pipe.coeff), dv.ptr(pipe.first_step), dv.ptr(pipe.theta), dv.ptr(pipe.n_active), dv.ptr(pipe.status), dv.ptr(clk), var, dv.stream()), "t")
  torch.cuda.synchronize()
  allc = clk.cpu().numpy(); t = allc[:pipe.Np]; sp = allc[pipe.Np:]; dt = np.diff(t)
  print("  steps with P not ready: %d, total spins %d" % ((sp > 0).sum(), sp.sum()))
  clk.zero_()
  print("variant %2d cycles/step: mean %.0f median %.0f | warm-up %.0f | steady %.0f" % (var, dt.mean(), np.median(dt), dt[:19].mean(), dt[64:].mean()))
  if var == 0: print("  first 40:", dt[:40].tolist())
