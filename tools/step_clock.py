"""Per-step clock64 profile of the critical warp (frame 0, user 0) at C1, with the
instrumentation build's timing variants (bit 1: no cp.async wait, 2: no takeover
row load, 4: no init wait, 8: background warps idle, 16: no __syncwarp, 32: no
per-step clock).  Variants other than 0 compute garbage; timing only."""
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
clk = torch.zeros(7 * pipe.Np + 8 * (pipe.Np // 4 + 2), dtype=torch.int64, device="cuda")
c = pipe.cfg
variants = [int(v) for v in sys.argv[1:]] or [0]
for var in variants:
    ts = []
    for rep in range(4):
        clk.zero_(); clk[5 * pipe.Np] = var
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(fn(dv.ptr(pipe.gram), pipe.ld, pipe.Np*pipe.ld, dv.ptr(pipe.rx), pipe.T*pipe.M*2, dv.ptr(pipe.pilots), 1, 6, pipe.Np, 2*pipe.M, c.window, float(c.epsilon), _lib.params(c.params), dv.ptr(pipe.qtab), dv.ptr(pipe.coeff), dv.ptr(pipe.first_step), dv.ptr(pipe.theta), dv.ptr(pipe.n_active), dv.ptr(pipe.status), dv.ptr(clk), var, dv.stream()), "t")
        e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    Np = pipe.Np; D = 8
    allc = clk.cpu().numpy(); t = allc[:pipe.Np]; sp = allc[pipe.Np:]; dt = np.diff(t)
    print("variant %2d: kernel %.1f us (min of 4) | status %s" % (var, min(ts), pipe.status.cpu().numpy().tolist()))
    if not (var & 32):
        print("  cycles/step: mean %.0f median %.0f p90 %.0f max %.0f | warm-up %.0f | steady %.0f | init spins %d" % (
            dt.mean(), np.median(dt), np.percentile(dt, 90), dt.max(), dt[:19].mean(), dt[64:].mean(), (sp > 0).sum()))
        print("  steps 64..96:", dt[64:96].tolist())
        mk = allc[7*Np:7*Np + 8*(Np//4)].reshape(-1, 8)
        print("  block marks (rel. to step n clock): [after step n, after publish/snap/wait, after step n+1, after takeover state+stage, after step n+2, after step n+3]")
        for jb in range(20, 26):
            print("   ", jb, (mk[jb, :6] - t[4*jb]).tolist(), "next block start", int(t[4*jb+4] - t[4*jb]))
        pub = allc[2*Np:3*Np]; bst = allc[3*Np:4*Np]; aend = allc[4*Np:5*Np]
        rows = []
        for m in range(400, 560):
            nm = (m - D) & ~3
            snapt = t[nm + 2] if nm + 2 < Np else 0
            dead = t[(m & ~3) - 2] if (m & ~3) - 2 < Np else 0
            bdone = allc[5*Np+1+m]
            rows.append((m, int(bst[m]-snapt), int(bdone-snapt), int(aend[m]-snapt), int(pub[m]-snapt), int(dead-snapt)))
        print("  m (rel. to CW step n_m+2 start): task-start, lastF-seen, early-part-seen, -, deadline")
        for r in rows[:24]: print("   ", r)
        late = [r for r in rows if r[4] > r[5]]; print('  late inits', len(late), 'of', len(rows))
