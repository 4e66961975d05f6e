"""The tensor-core detection screen (csrc/screen_tc.cu, tcgen05.mma TF32 into
TMEM) against the exact classification and against the FP32 SIMT screen.

The screen is a conservative dead/live classifier of (pilot, payload) kernel
blocks: it must never drop a pair whose kernel survives FP32 (exact squared
distance * inv2s < 88), it may add pairs only inside its stated TF32 margin
((nx + ny) / 128), and the detection finished from its output must match the
one finished from the SIMT screen (engine.py:137-147 semantics)."""

import numpy as np
import pytest
import torch

import paper_2201_05024_b200 as K
from paper_2201_05024_b200 import _device as dv, _lib

pytestmark = pytest.mark.gpu
P = K.KernelParams(0.5, 0.5, 0.05)
INV2S = 1.0 / (2 * P.sigma_sq)


def _ws(F, nt, nd):
    n = int(_lib.load().kapsm_screen_workspace_bytes(F, nt, nd))
    return torch.zeros(((n + 15) // 16 * 4,), dtype=torch.int32, device=dv.device())


def _bits(ws, F, nt, nd):
    NW = (nt + 31) // 32
    w = ws[:F * NW * nd].view(F, NW, nd).cpu().numpy().view(np.uint32)
    # -> (F, n_train, n_data) boolean
    out = np.zeros((F, NW * 32, nd), dtype=bool)
    for b in range(32):
        out[:, b::32, :] = (w >> np.uint32(b)) & 1
    return out[:, :nt, :]


def _exact(rx, nt):
    """Exact min realified distance * inv2s and the margin of every pair (FP64)."""
    x, y = rx[:nt], rx[nt:]
    nx = np.sum(np.abs(x) ** 2, 1)
    ny = np.sum(np.abs(y) ** 2, 1)
    c = np.conj(x) @ y.T                                   # x^H y, (nt, nd)
    dmin = nx[:, None] + ny[None, :] - 2 * np.maximum(c.real, np.abs(c.imag))
    return dmin * INV2S, (nx[:, None] + ny[None, :])


def _run(rx_c, nt, nd, simt):
    F, T, M = rx_c.shape
    rxd = dv.complex_to_dev(rx_c, "f32")
    ws = _ws(F, nt, nd)
    fn = (_lib.load().kapsm_internal_screen_simt_f32 if simt
          else dv.fn("kapsm_detect_screen", "f32"))
    _lib.check(fn(dv.ptr(rxd), T * M * 2, F, nt, nd, M, _lib.params(P), dv.ptr(ws), dv.stream()),
               "screen")
    torch.cuda.synchronize()
    return rxd, ws


CASES = [
    ("C1", 6, 16, 685, 3840, None),
    ("near-duplicates M=16", 6, 16, 200, 300, 0.02),
    ("odd M=3 overloaded", 6, 3, 90, 150, 0.05),
    ("M=32", 8, 32, 150, 260, 0.02),
    ("C4 M=64", 16, 64, 685, 700, 0.01),
]


@pytest.mark.parametrize("name,Kn,M,nt,nd,dup", CASES, ids=[c[0] for c in CASES])
def test_tc_screen_is_exact_superset(name, Kn, M, nt, nd, dup):
    scheme = "QAM16" if M == 64 else "QPSK"
    rx, _, _, _ = K.host_frames([7, 8], Kn, M, nt, nd, scheme)
    if dup is not None:                          # payload symbols next to pilots: live kernels
        rng = np.random.default_rng(1)
        for f in range(rx.shape[0]):
            src = rng.integers(0, nt, nd // 3)
            rx[f, nt:nt + nd // 3] = rx[f, src] + dup * (rng.standard_normal((src.size, M))
                                                         + 1j * rng.standard_normal((src.size, M)))
    _, ws_tc = _run(rx, nt, nd, simt=False)
    _, ws_simt = _run(rx, nt, nd, simt=True)
    tc = _bits(ws_tc, rx.shape[0], nt, nd)
    simt = _bits(ws_simt, rx.shape[0], nt, nd)
    for f in range(rx.shape[0]):
        d, s = _exact(rx[f], nt)
        must = d < 88.0                                      # alive in FP32
        assert not np.any(must & ~tc[f]), f"{name}: tensor-core screen dropped a live pair"
        assert not np.any(simt[f] & ~tc[f]), f"{name}: not a superset of the SIMT screen"
        loose = d < 88.0 + (s / 64.0) * INV2S                # twice the stated margin
        assert not np.any(tc[f] & ~loose), f"{name}: live pair outside the TF32 margin"
        if dup is not None:
            assert must.sum() > 0                            # the case exercises live pairs


@pytest.mark.parametrize("M,nt,nd", [(16, 685, 3840), (3, 90, 150), (64, 300, 400)])
def test_detection_from_tc_screen_matches_simt_screen(M, nt, nd):
    """detect_finish on either screen's workspace: same decisions, estimates
    within 1e-6 (extra live pairs add kernels that underflow)."""
    Kn, scheme = (16, "QAM16") if M == 64 else (6, "QPSK")
    rx, pil, tx, _ = K.host_frames([3], Kn, M, nt, nd, scheme)
    rng = np.random.default_rng(4)
    src = rng.integers(0, nt, nd // 4)
    rx[0, nt:nt + nd // 4] = rx[0, src] + 0.02 * (rng.standard_normal((src.size, M)) +
                                                  1j * rng.standard_normal((src.size, M)))
    pipe = K.FramePipeline(1, Kn, M, nt, nd, scheme, precision="f32")
    pipe.load(rx, pil, tx)
    pipe.launch()                                          # trained coefficients + tc screen
    torch.cuda.synchronize()
    outs = []
    for simt in (False, True):
        rxd, ws = _run(rx, nt, nd, simt)
        est = torch.zeros((1, Kn, nd, 2), dtype=torch.float32, device=dv.device())
        lab = torch.zeros((1, Kn, nd), dtype=torch.uint8, device=dv.device())
        be = torch.zeros((1, Kn), dtype=torch.int64, device=dv.device())
        se = torch.zeros((1, Kn), dtype=torch.int64, device=dv.device())
        _lib.check(dv.fn("kapsm_detect_finish", "f32")(
            dv.ptr(rxd), (nt + nd) * M * 2, 1, Kn, nt, nd, M, dv.ptr(pipe.coeff),
            dv.ptr(pipe.theta), _lib.params(P), dv.ptr(pipe.points), pipe.n_points, pipe.bps,
            dv.ptr(pipe.tx), dv.ptr(ws), dv.ptr(est), dv.ptr(lab), dv.ptr(be), dv.ptr(se),
            dv.stream()), "finish")
        torch.cuda.synchronize()
        outs.append((est.cpu().numpy(), lab.cpu().numpy(), be.cpu().numpy()))
    (e0, l0, b0), (e1, l1, b1) = outs
    assert np.array_equal(l0, l1) and np.array_equal(b0, b1)
    assert np.max(np.abs(e0 - e1)) <= 1e-6 * np.max(np.abs(e1))
    # and the pipeline itself (tc screen inside the captured pipeline) agrees
    r = pipe.results()
    assert np.array_equal(r["labels"], l0)
