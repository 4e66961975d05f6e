"""GPU parity of the general trainer (train_wide.cu): windows beyond the
latency kernel's W <= 23 and pilot counts beyond Np = 3072 -- BASELINE.json's
C3 dictionary/window sweep and the C4 full-band frame -- against the CPU
oracle (oracle/kapsm_oracle.py, pinned to the reference's golden vectors).
The ``force_wide`` fixture routes the small golden cases through the same
kernel (its C-ABI entry kapsm_train_general_*)."""

import glob
import os

import numpy as np
import pytest

import paper_2201_05024_b200 as K
from oracle import kapsm_oracle as O

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
SMALL = sorted(glob.glob(os.path.join(GOLDEN, "small_*.npz")))
P = K.KernelParams(0.5, 0.5, 0.05)


def maxrel(a, b):
    d = np.max(np.abs(b))
    return float(np.max(np.abs(a - b)) / d) if d else float(np.max(np.abs(a - b)))


@pytest.fixture
def force_wide(monkeypatch):
    monkeypatch.setattr(K.apsm, "_TRAIN_ENTRY", "kapsm_train_general")


def _check(f, ref, tol=1e-8):
    assert f.n_atoms == ref["n_atoms"]
    assert np.array_equal(f.atoms, ref["atoms"])                    # same atoms, same slot order
    np.testing.assert_allclose(f.coeffs, ref["coeffs"], rtol=tol, atol=1e-12)
    np.testing.assert_allclose(f.theta, ref["theta"], rtol=tol * 10, atol=1e-11)


@pytest.mark.parametrize("path", SMALL, ids=[os.path.basename(p) for p in SMALL])
def test_wide_f64_matches_golden(path, force_wide):
    g = np.load(path)
    fr = O.make_frame(int(g["seed"]), int(g["K"]), int(g["M"]), int(g["n_train"]),
                      int(g["n_data"]), str(g["scheme"]))
    nt = int(g["n_train"])
    R = O.realify(fr["rx"][:nt])
    for u in g["users"]:
        f = K.train(None, zip(fr["rx"][:nt], fr["symbols"][u, :nt]), K.ApsmConfig(),
                    precision="f64")
        assert f.n_atoms == int(g[f"u{u}_n_atoms"])
        assert np.array_equal(f.atoms, R[g[f"u{u}_atom_idx"]])
        np.testing.assert_allclose(f.theta, g[f"u{u}_theta"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(f.coeffs, g[f"u{u}_coeffs"], rtol=1e-8, atol=1e-12)
        f32 = K.train(None, zip(fr["rx"][:nt], fr["symbols"][u, :nt]), K.ApsmConfig(),
                      precision="f32")
        assert f32.n_atoms == int(g[f"u{u}_n_atoms"])
        assert maxrel(f32.theta, g[f"u{u}_theta"]) < 1e-4


def test_wide_generic_stream_and_warm_start(force_wide):
    rng = np.random.default_rng(12)
    cfg = K.ApsmConfig(window=6, epsilon=0.05, params=P)
    R = rng.standard_normal((120, 4)) * 0.3
    B = rng.standard_normal(120)
    tr = K.ApsmTrainer(4, cfg)
    for r, b in zip(R, B):
        tr.observe(r, b)
    _check(tr.state(), O.train_user(R, B, W=6, eps=0.05))
    # warm start (test_apsm.py:305-311): prefix kept, f0 feeds every response
    f0 = K.from_expansion([0.7, -0.2], [[0.1, 0.2, 0.0, 0.0], [0.0, 0.1, 0.3, -0.1]], P)
    t2 = K.ApsmTrainer(4, cfg, f0=f0)
    for r, b in zip(R[:40], B[:40]):
        t2.observe(r, b)
    s = t2.state()
    assert np.array_equal(s.atoms[:2], f0.atoms) and np.array_equal(s.coeffs[:2], f0.coeffs)
    # the same state from the oracle-checked default path (latency kernel)
    K.apsm._TRAIN_ENTRY = "kapsm_train"
    t3 = K.ApsmTrainer(4, cfg, f0=f0)
    for r, b in zip(R[:40], B[:40]):
        t3.observe(r, b)
    s3 = t3.state()
    assert s.n_atoms == s3.n_atoms and np.array_equal(s.atoms, s3.atoms)
    np.testing.assert_allclose(s.coeffs, s3.coeffs, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(s.theta, s3.theta, rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("W,n_train,M", [(24, 300, 16), (64, 685, 16), (128, 400, 16),
                                         (-1, 300, 8), (37, 200, 64)])
def test_wide_window_sweep_f64(W, n_train, M):
    """C3 window sweep rows (W in {64, 128} + the limits) against the oracle."""
    if W < 0:
        from paper_2201_05024_b200 import _lib
        W = _lib.load().kapsm_max_window()
        assert W >= 128
    fr = O.make_frame(W, 6, M, n_train, 8, "QPSK")
    R = O.realify(fr["rx"][:n_train])
    for u in (0, 5):
        B = O.realify_targets(fr["symbols"][u, :n_train])
        f = K.train(None, zip(fr["rx"][:n_train], fr["symbols"][u, :n_train]),
                    K.ApsmConfig(window=W), precision="f64")
        _check(f, O.train_user(R, B, W=W))


def test_many_samples_f64():
    """Np = 2 n_train = 3200 (beyond the latency trainer's former 3072 limit)
    against the oracle."""
    n_train = 1600
    fr = O.make_frame(2048, 6, 16, n_train, 8, "QPSK")
    R = O.realify(fr["rx"][:n_train])
    u = 3
    B = O.realify_targets(fr["symbols"][u, :n_train])
    f = K.train(None, zip(fr["rx"][:n_train], fr["symbols"][u, :n_train]), K.ApsmConfig(),
                precision="f64")
    _check(f, O.train_user(R, B, W=20))


def test_wide_frames_pipeline_large():
    """FramePipeline at a C3 point (n_train = 4096, W = 64): FP32 decisions and
    error counts equal the FP64 pipeline's, soft estimates within 1e-4."""
    import torch
    n_train, n_data, Kk, M = 4096, 512, 6, 16
    cfg = K.ApsmConfig(window=64)
    rx, pil, tx, _ = K.host_frames([5], Kk, M, n_train, n_data, "QPSK")
    out = {}
    for prec in ("f64", "f32"):
        p = K.FramePipeline(1, Kk, M, n_train, n_data, "QPSK", cfg=cfg, precision=prec)
        p.load(rx, pil, tx)
        p.launch()
        torch.cuda.synchronize()
        out[prec] = (p.labels.cpu().numpy(), p.bit_err.cpu().numpy(), p.est.cpu().numpy(),
                     p.status.cpu().numpy())
    assert not out["f64"][3].any() and not out["f32"][3].any()
    assert np.array_equal(out["f64"][0], out["f32"][0])
    assert np.array_equal(out["f64"][1], out["f32"][1])
    assert maxrel(out["f32"][2].astype(np.float64), out["f64"][2]) <= 1e-4


@pytest.mark.parametrize("n_train", [3500, 6000])
def test_large_np_paths_agree(n_train):
    """The latency trainer with staged targets (FP64 at Np = 7000, FP32 at
    Np = 12000) against the other precision's path (unstaged latency trainer,
    resp. the general trainer): identical decisions and error counts, soft
    estimates within 1e-4."""
    import torch
    Kk, M, n_data = 2, 16, 256
    rx, pil, tx, _ = K.host_frames([11], Kk, M, n_train, n_data, "QPSK")
    out = {}
    for prec in ("f64", "f32"):
        p = K.FramePipeline(1, Kk, M, n_train, n_data, "QPSK", precision=prec)
        p.load(rx, pil, tx)
        p.launch()
        torch.cuda.synchronize()
        out[prec] = (p.labels.cpu().numpy(), p.bit_err.cpu().numpy(), p.est.cpu().numpy(),
                     p.status.cpu().numpy(), p.n_active.cpu().numpy())
        del p
        torch.cuda.empty_cache()
    assert not out["f64"][3].any() and not out["f32"][3].any()
    assert np.array_equal(out["f64"][0], out["f32"][0])
    assert np.array_equal(out["f64"][1], out["f32"][1])
    assert np.array_equal(out["f64"][4], out["f32"][4])
    assert maxrel(out["f32"][2].astype(np.float64), out["f64"][2]) <= 1e-4


def test_large_np_latency_trainer_f64_vs_oracle():
    """Np = 4200 > 4096: the latency trainer's early parts come from the running
    linear part + live Gaussian lists (no Gram row streaming) -- FP64 against
    the oracle."""
    n_train = 2100
    fr = O.make_frame(4200, 6, 16, n_train, 8, "QPSK")
    R = O.realify(fr["rx"][:n_train])
    u = 1
    B = O.realify_targets(fr["symbols"][u, :n_train])
    f = K.train(None, zip(fr["rx"][:n_train], fr["symbols"][u, :n_train]), K.ApsmConfig(),
                precision="f64")
    _check(f, O.train_user(R, B, W=20))


@pytest.mark.parametrize("F,Kn,M,nt,W", [(2, 2, 2, 100, 25), (3, 2, 4, 100, 25), (2, 8, 2, 160, 40)])
def test_general_trainer_multi_frame_live_lists(F, Kn, M, nt, W):
    """FP64 pipelines of several frames at small M (many live Gaussian terms:
    the general trainer's per-frame live lists are used and overflow) against
    the oracle, every frame: coefficients and theta to 1e-9.  (Regression: the
    lists of frames >= 1 were written over frame 0's.)"""
    from oracle import kapsm_oracle as O
    seeds = list(range(100, 100 + F))
    rx, pil, tx, _ = K.host_frames(seeds, Kn, M, nt, 50, "QPSK")
    p = K.FramePipeline(F, Kn, M, nt, 50, "QPSK", cfg=K.ApsmConfig(window=W), precision="f64")
    p.load(rx, pil, tx)
    p.launch()
    r = p.results()
    for f in range(F):
        for u in (0, Kn - 1):
            ref = O.train_user(O.realify(rx[f, :nt]), O.realify_targets(pil[f, u]), W=W)
            assert int(r["n_active"][f, u]) == ref["n_atoms"], (f, u)
            assert np.max(np.abs(r["coeff"][f, u] - ref["coeff"])) <= 1e-9 * np.max(np.abs(ref["coeff"]))
            assert np.max(np.abs(r["theta"][f, u] - ref["theta"])) <= 1e-9 * np.max(np.abs(ref["theta"]))
