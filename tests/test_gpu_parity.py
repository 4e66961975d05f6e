"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle and the
reference's golden vectors.  Bars (north star): hard decisions and error
counts exact; soft estimates within 1e-4 relative (max-norm) in FP32; the
FP64 kernels within 1e-9 of the reference (its own engine tolerance,
test_engine.py:49-55)."""

import glob
import os

import numpy as np
import torch
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


def gram_np(R, p=P):
    d2 = ((R[:, None, :] - R[None, :, :]) ** 2).sum(-1)
    return p.w_l * (R @ R.T) + p.w_g * np.exp(-d2 / (2 * p.sigma_sq))


# --------------------------------------------------------------------------- K1
@pytest.mark.parametrize("prec,tol", [("f32", 2e-6), ("f64", 1e-13)])
def test_pilot_gram(prec, tol):
    import torch
    from paper_2201_05024_b200 import _device as dv, _lib
    rng = np.random.default_rng(0)
    for (T, M, scale) in ((37, 3, 0.3), (50, 16, 1.0), (20, 5, 0.05)):
        x = scale * (rng.standard_normal((T, M)) + 1j * rng.standard_normal((T, M)))
        x[7] = x[3] + 1e-3          # near-duplicate pilots: live Gaussian terms
        N, ld = 2 * T, 2 * T + 32
        xd = dv.complex_to_dev(x, prec)
        g = dv.empty((N, ld), prec)
        _lib.check(dv.fn("kapsm_pilot_gram", prec)(dv.ptr(xd), 2 * T * M, 1, T, M,
                                                    _lib.params(P), dv.ptr(g), ld, N * ld,
                                                    dv.stream()), "gram")
        G = g.cpu().numpy()[:, :N].astype(np.float64)
        assert np.array_equal(G, G.T)                       # exactly symmetric
        ref = gram_np(O.realify(x))
        assert maxrel(G, ref) < tol


# --------------------------------------------------------------------------- K2
def _frame(g):
    return O.make_frame(int(g["seed"]), int(g["K"]), int(g["M"]), int(g["n_train"]),
                        int(g["n_data"]), str(g["scheme"]))


@pytest.mark.parametrize("path", SMALL, ids=[os.path.basename(p) for p in SMALL])
def test_train_f64_matches_reference(path):
    g = np.load(path)
    fr = _frame(g)
    nt = int(g["n_train"])
    R = O.realify(fr["rx"][:nt])
    for u in g["users"]:
        f = K.train(None, zip(fr["rx"][:nt], fr["symbols"][u, :nt]), K.ApsmConfig(),
                    precision="f64")
        assert f.n_atoms == int(g[f"u{u}_n_atoms"])
        assert np.array_equal(f.atoms, R[g[f"u{u}_atom_idx"]])       # same atoms, same slot order
        np.testing.assert_allclose(f.theta, g[f"u{u}_theta"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(f.coeffs, g[f"u{u}_coeffs"], rtol=1e-8, atol=1e-12)


@pytest.mark.parametrize("path", SMALL, ids=[os.path.basename(p) for p in SMALL])
def test_train_f32_close_to_reference(path):
    g = np.load(path)
    fr = _frame(g)
    nt = int(g["n_train"])
    for u in g["users"]:
        f = K.train(None, zip(fr["rx"][:nt], fr["symbols"][u, :nt]), K.ApsmConfig(),
                    precision="f32")
        assert f.n_atoms == int(g[f"u{u}_n_atoms"])
        assert maxrel(f.theta, g[f"u{u}_theta"]) < 1e-4


def test_trainer_generic_stream_and_warm_start():
    """ApsmTrainer on an arbitrary real stream (apsm.py:304) with a warm start."""
    rng = np.random.default_rng(12)
    cfg = K.ApsmConfig(window=6, epsilon=0.05, params=P)
    R = rng.standard_normal((120, 4)) * 0.3
    B = rng.standard_normal(120)
    tr = K.ApsmTrainer(4, cfg)
    for r, b in zip(R, B):
        tr.observe(r, b)
    f = tr.state()
    ref = O.train_user(R, B, W=6, eps=0.05)
    assert f.n_atoms == ref["n_atoms"]
    np.testing.assert_allclose(f.theta, ref["theta"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(f.coeffs, ref["coeffs"], rtol=1e-8, atol=1e-12)
    # warm start: prefix preserved (test_apsm.py:305-311)
    f0 = K.from_expansion([0.7], [[0.1, 0.2, 0.0, 0.0]], P)
    t2 = K.ApsmTrainer(4, K.ApsmConfig(params=P), f0=f0)
    assert t2.state().n_atoms == 1
    t2.observe(R[0], 3.0)
    s = t2.state()
    assert np.array_equal(s.atoms[0], f0.atoms[0]) and s.coeffs[0] == 0.7
    # the warm-started update lands on the eps boundary (single projection)
    y = K.evaluate(s, R[0], P)
    assert abs(abs(y - 3.0) - 0.01) < 1e-9


def test_train_literal_path_equivalence():
    """Coalesced trainer == literal apsm_step path (test_apsm.py:220-243)."""
    rng = np.random.default_rng(7)
    cfg = K.ApsmConfig(window=5, epsilon=0.02, params=P)
    stream = [(rng.standard_normal(3) * 0.4 + 1j * rng.standard_normal(3) * 0.4,
               complex(rng.standard_normal(), rng.standard_normal())) for _ in range(40)]
    f_fast = K.train(None, stream, cfg)
    f = K.zero_filter(6)
    hist = []
    for r, b in stream:
        for s in K.complex_to_real_pair(r, b):
            hist.append(s)
            n = len(hist) - 1
            f = K.apsm_step(f, [hist[i] for i in K.window_indices(n, cfg.window)], cfg)
    assert f.n_atoms >= f_fast.n_atoms
    np.testing.assert_allclose(f_fast.theta, f.theta, rtol=1e-9, atol=1e-12)
    u = rng.standard_normal((30, 6)) * 0.5
    a = K.batch_evaluate(f_fast, u, P, K.EngineConfig())
    b = K.batch_evaluate(f, u, P, K.EngineConfig())
    np.testing.assert_allclose(a, b, rtol=1e-9, atol=1e-12)


def test_train_errors():
    rng = np.random.default_rng(11)
    cfg = K.ApsmConfig(window=4, epsilon=0.01, params=P, max_atoms=5)
    stream = [(rng.standard_normal(2) + 1j * rng.standard_normal(2), complex(3.0, 3.0))
              for _ in range(50)]
    with pytest.raises(K.DictionaryCapacityError):
        K.train(None, stream, cfg)
    lin = K.KernelParams(1.0, 0.0, 0.05)
    with pytest.raises(ValueError):
        K.train(None, [(np.zeros(2, complex), 1 + 1j)], K.ApsmConfig(params=lin))
    with pytest.raises(ValueError):
        K.train(None, [], K.ApsmConfig())
    f = K.train(None, [(rng.standard_normal(2) + 1j * rng.standard_normal(2), complex(1, -1))
                       for _ in range(30)], K.ApsmConfig(window=4, epsilon=0.02, params=lin))
    assert f.n_atoms == 0


# --------------------------------------------------------------------------- K3 / pipeline
@pytest.mark.parametrize("path", SMALL, ids=[os.path.basename(p) for p in SMALL])
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_pipeline_small_frames(path, prec):
    g = np.load(path)
    Kn, M, nt, nd, sch = int(g["K"]), int(g["M"]), int(g["n_train"]), int(g["n_data"]), str(g["scheme"])
    rx, pil, tx, bits = K.host_frames([int(g["seed"])], Kn, M, nt, nd, sch)
    pipe = K.FramePipeline(1, Kn, M, nt, nd, sch, precision=prec)
    pipe.load(rx, pil, tx)
    pipe.launch()
    r = pipe.results()
    tol = 1e-4 if prec == "f32" else 1e-9
    kbits = K.get_constellation(sch).bits_per_symbol
    for u in range(Kn):
        est = g[f"u{u}_est"]
        assert maxrel(r["est"][0, u], est) < tol, (u, maxrel(r["est"][0, u], est))
        assert int(r["bit_err"][0, u]) == int(g[f"u{u}_bit_err"])
        assert int(r["n_active"][0, u]) == int(g[f"u{u}_n_atoms"])
        ref_idx = O.demap_indices(est, sch)
        assert np.array_equal(r["labels"][0, u], ref_idx)
        assert int(r["sym_err"][0, u]) == int(np.sum(ref_idx != tx[0, u]))
    assert np.all(r["status"] == 0)


def test_pipeline_c1_paper_frame():
    """C1 (K=6, M=16, QPSK, 685/3840) FP32: estimates within 1e-4 of the
    reference (users 0, 1 golden; all users vs the oracle), decisions exact."""
    g = np.load(os.path.join(GOLDEN, "c1_s0_users01.npz"))
    rx, pil, tx, bits = K.host_frames([0], 6, 16, 685, 3840, "QPSK")
    pipe = K.FramePipeline(1, 6, 16, 685, 3840, "QPSK", precision="f32")
    pipe.load(rx, pil, tx)
    pipe.launch()
    r = pipe.results()
    for u in (0, 1):
        assert maxrel(r["est"][0, u], g[f"u{u}_est"]) < 1e-4
        assert int(r["bit_err"][0, u]) == int(g[f"u{u}_bit_err"])
        assert int(r["n_active"][0, u]) == int(g[f"u{u}_n_atoms"])
    fr = O.make_frame(0, 6, 16, 685, 3840, "QPSK")
    for res in O.run_frame(fr, 685, "QPSK", users=[2, 3, 4, 5]):
        u = res["user"]
        assert maxrel(r["est"][0, u], res["est"]) < 1e-4
        assert np.array_equal(r["labels"][0, u], res["rx_idx"])
        assert int(r["bit_err"][0, u]) == res["bit_err"]


def test_graph_replay_matches_eager():
    rx, pil, tx, _ = K.host_frames([3, 4], 6, 16, 100, 160, "QPSK")
    pipe = K.FramePipeline(2, 6, 16, 100, 160, "QPSK", precision="f32")
    pipe.load(rx, pil, tx)
    pipe.launch()
    a = pipe.results()
    pipe.capture()
    for _ in range(3):
        pipe.replay()
    b = pipe.results()
    assert np.array_equal(a["est"], b["est"])
    assert np.array_equal(a["labels"], b["labels"])
    assert np.array_equal(a["bit_err"], b["bit_err"])


def test_multiframe_batch_equals_single():
    """Frames in one batch are independent (weak-scaling shard property)."""
    seeds = [5, 6, 7]
    rx, pil, tx, _ = K.host_frames(seeds, 3, 4, 60, 80, "QPSK")
    pipe = K.FramePipeline(3, 3, 4, 60, 80, "QPSK", precision="f32")
    pipe.load(rx, pil, tx)
    pipe.launch()
    full = pipe.results()
    for i in range(3):
        p1 = K.FramePipeline(1, 3, 4, 60, 80, "QPSK", precision="f32")
        p1.load(rx[i:i + 1], pil[i:i + 1], tx[i:i + 1])
        p1.launch()
        one = p1.results()
        assert np.array_equal(one["est"][0], full["est"][i])
        assert np.array_equal(one["bit_err"][0], full["bit_err"][i])


def test_throughput_mode_many_tasks_per_group():
    """F*K > 4 x SMs: throughput mode (4 chains per SM) with several tasks per
    chain group (barriers re-armed between tasks).  Same decisions as the
    latency mode (a 2-CTA cluster per chain) frame by frame; soft estimates
    within the FP32 tolerance (the init dots are split differently)."""
    F, Kn, M, nt, nd = 110, 6, 4, 40, 48
    rx, pil, tx, _ = K.host_frames(list(range(300, 300 + F)), Kn, M, nt, nd, "QPSK")
    pipe = K.FramePipeline(F, Kn, M, nt, nd, "QPSK", precision="f32")
    pipe.load(rx, pil, tx)
    pipe.launch()
    full = pipe.results()
    assert not full["status"].any()
    for i in (0, 57, F - 1):
        p1 = K.FramePipeline(1, Kn, M, nt, nd, "QPSK", precision="f32")
        p1.load(rx[i:i + 1], pil[i:i + 1], tx[i:i + 1])
        p1.launch()
        one = p1.results()
        assert np.array_equal(one["n_active"][0], full["n_active"][i])
        assert np.array_equal(one["labels"][0], full["labels"][i])
        assert np.array_equal(one["bit_err"][0], full["bit_err"][i])
        assert maxrel(full["est"][i], one["est"][0]) <= 1e-4


@pytest.mark.parametrize("prec,tol", [("f32", 1e-5), ("f64", 1e-12)])
def test_overlap_pipeline_matches_fused(prec, tol):
    """The latency pipeline (screen on a side stream + finish) against the
    fused single-stream detection: same decisions and counts; the finish
    recomputes live kernels with explicit differences (FP32: within 1e-5)."""
    seeds = [11, 12]
    rx, pil, tx, _ = K.host_frames(seeds, 6, 16, 120, 256, "QPSK")
    out = []
    for ov in (False, True):
        pipe = K.FramePipeline(2, 6, 16, 120, 256, "QPSK", precision=prec, overlap=ov)
        pipe.load(rx, pil, tx)
        pipe.capture()
        pipe.replay()
        out.append(pipe.results())
    a, b = out
    assert np.array_equal(a["labels"], b["labels"])
    assert np.array_equal(a["bit_err"], b["bit_err"]) and np.array_equal(a["sym_err"], b["sym_err"])
    assert maxrel(b["est"], a["est"]) <= tol


def test_window_limits():
    """W up to kapsm_max_window() trains (the general trainer beyond 23); larger windows are refused."""
    from paper_2201_05024_b200 import _lib
    wmax = _lib.load().kapsm_max_window()
    assert wmax >= 20
    rng = np.random.default_rng(3)
    T, M = 50, 4
    rxp = (rng.standard_normal((T, M)) + 1j * rng.standard_normal((T, M))) / np.sqrt(2)
    sym = (rng.choice([-1, 1], T) + 1j * rng.choice([-1, 1], T)) / np.sqrt(2)
    stream = list(zip(rxp, sym))
    R = O.realify(rxp)
    B = O.realify_targets(sym)
    for W in (wmax, 7):
        f = K.train(None, stream, K.ApsmConfig(window=W), precision="f64")
        ref = O.train_user(R, B, W=W)
        assert f.n_atoms == ref["n_atoms"]
        assert np.array_equal(f.atoms, ref["atoms"])
        assert maxrel(f.coeffs, ref["coeffs"]) <= 1e-9
    with pytest.raises(NotImplementedError):
        K.train(None, stream, K.ApsmConfig(window=wmax + 1), precision="f64")


# --------------------------------------------------------------------------- engine API
def test_engine_golden_random_filter():
    g = np.load(os.path.join(GOLDEN, "engine_random.npz"))
    f = K.FilterState(g["theta"], g["atoms"], g["coeffs"])
    out64 = K.batch_evaluate(f, g["inputs"], P, K.EngineConfig())
    assert maxrel(out64, g["out_f64"]) <= 1e-9
    out32 = K.batch_evaluate(f, g["inputs"], P, K.EngineConfig(precision="f32"))
    assert maxrel(out32, g["out_f64"]) <= 1e-4
    assert out32.dtype == np.float64


@pytest.mark.parametrize("dim", [2, 5, 10, 33, 64])
def test_batch_evaluate_random(dim):
    rng = np.random.default_rng(dim)
    f = K.FilterState(rng.standard_normal(dim), rng.standard_normal((123, dim)) * 0.3,
                      rng.standard_normal(123))
    u = rng.standard_normal((57, dim)) * 0.3
    ref = O.evaluate_batch(f.theta, f.atoms, f.coeffs, u)
    assert maxrel(K.batch_evaluate(f, u, P, K.EngineConfig()), ref) <= 1e-9
    assert maxrel(K.batch_evaluate(f, u, P, K.EngineConfig(precision="f32")), ref) <= 1e-4


def test_batch_detect_and_edges():
    rng = np.random.default_rng(12)
    f = K.FilterState(rng.standard_normal(10), rng.standard_normal((80, 10)) * 0.3,
                      rng.standard_normal(80))
    rx = rng.standard_normal((40, 5)) * 0.3 + 1j * rng.standard_normal((40, 5)) * 0.3
    ref = O.detect_batch(f.theta, f.atoms, f.coeffs, rx)
    out = K.batch_detect(f, rx, P, K.EngineConfig())
    assert maxrel(out, ref) <= 1e-9
    assert K.detect_symbol(f, rx[3], P) == pytest.approx(ref[3], rel=1e-9)
    e = K.batch_detect(K.zero_filter(4), [], P, K.EngineConfig())
    assert e.shape == (0,) and e.dtype == np.complex128
    assert np.all(K.batch_evaluate(K.zero_filter(4), rng.standard_normal((9, 4)), P,
                                   K.EngineConfig()) == 0.0)
    with pytest.raises(ValueError):
        K.batch_evaluate(K.zero_filter(4), np.zeros((3, 5)), P, K.EngineConfig())
    lin = K.KernelParams(1.0, 0.0, 0.05)
    u = rng.standard_normal((15, 10))
    np.testing.assert_allclose(K.batch_evaluate(f, u, lin, K.EngineConfig()), u @ f.theta,
                               rtol=1e-12)


def test_demap_and_ber():
    assert list(K.demodulate_hard(np.array([0j]), "QPSK")) == [0, 0]
    assert list(K.demodulate_hard(np.array([0.9 + 0.8j]), "QPSK")) == [0, 0]
    for scheme in K.SCHEMES:
        con = K.get_constellation(scheme)
        rng = np.random.default_rng(0)
        bits = rng.integers(0, 2, 60 * con.bits_per_symbol)
        assert np.array_equal(K.demodulate_hard(K.modulate(bits, scheme), scheme), bits)
        est = rng.standard_normal(200) + 1j * rng.standard_normal(200)
        assert np.array_equal(K.demodulate_hard(est, scheme), O.demodulate_hard(est, scheme))
    assert K.ber([0, 1, 0], [1, 0, 1]) == 1.0
    assert K.ber([0, 0, 1, 1], [0, 0, 0, 0]) == 0.5
    with pytest.raises(ValueError):
        K.ber([], [])


def test_run_trial_reference_cases():
    """noma.run_trial cases of the reference suite (test_noma.py:245-272)."""
    rng = np.random.default_rng(40)
    ch = K.draw_channel(1, 2, "uniform", 0.0, rng)
    rep = K.run_trial(ch, K.FrameSpec(80, 200, "BPSK"), K.ApsmConfig(), K.EngineConfig(), 0, rng)
    assert rep.ber == 0.0 and rep.trained_atoms > 0 and rep.detect_us > 0
    ch = K.draw_channel(3, 4, "uniform", 0.05, np.random.default_rng(41))
    reps = [K.run_trial(ch, K.FrameSpec(60, 150, "QPSK"), K.ApsmConfig(), K.EngineConfig(), 0,
                        np.random.default_rng(7)) for _ in range(2)]
    assert reps[0].ber == reps[1].ber and reps[0].trained_atoms == reps[1].trained_atoms
    rng = np.random.default_rng(42)
    ch = K.draw_channel(6, 16, "uniform", K.noise_var_for_snr(np.ones(6), 20.0), rng)
    rep = K.run_trial(ch, K.FrameSpec(300, 600, "QPSK"), K.ApsmConfig(), K.EngineConfig(), 0, rng)
    assert rep.ber < 1e-2
    with pytest.raises(ValueError):
        K.run_trial(K.draw_channel(2, 2, "uniform", 0.0, np.random.default_rng(43)),
                    K.FrameSpec(10, 10), K.ApsmConfig(), K.EngineConfig(), 5,
                    np.random.default_rng(0))


def test_frame_stream_matches_pipeline():
    """FrameStream (overlapped pinned H2D/D2H) == one FramePipeline per frame."""
    import torch
    Kk, M, nt, nd = 3, 8, 120, 200
    rx, pil, tx, _ = K.host_frames(range(5), Kk, M, nt, nd, "QPSK")
    rx_p = torch.from_numpy(np.stack([rx.real, rx.imag], -1).astype(np.float32)).pin_memory()
    pil_p = torch.from_numpy(np.stack([pil.real, pil.imag], -1).astype(np.float32)).pin_memory()
    tx_p = torch.from_numpy(tx.astype(np.uint8)).pin_memory()
    fs = K.FrameStream(Kk, M, nt, nd, "QPSK", depth=2)
    ref = K.FramePipeline(1, Kk, M, nt, nd, "QPSK", precision="f32")
    got = []
    for i in range(5):
        t = fs.submit(rx_p[i:i + 1], pil_p[i:i + 1], tx_p[i:i + 1])
        if i >= 1:
            lab, be, se = fs.result(t - 1)
            got.append((t - 1, lab.clone(), be.clone(), se.clone()))
    lab, be, se = fs.result(4)
    got.append((4, lab.clone(), be.clone(), se.clone()))
    with pytest.raises(ValueError):
        fs.result(0)
    # device-resident frames: read in place by direct launches, concurrent slots
    fd = K.FrameStream(Kk, M, nt, nd, "QPSK", depth=3, concurrent=True)
    rx_d, pil_d, tx_d = rx_p.cuda(), pil_p.cuda(), tx_p.cuda()
    dev_got = {}
    for i in range(5):
        t = fd.submit(rx_d[i:i + 1], pil_d[i:i + 1], tx_d[i:i + 1])
        if i >= 2:
            lab, be, _ = fd.result(t - 2)
            dev_got[t - 2] = (lab.clone(), be.clone())
    for t in (3, 4):
        lab, be, _ = fd.result(t)
        dev_got[t] = (lab.clone(), be.clone())
    for i, lab, be, se in got:
        assert np.array_equal(dev_got[i][0].numpy(), lab.numpy())
        assert np.array_equal(dev_got[i][1].numpy(), be.numpy())
    for i, lab, be, se in got:
        ref.load(rx[i:i + 1], pil[i:i + 1], tx[i:i + 1])
        ref.launch()
        r = ref.results(est=False)
        assert np.array_equal(lab.numpy(), r["labels"])
        assert np.array_equal(be.numpy(), r["bit_err"]) and np.array_equal(se.numpy(), r["sym_err"])


def test_frame_stream_batched_exchange_hook():
    """The N > 1 bench hook at world 1: BatchedExchange on the FrameStream's
    collective stream sees every frame's decisions and counters in order."""
    import torch
    from paper_2201_05024_b200 import dist as D
    Kk, M, nt, nd = 3, 8, 120, 200
    rx, pil, tx, _ = K.host_frames(range(8), Kk, M, nt, nd, "QPSK")
    rx_p = torch.from_numpy(np.stack([rx.real, rx.imag], -1).astype(np.float32)).pin_memory()
    pil_p = torch.from_numpy(np.stack([pil.real, pil.imag], -1).astype(np.float32)).pin_memory()
    tx_p = torch.from_numpy(tx.astype(np.uint8)).pin_memory()
    ex = D.BatchedExchange(4, (Kk, nd), torch.device("cuda"))
    fs = K.FrameStream(Kk, M, nt, nd, "QPSK", depth=3, concurrent=True,
                       post=lambda p: ex.add(p.labels, torch.cat([p.bit_err[0], p.sym_err[0]])))
    labs, errs = [], []
    for i in range(8):
        t = fs.submit(rx_p[i:i + 1], pil_p[i:i + 1], tx_p[i:i + 1])
        lab, be, se = fs.result(t)
        labs.append(lab.clone())
        errs.append(torch.cat([be[0], se[0]]).clone())
    torch.cuda.synchronize()
    assert ex.n == 8
    assert np.array_equal(ex.gathered[0].cpu().numpy(), torch.cat(labs[4:]).numpy())
    assert np.array_equal(ex.totals.cpu().numpy(), sum(e.numpy() for e in errs[4:]))


def test_launch_on_device_frames_in_place():
    """FramePipeline.launch_on reads device-resident frames in place (no copy
    into the static buffers) and matches load + launch; bad tensors raise."""
    import torch
    Kk, M, nt, nd = 3, 8, 120, 200
    rx, pil, tx, _ = K.host_frames([21], Kk, M, nt, nd, "QPSK")
    p = K.FramePipeline(1, Kk, M, nt, nd, "QPSK", precision="f32")
    p.load(rx, pil, tx)
    p.launch()
    ref = p.results(est=True)
    rx_d = torch.from_numpy(np.stack([rx.real, rx.imag], -1).astype(np.float32)).cuda()
    pil_d = torch.from_numpy(np.stack([pil.real, pil.imag], -1).astype(np.float32)).cuda()
    tx_d = torch.from_numpy(tx.astype(np.uint8)).cuda()
    q = K.FramePipeline(1, Kk, M, nt, nd, "QPSK", precision="f32")
    q.launch_on(rx_d, pil_d, tx_d)
    got = q.results(est=True)
    assert np.array_equal(got["labels"], ref["labels"])
    assert np.array_equal(got["bit_err"], ref["bit_err"])
    assert np.array_equal(got["est"], ref["est"])
    with pytest.raises(ValueError):
        q.launch_on(rx_d.double(), pil_d, tx_d)


@pytest.mark.parametrize("labels_in", [False, True])
def test_frame_stream_batches_throughput_mode(labels_in):
    """FrameStream(frames=F) with F x K > SMs (the bench's e2e path: the
    one-warp trainer inside the captured pipelines), fed from the pinned ring
    of FrameGenerator -- with complex pilot targets, or (the bench's e2e) with
    pilot labels expanded on the device: every batch's decisions and counts
    equal one FramePipeline launch per batch on the complex targets."""
    from paper_2201_05024_b200.framegen import FrameGenerator
    F, Kk, M, nt, nd = 30, 6, 16, 200, 160          # 180 chains > 148 SMs
    gen = FrameGenerator(F, Kk, M, nt, nd, "QPSK", slots=2, workers=2)
    try:
        fs = K.FrameStream(Kk, M, nt, nd, "QPSK", depth=2, concurrent=True, frames=F,
                           pilot_labels=labels_in)
        seeds = [list(range(700 + F * b, 700 + F * (b + 1))) for b in range(3)]
        out = []
        for b in range(3):
            gen.fill(b % 2, seeds[b]).wait()
            t = fs.submit(gen.rx[b % 2], (gen.plab if labels_in else gen.pilots)[b % 2],
                          gen.tx[b % 2])
            lab, be, se = fs.result(t)
            out.append((lab.clone(), be.clone(), se.clone()))
        for b in range(3):
            rx, pil, tx, _ = K.host_frames(seeds[b], Kk, M, nt, nd, "QPSK")
            ref = K.FramePipeline(F, Kk, M, nt, nd, "QPSK", precision="f32", store_est=False)
            ref.load(rx, pil, tx)
            ref.launch()
            r = ref.results(est=False)
            assert np.array_equal(out[b][0].numpy(), r["labels"])
            assert np.array_equal(out[b][1].numpy(), r["bit_err"])
            assert np.array_equal(out[b][2].numpy(), r["sym_err"])
    finally:
        gen.close()



def test_pipeline_pilot_labels_equal_targets():
    """FramePipeline(pilot_labels=True): the targets expanded on the device
    from the pilot labels (kapsm_targets_from_labels) are the complex targets,
    bit for bit, and the whole pipeline's outputs are identical."""
    from paper_2201_05024_b200.noma import seeded_frame, symbol_labels
    Kk, M, nt, nd, sch = 6, 16, 150, 200, "QAM16"
    seeds = [41, 42]
    rx, pil, tx, _ = K.host_frames(seeds, Kk, M, nt, nd, sch)
    k = 4
    plab = np.stack([symbol_labels(seeded_frame(s, Kk, M, nt, nd, sch)["bits"][:, :nt * k], k)
                     for s in seeds]).astype(np.uint8)
    a = K.FramePipeline(2, Kk, M, nt, nd, sch, precision="f32")
    a.load(rx, pil, tx)
    a.launch()
    b = K.FramePipeline(2, Kk, M, nt, nd, sch, precision="f32", pilot_labels=True)
    b.load(rx, plab, tx)
    b.launch()
    torch.cuda.synchronize()
    assert torch.equal(a.pilots, b.pilots)
    ra, rb = a.results(), b.results()
    for key in ("labels", "bit_err", "n_active", "est", "theta", "coeff"):
        assert np.array_equal(ra[key], rb[key]), key
