"""Pin the CPU oracle (oracle/kapsm_oracle.py) against golden vectors made by the
unmodified reference (tests/golden/make_golden.py) and against the reference's
own known-answer tests.  CPU only."""

import glob
import hashlib
import os

import numpy as np
import pytest

from oracle import kapsm_oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
SMALL = sorted(glob.glob(os.path.join(GOLDEN, "small_*.npz")))


def _frame_of(g):
    fr = O.make_frame(int(g["seed"]), int(g["K"]), int(g["M"]), int(g["n_train"]),
                      int(g["n_data"]), str(g["scheme"]))
    return fr


@pytest.mark.parametrize("path", SMALL, ids=[os.path.basename(p) for p in SMALL])
def test_small_frames_match_reference(path):
    g = np.load(path)
    fr = _frame_of(g)
    # seeded inputs are bit-identical to the reference's
    assert np.array_equal(fr["rx"], g["rx"])
    assert np.array_equal(fr["bits"], g["bits"])
    res = O.run_frame(fr, int(g["n_train"]), str(g["scheme"]), users=list(g["users"]))
    for r in res:
        u = r["user"]
        m = r["model"]
        assert m["n_atoms"] == int(g[f"u{u}_n_atoms"])
        assert np.array_equal(m["slot_index"], g[f"u{u}_atom_idx"])       # slot order
        np.testing.assert_allclose(m["theta"], g[f"u{u}_theta"], rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(m["coeffs"], g[f"u{u}_coeffs"], rtol=1e-11, atol=1e-13)
        est = g[f"u{u}_est"]
        assert np.max(np.abs(r["est"] - est)) <= 1e-12 * np.max(np.abs(est))
        assert r["bit_err"] == int(g[f"u{u}_bit_err"])


def test_c1_paper_frame_users01():
    """Paper scenario (K=6, M=16, QPSK, 685/3840): the oracle reproduces the
    reference's trained filters and decisions for users 0 and 1."""
    g = np.load(os.path.join(GOLDEN, "c1_s0_users01.npz"))
    fr = _frame_of(g)
    assert hashlib.sha256(np.ascontiguousarray(fr["rx"]).tobytes()).hexdigest() == str(g["rx_sha"])
    res = O.run_frame(fr, 685, "QPSK", users=[0, 1])
    for r in res:
        u = r["user"]
        assert r["model"]["n_atoms"] == int(g[f"u{u}_n_atoms"])
        assert np.array_equal(r["model"]["slot_index"], g[f"u{u}_atom_idx"])
        est = g[f"u{u}_est"]
        assert np.max(np.abs(r["est"] - est)) <= 1e-12 * np.max(np.abs(est))
        assert r["bit_err"] == int(g[f"u{u}_bit_err"])


def test_uniform_weights_known_answers():
    g = np.load(os.path.join(GOLDEN, "uniform_weights.npz"))
    for n in range(1, 161):
        w = O.uniform_weights(n)
        assert np.array_equal(w, g[f"w{n}"])
        assert float(np.sum(w)) == 1.0


def test_engine_random_filter():
    g = np.load(os.path.join(GOLDEN, "engine_random.npz"))
    out = O.evaluate_batch(g["theta"], g["atoms"], g["coeffs"], g["inputs"])
    np.testing.assert_allclose(out, g["out_f64"], rtol=1e-12, atol=1e-13)


def test_reference_known_answers():
    # complex_to_real_pair example (test_apsm.py:65-70) via realify
    r = O.realify(np.array([[1 + 2j]]))
    assert np.array_equal(r, [[1.0, 2.0], [2.0, -1.0]])
    assert np.array_equal(O.realify_targets([3 + 4j]), [3.0, 4.0])
    # QPSK table (test_noma.py:70-80), origin tie -> 00 (test_noma.py:125-127)
    s = 1 / np.sqrt(2)
    assert np.allclose(O.modulate([0, 0, 0, 1, 1, 1, 1, 0], "QPSK"),
                       [(1 + 1j) * s, (-1 + 1j) * s, (-1 - 1j) * s, (1 - 1j) * s])
    assert list(O.demodulate_hard(np.array([0j]), "QPSK")) == [0, 0]
    # 16-QAM axis convention (test_noma.py:82-85)
    s = 1 / np.sqrt(10)
    assert np.allclose(O.modulate([0, 0, 0, 0, 1, 0, 0, 1], "QAM16"), [(-3 - 3j) * s, (3 - 1j) * s])
    # beta: single unit sample, zero filter, eps 0.1 (test_apsm.py:101-110)
    m = O.train_user(np.array([[1.0, 0.0]]), np.array([1.0]), W=1, eps=0.1)
    assert abs(m["coeff"][0] - 0.9) < 1e-15
    m = O.train_user(np.array([[1.0, 0.0]]), np.array([0.05]), W=1, eps=0.1)
    assert m["coeff"][0] == 0.0 and m["n_atoms"] == 0
    m = O.train_user(np.array([[1.0, 0.0]]), np.array([-1.0]), W=1, eps=0.1)
    assert abs(m["coeff"][0] + 0.9) < 1e-15


def test_c1_seed_table_spot_checks():
    """The oracle reproduces the reference's C1 seed table (c1_seeds20.npz,
    tests/golden/make_golden_r2.py) on two (seed, user) pairs."""
    g = np.load(os.path.join(GOLDEN, "c1_seeds20.npz"))
    sub = int(g["sub"])
    for seed, u in ((7, 3), (19, 5)):
        fr = O.make_frame(seed, 6, 16, 685, 3840, "QPSK")
        r = O.run_frame(fr, 685, "QPSK", users=[u])[0]
        assert r["model"]["n_atoms"] == int(g["n_atoms"][seed, u])
        assert r["bit_err"] == int(g["bit_err"][seed, u])
        assert r["sym_err"] == int(g["sym_err"][seed, u])
        assert np.array_equal(r["rx_idx"], g["labels"][seed, u])
        dev = np.max(np.abs(r["est"][::sub] - g["est_sub"][seed, u])) / g["est_max"][seed, u]
        assert dev < 1e-6                      # fixture stored as complex64


def test_c4_massive_frame_user0():
    """C4 (K=16, M=64, 16-QAM): the oracle reproduces the reference's user-0
    filter (slot order) and soft estimates."""
    g = np.load(os.path.join(GOLDEN, "c4_s0_users0123.npz"))
    fr = O.make_frame(0, 16, 64, 685, 3840, "QAM16")
    assert np.array_equal(fr["rx"][:4], g["rx_head"])
    r = O.run_frame(fr, 685, "QAM16", users=[0])[0]
    assert r["model"]["n_atoms"] == int(g["u0_n_atoms"])
    assert np.array_equal(r["model"]["slot_index"], g["u0_atom_idx"])
    np.testing.assert_allclose(r["model"]["theta"], g["u0_theta"], rtol=1e-11, atol=1e-13)
    assert np.max(np.abs(r["est"] - g["u0_est"])) <= 1e-11 * np.max(np.abs(g["u0_est"]))
    assert r["bit_err"] == int(g["u0_bit_err"])


def test_trial_anchor_means_match_frozen_log():
    """trial_anchors.npz (reference run_trial, 20 seeds per cell) reproduces
    the frozen acceptance means of pkg/test_output.txt:246-248, and the
    float32 engine gives the same per-seed BER as the float64 one."""
    g = np.load(os.path.join(GOLDEN, "trial_anchors.npz"))
    m = dict(zip([str(c) for c in g["cells"]], g["ber_f64"].mean(1)))
    assert m["BPSK|0|16|partial"] == 0 and m["QPSK|1|16|partial"] == 0
    assert f"{m['QAM16|2|16|partial']:.2e}" == "3.26e-06"
    assert f"{m['QPSK|1|4|partial']:.2e}" == "1.74e-01"
    assert f"{m['QPSK|1|3|partial']:.4f}" == "0.2058" and f"{m['QPSK|1|3|linear']:.4f}" == "0.2133"
    assert np.array_equal(g["ber_f64"], g["ber_f32"])
