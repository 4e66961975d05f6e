"""Round-2 golden fixtures from the UNMODIFIED reference package.

Run in the build container (where the reference is importable):

    PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=1 \
        python tests/golden/make_golden_r2.py

Writes
* ``c4_s0_users0123.npz`` -- the massive-MIMO config C4 (K=16, M=64, 16-QAM,
  685 pilots / 3840 data, seed 0): trained filters (theta, coeffs, atom pilot
  indices in slot order), soft estimates, bit errors of users 0-3;
* ``c1_seeds20.npz`` -- the paper config C1 (K=6, M=16, QPSK) on seeds 0..19,
  every user: n_atoms, bit / symbol errors, the full decision labels and the
  soft estimates of every 8th payload symbol (+ max |est| of the full frame);
* ``c4_s0_all_users.npz`` -- the same per-user table for C4 seed 0, all 16
  users;
* ``trial_anchors.npz`` -- ``run_trial`` exactly as the reference acceptance
  suite drives it (pkg/tests/test_acceptance.py:63-75, criteria 5/6/7 at
  :272-312): per-seed BER and trained_atoms for every (scheme, M, params)
  cell over seeds 0..19, with the default float64 engine and with
  ``EngineConfig(precision="f32")``.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time

import numpy as np

import kapsm  # the reference package
from kapsm import (ApsmConfig, EngineConfig, FrameSpec, KernelParams, batch_detect,
                   demodulate_hard, draw_channel, modulate, run_trial, synthesize_received,
                   train, zero_filter)

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import atom_index, frame  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
SUB = 8                         # soft estimates kept for every SUB-th payload symbol

# test_acceptance.py:40-53 constants
NOISE_VAR = 0.06
N_TRAIN, N_DATA = 685, 3840
PARTIAL = KernelParams(0.5, 0.5, 0.05)
LINEAR = KernelParams(1.0, 0.0, 0.05)
# (scheme, scheme_idx, M, params) cells of criteria 5, 6, 7
CELLS = [("BPSK", 0, 16, "partial"), ("QPSK", 1, 16, "partial"), ("QAM16", 2, 16, "partial"),
         ("QPSK", 1, 4, "partial"), ("QPSK", 1, 8, "partial"), ("QPSK", 1, 12, "partial"),
         ("QPSK", 1, 3, "partial"), ("QPSK", 1, 3, "linear")]


def c1_user(args, K=6, M=16, scheme="QPSK"):
    seed, u = args
    bits, symbols, rx, k = frame(seed, K, M, scheme, N_TRAIN, N_DATA)
    f = train(zero_filter(2 * M), zip(rx[:N_TRAIN], symbols[u, :N_TRAIN]), ApsmConfig())
    est = batch_detect(f, rx[N_TRAIN:], PARTIAL, EngineConfig())
    rb = demodulate_hard(est, scheme).reshape(-1, k)
    tb = bits[u, N_TRAIN * k:].reshape(-1, k)
    lab = (rb * (1 << np.arange(k - 1, -1, -1))).sum(1).astype(np.uint8)
    return (seed, u, f.n_atoms, int(np.sum(rb != tb)), int(np.sum(np.any(rb != tb, 1))), lab,
            est[::SUB].copy(), float(np.max(np.abs(est))))


def c4_user(args):
    return c1_user(args, 16, 64, "QAM16")


def seeds_table(pool, fn, seeds, K):
    """Per (seed, user): n_atoms, bit/symbol errors, labels, every SUB-th soft estimate."""
    res = pool.map(fn, [(s, u) for s in seeds for u in range(K)], chunksize=1)
    S = len(seeds)
    n = np.zeros((S, K), np.int64)
    be = np.zeros((S, K), np.int64)
    se = np.zeros((S, K), np.int64)
    lab = np.zeros((S, K, N_DATA), np.uint8)
    est = np.zeros((S, K, N_DATA // SUB), np.complex128)
    emax = np.zeros((S, K))
    for seed, u, na, b, s, lb, es, em in res:
        i = seeds.index(seed)
        n[i, u], be[i, u], se[i, u] = na, b, s
        lab[i, u], est[i, u], emax[i, u] = lb, es, em
    return dict(seeds=np.asarray(seeds), n_atoms=n, bit_err=be, sym_err=se, labels=lab,
                est_sub=est.astype(np.complex64), est_max=emax, sub=SUB)


def anchor(args):
    """One run_trial of the acceptance suite, replayed twice: the float64
    engine (run_trial itself) and the float32 engine (same rng state)."""
    cell, seed = args
    scheme, si, m, pname = CELLS[cell]
    params = PARTIAL if pname == "partial" else LINEAR
    out = []
    for eng in (EngineConfig(), EngineConfig(precision="f32")):
        rng = np.random.default_rng([seed, si, m])
        ch = draw_channel(6, m, "uniform", NOISE_VAR, rng)
        rep = run_trial(ch, FrameSpec(N_TRAIN, N_DATA, scheme), ApsmConfig(params=params), eng,
                        0, rng)
        out.append((rep.ber, rep.trained_atoms))
    return cell, seed, out[0][0], out[1][0], out[0][1]


def main():
    t0 = time.time()
    ctx = mp.get_context("fork")
    with ctx.Pool(os.cpu_count()) as pool:
        # ---- C1, 20 seeds x 6 users; C4, seed 0 x 16 users ----
        np.savez_compressed(os.path.join(HERE, "c1_seeds20.npz"),
                            **seeds_table(pool, c1_user, list(range(20)), 6))
        np.savez_compressed(os.path.join(HERE, "c4_s0_all_users.npz"),
                            **seeds_table(pool, c4_user, [0], 16))
        print(f"c1 / c4 seed tables done {time.time() - t0:.0f}s", file=sys.stderr)
        if "--tables-only" in sys.argv:
            return

        # ---- run_trial anchors ----
        res = pool.map(anchor, [(c, s) for c in range(len(CELLS)) for s in range(20)],
                       chunksize=1)
        b64 = np.zeros((len(CELLS), 20))
        b32 = np.zeros((len(CELLS), 20))
        na = np.zeros((len(CELLS), 20), np.int64)
        for c, s, x64, x32, a in res:
            b64[c, s], b32[c, s], na[c, s] = x64, x32, a
        np.savez_compressed(os.path.join(HERE, "trial_anchors.npz"),
                            cells=np.array([f"{a}|{b}|{c}|{d}" for a, b, c, d in CELLS]),
                            ber_f64=b64, ber_f32=b32, trained_atoms=na)
        print(f"anchors done {time.time() - t0:.0f}s; means f64 "
              f"{np.round(b64.mean(1), 6).tolist()}", file=sys.stderr)

    # ---- C4 paper frame, users 0-3 ----
    K, M, scheme = 16, 64, "QAM16"
    bits, symbols, rx, k = frame(0, K, M, scheme, N_TRAIN, N_DATA)
    R = kapsm.realify_batch(rx[:N_TRAIN])
    out = dict(seed=0, K=K, M=M, scheme=scheme, n_train=N_TRAIN, n_data=N_DATA,
               rx_head=rx[:4].copy(), users=np.arange(4))
    for u in range(4):
        f = train(zero_filter(2 * M), zip(rx[:N_TRAIN], symbols[u, :N_TRAIN]), ApsmConfig())
        e = batch_detect(f, rx[N_TRAIN:], PARTIAL, EngineConfig())
        rb = demodulate_hard(e, scheme)
        out[f"u{u}_theta"] = f.theta
        out[f"u{u}_coeffs"] = f.coeffs
        out[f"u{u}_atom_idx"] = atom_index(f.atoms, R)
        out[f"u{u}_n_atoms"] = f.n_atoms
        out[f"u{u}_est"] = e
        out[f"u{u}_bit_err"] = int(np.sum(rb != bits[u, N_TRAIN * k:]))
    np.savez_compressed(os.path.join(HERE, "c4_s0_users0123.npz"), **out)
    print(f"all done {time.time() - t0:.0f}s", file=sys.stderr)


if __name__ == "__main__":
    main()
