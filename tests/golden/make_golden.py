"""Generate golden vectors from the UNMODIFIED reference package.

Run in the build container (where the reference is importable):

    PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=1 \
        python tests/golden/make_golden.py

It imports ``kapsm`` (the reference, /root/reference/pkg/src/kapsm) and writes
``tests/golden/*.npz``.  These fixtures pin the CPU oracle
(``oracle/kapsm_oracle.py``) and, through it, the CUDA path.  The reference
itself is never needed on the GPU box.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

import kapsm  # the reference package
from kapsm import (ApsmConfig, EngineConfig, FilterState, KernelParams, batch_detect,
                   batch_evaluate, demodulate_hard, draw_channel, modulate, noise_var_for_snr,
                   synthesize_received, train, uniform_weights, zero_filter, realify_batch)

HERE = os.path.dirname(os.path.abspath(__file__))
SCHEME_IDX = {"BPSK": 0, "QPSK": 1, "QAM16": 2, "QAM64": 3}


def frame(seed, K, M, scheme, n_train, n_data, snr_db=20.0):
    """run_trial's RNG order (noma.py:267-269) with the acceptance seeding
    (test_acceptance.py:69)."""
    rng = np.random.default_rng([seed, SCHEME_IDX[scheme], M])
    ch = draw_channel(K, M, "uniform", noise_var_for_snr(np.ones(K), snr_db), rng)
    k = kapsm.get_constellation(scheme).bits_per_symbol
    t = n_train + n_data
    bits = rng.integers(0, 2, size=(K, t * k))
    symbols = np.stack([modulate(bits[u], scheme) for u in range(K)])
    rx = synthesize_received(symbols, ch, rng)
    return bits, symbols, rx, k


def atom_index(atoms, R):
    """Map each trained atom back to the realified pilot row it copies."""
    idx = np.empty(atoms.shape[0], dtype=np.int64)
    for a in range(atoms.shape[0]):
        hit = np.nonzero(np.all(R == atoms[a], axis=1))[0]
        assert hit.size >= 1
        idx[a] = hit[0]
    return idx


def per_frame(seed, K, M, scheme, n_train, n_data, users, store_rx, cfg=None):
    bits, symbols, rx, k = frame(seed, K, M, scheme, n_train, n_data)
    cfg = cfg or ApsmConfig()
    R = realify_batch(rx[:n_train])
    out = dict(seed=seed, K=K, M=M, scheme=scheme, n_train=n_train, n_data=n_data,
               rx_sha=hashlib.sha256(np.ascontiguousarray(rx).tobytes()).hexdigest(),
               rx_head=rx[:4].copy(), users=np.asarray(users))
    if store_rx:
        out.update(rx=rx, bits=bits)
    for u in users:
        f = train(zero_filter(2 * M), zip(rx[:n_train], symbols[u, :n_train]), cfg)
        est = batch_detect(f, rx[n_train:], cfg.params, EngineConfig())
        rx_bits = demodulate_hard(est, scheme)
        tx_bits = bits[u, n_train * k:]
        out[f"u{u}_theta"] = f.theta
        out[f"u{u}_coeffs"] = f.coeffs
        out[f"u{u}_atom_idx"] = atom_index(f.atoms, R)
        out[f"u{u}_n_atoms"] = f.n_atoms
        out[f"u{u}_est"] = est
        out[f"u{u}_bit_err"] = int(np.sum(rx_bits != tx_bits))
    return out


def main():
    # Small frames: full data stored (CPU-fast; used by CPU + GPU parity tests).
    small = [
        (0, 3, 4, "QPSK", 40, 64),
        (1, 6, 3, "QPSK", 60, 100),     # overloaded cell (K > M), live Gaussian terms
        (2, 4, 8, "QAM16", 80, 120),
        (3, 2, 2, "BPSK", 30, 50),
        (4, 6, 16, "QPSK", 100, 160),   # paper antenna/user geometry, short frame
    ]
    for (seed, K, M, scheme, nt, nd) in small:
        d = per_frame(seed, K, M, scheme, nt, nd, list(range(K)), True)
        np.savez_compressed(os.path.join(HERE, f"small_s{seed}_K{K}_M{M}_{scheme}.npz"), **d)
    # Paper scenario C1 (K=6, M=16, QPSK, 685/3840): two users, rx regenerated from the seed.
    d = per_frame(0, 6, 16, "QPSK", 685, 3840, [0, 1], False)
    np.savez_compressed(os.path.join(HERE, "c1_s0_users01.npz"), **d)

    # Known answers for uniform_weights (apsm.py:139-153).
    np.savez_compressed(os.path.join(HERE, "uniform_weights.npz"),
                        **{f"w{n}": uniform_weights(n) for n in range(1, 161)})

    # Engine: random filter, f64 and f32 batch_evaluate (engine.py:206-243).
    rng = np.random.default_rng(2024)
    f = FilterState(rng.standard_normal(10), rng.standard_normal((123, 10)) * 0.3,
                    rng.standard_normal(123))
    u = rng.standard_normal((57, 10)) * 0.3
    p = KernelParams(0.5, 0.5, 0.05)
    np.savez_compressed(os.path.join(HERE, "engine_random.npz"), theta=f.theta, atoms=f.atoms,
                        coeffs=f.coeffs, inputs=u,
                        out_f64=batch_evaluate(f, u, p, EngineConfig(stage="baseline")),
                        out_f32=batch_evaluate(f, u, p, EngineConfig(precision="f32")))
    print("golden fixtures written to", HERE, file=sys.stderr)


if __name__ == "__main__":
    main()
