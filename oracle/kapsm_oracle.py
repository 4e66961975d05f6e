"""CPU oracle for the APSM partially linear multiuser detector hot path.

TEST INFRASTRUCTURE ONLY.  This module is a float64 numpy restatement of the
reference algorithm (``/root/reference/pkg/src/kapsm``) used as the checker for
the CUDA path.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it.
The product package ``paper_2201_05024_b200`` never imports it: the product
path fails loudly when its CUDA library is missing.

Parity pinning: every function below is checked against golden vectors
produced by the unmodified reference (``tests/golden/make_golden.py`` ->
``tests/golden/*.npz``) and against the reference's own known-answer tests
(``tests/test_oracle_golden.py``).

Each function cites the reference ``file:line`` it restates (paths relative to
``/root/reference/pkg/src/kapsm``).
"""

from __future__ import annotations

import numpy as np

# ---------------------------------------------------------------------------
# constellations (noma.py:57-107)
# ---------------------------------------------------------------------------

_AXIS2 = {0: -3.0, 1: -1.0, 3: 1.0, 2: 3.0}          # noma.py:57  (Gray 00,01,11,10)
_AXIS3 = {0: -7.0, 1: -5.0, 3: -3.0, 2: -1.0,          # noma.py:58-67
          6: 1.0, 7: 3.0, 5: 5.0, 4: 7.0}
SCHEMES = ("BPSK", "QPSK", "QAM16", "QAM64")          # noma.py:52


def constellation(scheme: str):
    """(points complex128[Q], bits_per_symbol) -- noma.py:86-102."""
    if scheme == "BPSK":
        return np.array([1.0 + 0j, -1.0 + 0j]), 1
    if scheme == "QPSK":
        return np.array([1 + 1j, -1 + 1j, 1 - 1j, -1 - 1j]) / np.sqrt(2.0), 2
    if scheme in ("QAM16", "QAM64"):
        half = 2 if scheme == "QAM16" else 3
        axis = _AXIS2 if half == 2 else _AXIS3
        scale = 1.0 / np.sqrt(10.0 if half == 2 else 42.0)
        n = 1 << (2 * half)
        pts = np.empty(n, dtype=np.complex128)
        for idx in range(n):
            pts[idx] = scale * (axis[idx >> half] + 1j * axis[idx & ((1 << half) - 1)])
        return pts, 2 * half
    raise ValueError(scheme)


def modulate(bits, scheme):
    """MSB-first label -> point (noma.py:110-122)."""
    pts, k = constellation(scheme)
    bits = np.asarray(bits, dtype=np.int64)
    idx = bits.reshape(-1, k) @ (1 << np.arange(k - 1, -1, -1))
    return pts[idx]


def demap_indices(est, scheme):
    """argmin |est - p| with lowest-index tie break (noma.py:125-135)."""
    pts, _ = constellation(scheme)
    est = np.atleast_1d(np.asarray(est, dtype=np.complex128))
    return np.abs(est[:, None] - pts[None, :]).argmin(axis=1)


def demodulate_hard(est, scheme):
    """Hard decision bits, MSB first (noma.py:125-135)."""
    _, k = constellation(scheme)
    idx = demap_indices(est, scheme)
    shifts = np.arange(k - 1, -1, -1)
    return ((idx[:, None] >> shifts) & 1).astype(np.int64).reshape(-1)


def ber(tx_bits, rx_bits):
    """noma.py:284-292."""
    return float(np.mean(np.asarray(tx_bits) != np.asarray(rx_bits)))


# ---------------------------------------------------------------------------
# seeded frame generation in run_trial's RNG order (noma.py:195-246, 267-269)
# ---------------------------------------------------------------------------

def noise_var_for_snr(powers, snr_db):
    """noma.py:216-226."""
    return float(np.sum(np.asarray(powers, dtype=np.float64))) / 10.0 ** (snr_db / 10.0)


def make_frame(seed, K, M, n_train, n_data, scheme, snr_db=20.0, scheme_idx=None):
    """One frame exactly as the reference acceptance suite builds it.

    rng = default_rng([seed, scheme_idx, M]) (test_acceptance.py:69);
    draw_channel (noma.py:206-213) then bits/modulate/synthesize in the order
    of run_trial (noma.py:267-269).  Returns dict with h, bits (K x T*k),
    symbols (K x T), rx (T x M).
    """
    if scheme_idx is None:
        scheme_idx = {"BPSK": 0, "QPSK": 1, "QAM16": 2, "QAM64": 3}[scheme]
    rng = np.random.default_rng([seed, scheme_idx, M])
    nv = noise_var_for_snr(np.ones(K), snr_db)
    h = (rng.standard_normal((K, M)) + 1j * rng.standard_normal((K, M))) / np.sqrt(2.0)
    p = np.ones(K)
    _, k = constellation(scheme)
    t = n_train + n_data
    bits = rng.integers(0, 2, size=(K, t * k))
    symbols = np.stack([modulate(bits[u], scheme) for u in range(K)])
    rx = symbols.T @ (np.sqrt(p)[:, None] * h)
    if nv > 0:
        scale = np.sqrt(nv / 2.0)
        rx = rx + scale * (rng.standard_normal((t, M)) + 1j * rng.standard_normal((t, M)))
    return dict(h=h, bits=bits, symbols=symbols, rx=rx, noise_var=nv, bps=k)


# ---------------------------------------------------------------------------
# realification (apsm.py:156-182)
# ---------------------------------------------------------------------------

def realify(rx):
    """Row 2t = [Re; Im], row 2t+1 = [Im; -Re] (apsm.py:172-182)."""
    rx = np.atleast_2d(np.asarray(rx, dtype=np.complex128))
    out = np.empty((2 * rx.shape[0], 2 * rx.shape[1]))
    out[0::2] = np.hstack([rx.real, rx.imag])
    out[1::2] = np.hstack([rx.imag, -rx.real])
    return out


def realify_targets(b):
    """Targets Re b, Im b interleaved (apsm.py:167-169)."""
    b = np.asarray(b, dtype=np.complex128)
    out = np.empty(2 * b.shape[0])
    out[0::2] = b.real
    out[1::2] = b.imag
    return out


# ---------------------------------------------------------------------------
# APSM trainer (apsm.py:132-153, 254-372)
# ---------------------------------------------------------------------------

def uniform_weights(count):
    """1/count with the rounding defect folded into the last entry until the
    numpy sum is exactly 1.0 (apsm.py:139-153)."""
    w = np.full(count, 1.0 / count)
    for _ in range(10):
        defect = 1.0 - float(np.sum(w))
        if defect == 0.0:
            break
        w[-1] += defect
    return w


def train_user(R, B, W=20, eps=0.01, w_l=0.5, w_g=0.5, sigma_sq=0.05, max_atoms=None):
    """Run the APSM trainer over realified samples R (N x D) with targets B.

    Restates ApsmTrainer.observe (apsm.py:304-359) with a zero warm start:
    window J_n = [max(0, n-W+1), n] (apsm.py:132-136), response of the
    current filter on the window (apsm.py:288-302), three-case beta
    (apsm.py:329-332), uniform weights (apsm.py:139-153), theta update
    (apsm.py:338) and first-activation slots (apsm.py:341-359).

    Returns dict(theta, coeff (per sample, 0 if never active), first_step
    (-1 if never), atoms/coeffs in slot order, n_atoms, capacity_error).
    """
    R = np.asarray(R, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    N, D = R.shape
    inv2s = 1.0 / (2.0 * sigma_sq)
    theta = np.zeros(D)
    norms = np.einsum("ij,ij->i", R, R)
    coeff = np.zeros(N)
    first = np.full(N, -1, dtype=np.int64)
    slots = []          # sample index per slot, in creation order
    cap_err = False
    for n in range(N):
        lo = max(0, n - W + 1)
        rw = R[lo:n + 1]
        y = rw @ theta
        if w_g != 0.0 and slots:
            idx = np.asarray(slots)
            d2 = norms[idx][:, None] + norms[lo:n + 1][None, :] - 2.0 * (R[idx] @ rw.T)
            np.maximum(d2, 0.0, out=d2)
            y = y + w_g * (coeff[idx] @ np.exp(-d2 * inv2s))
        res = y - B[lo:n + 1]
        den = w_l * norms[lo:n + 1] + w_g
        if np.any(den <= 0.0):
            raise ValueError("degenerate sample")
        beta = np.where(res < -eps, (-res - eps) / den, np.where(res > eps, (-res + eps) / den, 0.0))
        active = np.nonzero(beta)[0]
        if active.size == 0:
            continue
        q = uniform_weights(n + 1 - lo)
        qb = q[active] * beta[active]
        theta += w_l * (qb @ R[lo + active])
        if w_g == 0.0:
            # pure linear: coefficients only feed theta (apsm.py:339-340)
            coeff[lo + active] += qb
            continue
        for s, j in enumerate(active):
            i = lo + int(j)
            if first[i] < 0:
                if max_atoms is not None and len(slots) >= max_atoms:
                    cap_err = True
                first[i] = n
                slots.append(i)
            coeff[i] += qb[s]
    slot_idx = np.asarray(slots, dtype=np.int64)
    return dict(theta=theta, coeff=coeff, first_step=first, slot_index=slot_idx,
                atoms=R[slot_idx] if slot_idx.size else np.empty((0, D)),
                coeffs=coeff[slot_idx] if slot_idx.size else np.empty(0),
                n_atoms=int(slot_idx.size), capacity_error=cap_err)


# ---------------------------------------------------------------------------
# evaluation / detection (kernels.py:187-206, engine.py:206-261)
# ---------------------------------------------------------------------------

def evaluate_batch(theta, atoms, coeffs, U, w_g=0.5, sigma_sq=0.05):
    """theta.u + w_g sum_i coeffs_i exp(-||a_i - u||^2 / 2 sigma^2), explicit
    differences as in kernels.py:187-206 (the engine's baseline stage,
    engine.py:116-123)."""
    U = np.atleast_2d(np.asarray(U, dtype=np.float64))
    y = U @ np.asarray(theta, dtype=np.float64)
    atoms = np.asarray(atoms, dtype=np.float64)
    if w_g != 0.0 and atoms.shape[0]:
        inv2s = 1.0 / (2.0 * sigma_sq)
        for c0 in range(0, U.shape[0], 256):
            u = U[c0:c0 + 256]
            d2 = ((atoms[None, :, :] - u[:, None, :]) ** 2).sum(-1)
            y[c0:c0 + 256] += w_g * (np.exp(-d2 * inv2s) @ coeffs)
    return y


def detect_batch(theta, atoms, coeffs, rx, w_g=0.5, sigma_sq=0.05):
    """g(r) = f(r1) + i f(r2) (engine.py:246-261, apsm.py:399-406)."""
    y = evaluate_batch(theta, atoms, coeffs, realify(rx), w_g, sigma_sq)
    return y[0::2] + 1j * y[1::2]


def run_frame(frame, n_train, scheme, users=None, W=20, eps=0.01, w_l=0.5, w_g=0.5,
              sigma_sq=0.05):
    """Train every requested user on the frame's pilots, detect the payload,
    demap and count errors (run_trial for each target user, noma.py:249-281).
    Returns per-user dicts with est, rx_idx, bit_err, sym_err, ber, trained model."""
    rx = frame["rx"]
    sym = frame["symbols"]
    bits = frame["bits"]
    k = frame["bps"]
    K = sym.shape[0]
    users = range(K) if users is None else users
    R = realify(rx[:n_train])
    out = []
    for u in users:
        m = train_user(R, realify_targets(sym[u, :n_train]), W, eps, w_l, w_g, sigma_sq)
        est = detect_batch(m["theta"], m["atoms"], m["coeffs"], rx[n_train:], w_g, sigma_sq)
        rx_bits = demodulate_hard(est, scheme)
        tx_bits = bits[u, n_train * k:]
        idx = demap_indices(est, scheme)
        tx_idx = tx_bits.reshape(-1, k) @ (1 << np.arange(k - 1, -1, -1))
        out.append(dict(user=u, model=m, est=est, rx_idx=idx,
                        bit_err=int(np.sum(tx_bits != rx_bits)),
                        sym_err=int(np.sum(idx != tx_idx)),
                        ber=ber(tx_bits, rx_bits)))
    return out
