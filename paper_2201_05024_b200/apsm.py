"""APSM learner API (mirror of kapsm/apsm.py) backed by the persistent CUDA trainer.

``train`` / ``ApsmTrainer`` run the whole sequential pilot loop of one user in
one launch of the K2 kernel (``csrc/train.cu``) on the Gram matrix from K1
(``csrc/gram.cu``).  The returned ``FilterState`` reproduces the reference's
representation: theta, then one atom per sample that ever received a nonzero
projection, in first-activation (slot) order (apsm.py:341-359).

Precision: ``train(..., precision="f64")`` (default, like the reference's
64-bit path) or ``"f32"`` (the performance path used by the frame pipeline).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from functools import lru_cache
from typing import Iterable, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _device as dv
from . import _lib
from .kernels import FilterState, KernelParams, zero_filter

__all__ = [
    "TrainingSample", "ApsmConfig", "DegenerateSampleError", "DictionaryCapacityError",
    "window_indices", "uniform_weights", "complex_to_real_pair", "realify_batch", "beta",
    "apsm_step", "ApsmTrainer", "train", "detect_symbol",
]


class DegenerateSampleError(ValueError):
    """kappa(r, r) = 0 (apsm.py:69-70)."""


class DictionaryCapacityError(RuntimeError):
    """An update would push the dictionary past max_atoms (apsm.py:73-74)."""


@dataclass(frozen=True)
class TrainingSample:
    """One realified pair (r, b) (apsm.py:77-91)."""

    r: np.ndarray
    b: float

    def __post_init__(self):
        r = np.asarray(self.r, dtype=np.float64)
        if r.ndim != 1:
            raise ValueError("sample vector must be 1-D")
        if not np.all(np.isfinite(r)) or not np.isfinite(self.b):
            raise ValueError("training sample must be finite")
        object.__setattr__(self, "r", r)
        object.__setattr__(self, "b", float(self.b))


@dataclass(frozen=True)
class ApsmConfig:
    """apsm.py:94-129 (fields, defaults and validation unchanged)."""

    window: int = 20
    epsilon: float = 0.01
    params: KernelParams = field(default_factory=KernelParams)
    weight_scheme: str = "uniform"
    max_atoms: Optional[int] = None

    def __post_init__(self):
        if self.window < 1:
            raise ValueError(f"window must be >= 1, got {self.window}")
        if not self.epsilon > 0:
            raise ValueError(f"epsilon must be > 0, got {self.epsilon}")
        if self.weight_scheme != "uniform":
            raise ValueError(f"unsupported weight_scheme {self.weight_scheme!r}")
        if self.max_atoms is not None and self.max_atoms < 1:
            raise ValueError(f"max_atoms must be >= 1 or None, got {self.max_atoms}")


def window_indices(n: int, window: int) -> range:
    """J_n = {max(0, n-W+1), ..., n} (apsm.py:132-136)."""
    if n < 0:
        raise ValueError(f"sample index must be >= 0, got {n}")
    return range(max(0, n - window + 1), n + 1)


def uniform_weights(count: int) -> np.ndarray:
    """1/count weights summing to exactly 1.0, the defect in the last entry
    (apsm.py:139-153).  Also the source of the trainer's q table."""
    if count < 1:
        raise ValueError("weight count must be >= 1")
    w = np.full(count, 1.0 / count)
    for _ in range(10):
        defect = 1.0 - float(np.sum(w))
        if defect == 0.0:
            break
        w[-1] += defect
    return w


@lru_cache(maxsize=64)
def _qtab_host(window: int) -> np.ndarray:
    q = np.empty(2 * window)
    for j in range(1, window + 1):
        w = uniform_weights(j)
        q[2 * (j - 1)] = w[0]
        q[2 * (j - 1) + 1] = w[-1]
    return q


_QTAB_DEV = {}


def qtab_device(window: int, prec: str):
    key = (window, prec, torch.cuda.current_device())
    t = _QTAB_DEV.get(key)
    if t is None:
        t = dv.to_dev(_qtab_host(window), prec)
        _QTAB_DEV[key] = t
    return t


def complex_to_real_pair(r, b) -> Tuple[TrainingSample, TrainingSample]:
    """([Re r; Im r], Re b), ([Im r; -Re r], Im b) (apsm.py:156-169)."""
    r = np.asarray(r, dtype=np.complex128)
    if r.ndim != 1:
        raise ValueError("received vector must be 1-D")
    b = complex(b)
    r1 = np.concatenate([r.real, r.imag])
    r2 = np.concatenate([r.imag, -r.real])
    return TrainingSample(r1, b.real), TrainingSample(r2, b.imag)


def realify_batch(rx) -> np.ndarray:
    """Rows 2t = [Re; Im], 2t+1 = [Im; -Re] (apsm.py:172-182)."""
    rx = np.atleast_2d(np.asarray(rx, dtype=np.complex128))
    out = np.empty((2 * rx.shape[0], 2 * rx.shape[1]))
    out[0::2] = np.hstack([rx.real, rx.imag])
    out[1::2] = np.hstack([rx.imag, -rx.real])
    return out


def _three_case(res: np.ndarray, eps: float, den: np.ndarray) -> np.ndarray:
    """Three-case projection coefficient (apsm.py:185-191, 329-332)."""
    return np.where(res < -eps, (-res - eps) / den, np.where(res > eps, (-res + eps) / den, 0.0))


def beta(f: FilterState, s: TrainingSample, epsilon: float, params: KernelParams) -> float:
    """Projection coefficient onto C_s (apsm.py:194-209); f(r) evaluated on the GPU."""
    from .engine import _evaluate_rows
    if not epsilon > 0:
        raise ValueError(f"epsilon must be > 0, got {epsilon}")
    denom = float(params.w_l * (s.r @ s.r) + params.w_g)
    if denom <= 0.0:
        raise DegenerateSampleError(
            "kappa(r, r) = 0: zero sample vector with a weightless Gaussian kernel")
    y = float(_evaluate_rows(f, s.r[None, :], params, "f64")[0])
    return float(_three_case(np.array([y - s.b]), epsilon, np.array([denom]))[0])


def apsm_step(f: FilterState, window: Sequence[TrainingSample], cfg: ApsmConfig) -> FilterState:
    """Literal one-step update with per-projection appends (apsm.py:212-238).
    All betas come from one GPU evaluation of the input filter."""
    from .engine import _evaluate_rows
    if not window:
        raise ValueError("window must contain at least one sample")
    p = cfg.params
    rows = np.stack([s.r for s in window])
    targets = np.array([s.b for s in window])
    den = p.w_l * np.einsum("ij,ij->i", rows, rows) + p.w_g
    if np.any(den <= 0.0):
        raise DegenerateSampleError(
            "kappa(r, r) = 0: zero sample vector with a weightless Gaussian kernel")
    y = _evaluate_rows(f, rows, p, "f64")
    betas = _three_case(y - targets, cfg.epsilon, den)
    active = np.nonzero(betas)[0]
    if active.size == 0:
        return f
    if cfg.max_atoms is not None and f.n_atoms + active.size > cfg.max_atoms:
        raise DictionaryCapacityError(
            f"update needs {active.size} new atoms but the dictionary holds "
            f"{f.n_atoms} of max {cfg.max_atoms}")
    q = uniform_weights(len(window))
    qb = q[active] * betas[active]
    theta = f.theta + p.w_l * (qb @ rows[active])
    atoms = np.vstack([f.atoms, rows[active]]) if f.n_atoms else rows[active]
    coeffs = np.concatenate([f.coeffs, qb])
    return FilterState(theta, atoms, coeffs)


# ---------------------------------------------------------------------------
# GPU training driver
# ---------------------------------------------------------------------------

def _ld(n: int) -> int:
    """Gram row stride: 128-byte aligned rows with >= 16 zero columns past the
    last sample (the trainer's TMA copies read whole 16-byte granules and the
    staged column segments run up to 11 columns past the last sample)."""
    return (n + 16 + 31) // 32 * 32


# C-ABI trainer entry: "kapsm_train" picks the latency kernel or the general
# trainer by window / size; tests point it at "kapsm_train_general" to check
# the general trainer on the small golden frames.
_TRAIN_ENTRY = "kapsm_train"


def _train_device(cfg: ApsmConfig, prec: str, *, rx_pilots=None, targets_c=None,
                  samples=None, targets_r=None, f0: Optional[FilterState] = None):
    """Run K1 + K2 for one (frame, user).

    Either complex pilots rx_pilots (T x M) with complex targets (T,), or
    realified samples (N x D) with real targets (N,).  Returns host arrays
    (theta, coeff, first_step, status).
    """
    p = cfg.params
    lib = _lib.load()
    kp = _lib.params(p)
    st = dv.stream()
    if rx_pilots is not None:
        T, M = rx_pilots.shape
        N, D = 2 * T, 2 * M
        rxd = dv.complex_to_dev(rx_pilots, prec)                 # (T, M, 2)
        tgt = dv.complex_to_dev(np.asarray(targets_c), prec)     # (T, 2) == realified targets
    else:
        N, D = samples.shape
        sd = dv.to_dev(samples, prec)
        tgt = dv.to_dev(np.asarray(targets_r, dtype=np.float64), prec)
    if cfg.window > lib.kapsm_max_window() or N > lib.kapsm_max_samples():
        raise NotImplementedError(
            f"window {cfg.window} / {N} realified samples exceed this build's trainer limits "
            f"(window <= {lib.kapsm_max_window()}, samples <= {lib.kapsm_max_samples()})")
    ld = _ld(N)
    gram = dv.zeros((N + 32, ld), prec)        # + the trainer's zero tail rows
    if rx_pilots is not None:
        _lib.check(dv.fn("kapsm_pilot_gram", prec)(dv.ptr(rxd), N * M, 1, T, M, kp, dv.ptr(gram),
                                                   ld, N * ld, st), "pilot_gram")
    else:
        _lib.check(dv.fn("kapsm_sample_gram", prec)(dv.ptr(sd), N * D, 1, N, D, kp, dv.ptr(gram),
                                                    ld, N * ld, st), "sample_gram")
    base0 = theta0 = None
    if f0 is not None and (f0.n_atoms or np.any(f0.theta != 0)):
        from .engine import _evaluate_rows, detect_complex
        if rx_pilots is not None:
            g = detect_complex(f0, rx_pilots, p, prec)
            b0 = np.empty(N)
            b0[0::2] = g.real
            b0[1::2] = g.imag
        else:
            b0 = _evaluate_rows(f0, samples, p, prec)
        base0 = dv.to_dev(b0, prec)
        theta0 = dv.to_dev(f0.theta, prec)
    coeff = dv.empty((N,), prec)
    fs = torch.empty((N,), dtype=torch.int32, device=dv.device())
    theta = dv.empty((D,), prec)
    nact = torch.empty((1,), dtype=torch.int32, device=dv.device())
    status = torch.empty((1,), dtype=torch.int32, device=dv.device())
    q = qtab_device(cfg.window, prec)
    _lib.check(dv.fn(_TRAIN_ENTRY, prec)(
        dv.ptr(gram), ld, N * ld,
        dv.ptr(rxd) if rx_pilots is not None else dv.ptr(None), N * M if rx_pilots is not None else 0,
        dv.ptr(sd) if rx_pilots is None else dv.ptr(None), N * D if rx_pilots is None else 0,
        D, dv.ptr(tgt), 1, 1, N, cfg.window, float(cfg.epsilon), kp, dv.ptr(q), dv.ptr(base0),
        dv.ptr(theta0), dv.ptr(coeff), dv.ptr(fs), dv.ptr(theta), dv.ptr(nact), dv.ptr(status),
        st), "train")
    return (theta.cpu().numpy().astype(np.float64), coeff.cpu().numpy().astype(np.float64),
            fs.cpu().numpy().astype(np.int64), int(status.cpu()[0]))


def _assemble(cfg: ApsmConfig, rows: np.ndarray, theta, coeff, first_step, status,
              f0: Optional[FilterState]) -> FilterState:
    """Device results -> FilterState in the reference's slot order."""
    if status & _lib.TRAIN_DEGENERATE:
        raise DegenerateSampleError(
            "kappa(r, r) = 0: zero sample vector with a weightless Gaussian kernel")
    if status & _lib.TRAIN_STALLED:
        raise RuntimeError("kapsm trainer pipeline watchdog fired")
    p = cfg.params
    base_atoms = f0.atoms if f0 is not None else np.empty((0, rows.shape[1]))
    base_coeffs = f0.coeffs if f0 is not None else np.empty(0)
    if p.w_g == 0.0:
        # pure linear: no dictionary growth (apsm.py:339-340)
        return FilterState(theta, base_atoms.copy(), base_coeffs.copy())
    active = np.nonzero(first_step >= 0)[0]
    if cfg.max_atoms is not None and active.size and base_atoms.shape[0] + active.size > cfg.max_atoms:
        raise DictionaryCapacityError(f"dictionary is at its cap of {cfg.max_atoms} atoms")
    order = active[np.lexsort((active, first_step[active]))]
    atoms = np.vstack([base_atoms, rows[order]]) if base_atoms.shape[0] else rows[order]
    coeffs = np.concatenate([base_coeffs, coeff[order]])
    return FilterState(theta, atoms, coeffs)


class ApsmTrainer:
    """Incremental APSM learner (apsm.py:241-372).

    ``observe`` validates and buffers the realified sample (shape and
    degenerate-sample errors are raised immediately, as in the reference);
    ``state`` runs the persistent GPU trainer over the buffered stream and
    returns the identical FilterState.  With a ``max_atoms`` cap,
    DictionaryCapacityError comes from the observe that crosses the cap, as
    in apsm.py:341-349: every sample owns at most one slot, so while
    ``f0.n_atoms + n_seen <= max_atoms`` no observe can cross it; past that
    point each observe runs the chain over the buffered stream (one launch)
    and raises if the slot count passes the cap.
    """

    def __init__(self, dim: int, cfg: ApsmConfig, f0: Optional[FilterState] = None,
                 precision: str = "f64"):
        if dim < 1:
            raise ValueError(f"dim must be >= 1, got {dim}")
        if f0 is None:
            f0 = zero_filter(dim)
        if f0.dim != dim:
            raise ValueError(f"f0 has dimension {f0.dim}, expected {dim}")
        if precision not in dv.DTYPES:
            raise ValueError(f"precision must be 'f64' or 'f32', got {precision!r}")
        self.cfg = cfg
        self.dim = dim
        self.f0 = f0
        self.precision = precision
        self._rows = []
        self._targets = []
        self._cache = None

    @property
    def n_seen(self) -> int:
        return len(self._rows)

    def observe(self, r, b: float):
        r = np.asarray(r, dtype=np.float64)
        if r.shape != (self.dim,):
            raise ValueError(f"sample has shape {r.shape}, trainer dimension is {self.dim}")
        p = self.cfg.params
        if p.w_l * float(r @ r) + p.w_g <= 0.0:
            raise DegenerateSampleError(
                "kappa(r, r) = 0: zero sample vector with a weightless Gaussian kernel")
        self._rows.append(r.copy())
        self._targets.append(float(b))
        self._cache = None
        cap = self.cfg.max_atoms
        if cap is not None and p.w_g != 0.0 and self.f0.n_atoms + len(self._rows) > cap:
            self.state()            # raises DictionaryCapacityError past the cap

    def observe_symbol(self, r, b):
        s1, s2 = complex_to_real_pair(r, b)
        self.observe(s1.r, s1.b)
        self.observe(s2.r, s2.b)

    def state(self) -> FilterState:
        if self._cache is not None:
            return self._cache
        if not self._rows:
            f = self.f0
            self._cache = FilterState(f.theta.copy(), f.atoms.copy(), f.coeffs.copy())
            return self._cache
        rows = np.stack(self._rows)
        res = _train_device(self.cfg, self.precision, samples=rows,
                            targets_r=np.asarray(self._targets), f0=self.f0)
        self._cache = _assemble(self.cfg, rows, *res, self.f0)
        return self._cache


def train(f0: Optional[FilterState], stream: Iterable[Tuple[np.ndarray, complex]],
          cfg: ApsmConfig, *, precision: str = "f64") -> FilterState:
    """Train over (complex received vector, complex pilot) pairs (apsm.py:375-396):
    2 realified updates per symbol, one persistent GPU launch for the whole loop."""
    rs, bs = [], []
    for r, b in stream:
        rs.append(np.asarray(r, dtype=np.complex128))
        bs.append(complex(b))
    if not rs:
        if f0 is None:
            raise ValueError("empty stream with no initial filter: dimension unknown")
        return f0
    M = rs[0].shape[0]
    if any(r.shape != (M,) for r in rs):
        raise ValueError("received vectors must all be 1-D of the same length")
    if f0 is not None and f0.dim != 2 * M:
        raise ValueError(f"f0 has dimension {f0.dim}, expected {2 * M}")
    rx = np.stack(rs)
    p = cfg.params
    if p.w_g == 0.0 and np.any(np.all(rx == 0, axis=1)):
        raise DegenerateSampleError(
            "kappa(r, r) = 0: zero sample vector with a weightless Gaussian kernel")
    res = _train_device(cfg, precision, rx_pilots=rx, targets_c=np.asarray(bs), f0=f0)
    return _assemble(cfg, realify_batch(rx), *res, f0)


def detect_symbol(f: FilterState, r, params: KernelParams) -> complex:
    """g(r) = f(r1) + i f(r2) (apsm.py:399-406), on the GPU in float64."""
    from .engine import detect_complex
    r = np.asarray(r, dtype=np.complex128)
    if r.ndim != 1 or 2 * r.shape[0] != f.dim:
        raise ValueError(f"received vector of length {r.shape} does not match filter dim {f.dim}")
    return complex(detect_complex(f, r[None, :], params, "f64")[0])
