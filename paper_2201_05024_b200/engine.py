"""Batch evaluation engine (mirror of kapsm/engine.py) on the B200.

``EngineConfig`` keeps the reference's fields and validation (engine.py:49-75)
so callers are unchanged.  There is exactly one execution path: the CUDA
kernels.  ``stage``, ``tile_atoms``, ``tile_inputs``, ``chunk_dim``,
``workers`` and ``deterministic_reduction`` select CPU cache-blocking
strategies in the reference; on the GPU they are accepted and ignored (every
call is deterministic: fixed reduction order, no float atomics).
``precision`` selects the float32 (performance) or float64 kernels; results
are returned as float64 / complex128 like the reference (engine.py:243).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dv
from . import _lib
from .kernels import FilterState, KernelParams

__all__ = ["EngineConfig", "STAGES", "batch_evaluate", "batch_detect"]

STAGES = ("baseline", "grouped", "tiled", "balanced")


@dataclass(frozen=True)
class EngineConfig:
    """engine.py:49-75 (fields, defaults and validation unchanged)."""

    stage: str = "balanced"
    tile_atoms: int = 256
    tile_inputs: int = 8
    chunk_dim: int = 16
    workers: int = 1
    deterministic_reduction: bool = True
    precision: str = "f64"

    def __post_init__(self):
        if self.stage not in STAGES:
            raise ValueError(f"unknown stage {self.stage!r}; expected one of {STAGES}")
        for name in ("tile_atoms", "tile_inputs", "chunk_dim", "workers"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be >= 1, got {getattr(self, name)}")
        if self.precision not in ("f64", "f32"):
            raise ValueError(f"precision must be 'f64' or 'f32', got {self.precision!r}")


def _filter_to_dev(f: FilterState, prec: str):
    theta = dv.to_dev(f.theta, prec)
    if f.n_atoms:
        atoms = dv.to_dev(f.atoms, prec)
        coeffs = dv.to_dev(f.coeffs, prec)
    else:
        atoms = coeffs = None
    return theta, atoms, coeffs


def _evaluate_rows(f: FilterState, u: np.ndarray, p: KernelParams, prec: str) -> np.ndarray:
    """GPU evaluation of f on realified rows u (n x dim) -> float64[n]."""
    n = u.shape[0]
    theta, atoms, coeffs = _filter_to_dev(f, prec)
    ud = dv.to_dev(u, prec)
    out = dv.empty((n,), prec)
    n_atoms = f.n_atoms if p.w_g != 0.0 else 0
    _lib.check(dv.fn("kapsm_batch_evaluate", prec)(
        dv.ptr(theta), dv.ptr(atoms), dv.ptr(coeffs), n_atoms, f.dim, dv.ptr(ud), n,
        _lib.params(p), dv.ptr(out), dv.stream()), "batch_evaluate")
    return out.to("cpu").numpy().astype(np.float64, copy=False)


def batch_evaluate(f: FilterState, inputs, p: KernelParams, cfg: EngineConfig) -> np.ndarray:
    """Evaluate f on every input row (engine.py:206-243); float64 result."""
    if len(inputs) == 0:
        return np.empty(0)
    u = np.atleast_2d(np.asarray(inputs, dtype=np.float64))
    if u.ndim != 2 or u.shape[1] != f.dim:
        raise ValueError(f"inputs have shape {u.shape}, filter dimension is {f.dim}")
    return _evaluate_rows(f, u, p, cfg.precision)


def detect_complex(f: FilterState, rx: np.ndarray, p: KernelParams, prec: str) -> np.ndarray:
    """GPU g(r) = f(r1) + i f(r2) for complex rows rx (T x M) -> complex128[T]."""
    t = rx.shape[0]
    theta, atoms, coeffs = _filter_to_dev(f, prec)
    rd = dv.complex_to_dev(rx, prec)
    out = dv.empty((t, 2), prec)
    n_atoms = f.n_atoms if p.w_g != 0.0 else 0
    _lib.check(dv.fn("kapsm_batch_detect", prec)(
        dv.ptr(theta), dv.ptr(atoms), dv.ptr(coeffs), n_atoms, f.dim, dv.ptr(rd), t,
        _lib.params(p), dv.ptr(out), dv.stream()), "batch_detect")
    o = out.to("cpu").numpy().astype(np.float64)
    return o[:, 0] + 1j * o[:, 1]


def batch_detect(f: FilterState, inputs, p: KernelParams, cfg: EngineConfig) -> np.ndarray:
    """Complex detection g(r) = f(r1) + i f(r2) (engine.py:246-261)."""
    if len(inputs) == 0:
        return np.empty(0, dtype=np.complex128)
    rx = np.atleast_2d(np.asarray(inputs, dtype=np.complex128))
    if 2 * rx.shape[1] != f.dim:
        raise ValueError(
            f"received vectors of length {rx.shape[1]} do not match filter dim {f.dim}")
    return detect_complex(f, rx, p, cfg.precision)
