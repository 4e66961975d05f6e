"""Device plumbing: torch owns device memory and streams; compute is the C ABI."""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib

DTYPES = {"f32": (torch.float32, np.float32), "f64": (torch.float64, np.float64)}


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2201_05024_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def new_stream() -> torch.cuda.ExternalStream:
    """A distinct CUDA stream created by the C library (torch.cuda.Stream() hands
    out streams from a small round-robin pool, so two of them can alias).  It
    lives as long as the process: torch's pinned-memory allocator may still
    record events on it while tensors are freed at exit."""
    h = C.c_void_p()
    _lib.check(_lib.load().kapsm_stream_create(C.byref(h)), "stream_create")
    return torch.cuda.ExternalStream(h.value, device=device())


def ptr(t) -> C.c_void_p:
    if t is None:
        return C.c_void_p(None)
    return C.c_void_p(t.data_ptr())


def to_dev(a, prec: str):
    """Host array -> contiguous device tensor of the precision's dtype."""
    tdt, ndt = DTYPES[prec]
    a = np.ascontiguousarray(np.asarray(a, dtype=ndt))
    return torch.from_numpy(a).to(device(), non_blocking=False)


def complex_to_dev(z, prec: str):
    """Complex host array (..., M) -> interleaved (re, im) device tensor (..., M, 2)."""
    z = np.asarray(z, dtype=np.complex128)
    ri = np.stack([z.real, z.imag], axis=-1)
    return to_dev(ri, prec)


def fn(name: str, prec: str):
    return getattr(_lib.load(), f"{name}_{prec}")


def zeros(shape, prec: str):
    return torch.zeros(shape, dtype=DTYPES[prec][0], device=device())


def empty(shape, prec: str):
    return torch.empty(shape, dtype=DTYPES[prec][0], device=device())
