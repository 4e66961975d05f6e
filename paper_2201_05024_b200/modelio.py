"""File containers of the file-driven path, byte-compatible
with the reference's kapsm/modelio.py:1-24 layouts so files move between the
two implementations:

* IQ capture: 8-byte magic ``APSMIQ\\0\\0``, u32 antennas M, u32 samples T,
  then T x M complex samples as little-endian float32 (I, Q) pairs, antenna
  fastest;
* model: 8-byte magic ``APSMMDL1``, u32 M, u32 atom count A, f64 w_l, w_g,
  sigma^2, then theta (2M f64), atoms (A x 2M f64, row-major), coefficients
  (A f64);
* symbol estimates: headerless float32 (I, Q) pairs.

Readers validate magic, header values, payload length and trailing bytes and
raise :class:`FileFormatError` (a ValueError, as modelio.py:50-51) naming the
byte offset.  Host-side I/O only: the detector work behind ``kapsm_b200``'s
``train``/``detect`` commands runs on the GPU.
"""

from __future__ import annotations

import os
from typing import Tuple

import numpy as np

from .kernels import FilterState, KernelParams

__all__ = ["FileFormatError", "IQ_MAGIC", "MODEL_MAGIC", "save_iq", "load_iq", "save_model",
           "load_model", "save_symbols", "load_symbols"]

IQ_MAGIC = b"APSMIQ\x00\x00"
MODEL_MAGIC = b"APSMMDL1"
_IQ_HEAD = np.dtype([("magic", "S8"), ("m", "<u4"), ("t", "<u4")])
_MODEL_HEAD = np.dtype([("magic", "S8"), ("m", "<u4"), ("a", "<u4"), ("w_l", "<f8"),
                        ("w_g", "<f8"), ("sigma_sq", "<f8")])
_U32 = np.iinfo(np.uint32).max


class FileFormatError(ValueError):
    """A container failed validation (magic, header, truncation, trailing data)."""


class _Reader:
    """Sequential validated reads over one file's bytes."""

    def __init__(self, path, kind: str):
        self.path, self.kind = path, kind
        with open(path, "rb") as fh:
            self.buf = fh.read()
        self.pos = 0

    def fail(self, msg: str):
        raise FileFormatError(f"{self.path}: {msg}")

    def header(self, dtype: np.dtype, magic: bytes):
        """Magic first (offset 0), then the rest of the header as one read at
        offset 8, so a short file names the field that is cut (modelio.py:53-72)."""
        n = len(self.buf)
        if n < len(magic):
            self.fail(f"truncated {self.kind} file: {n} bytes, header needs {len(magic)} "
                      f"at offset 0")
        if self.buf[:len(magic)] != magic:
            self.fail(f"bad {self.kind} magic at offset 0: {self.buf[:len(magic)]!r} != {magic!r}")
        self.pos = len(magic)
        rest = np.dtype([(k, dtype.fields[k][0]) for k in dtype.names if k != "magic"])
        self.array(rest, 1, f"{self.kind} header")
        return np.frombuffer(self.buf, dtype=dtype, count=1, offset=0)[0]

    def array(self, dtype, count: int, what: str):
        dtype = np.dtype(dtype)
        need = dtype.itemsize * int(count)
        if len(self.buf) - self.pos < need:
            self.fail(f"truncated file: {what} needs {need} bytes at offset {self.pos}, "
                      f"file ends at {len(self.buf)}")
        a = np.frombuffer(self.buf, dtype=dtype, count=int(count), offset=self.pos)
        self.pos += need
        return a

    def finish(self):
        extra = len(self.buf) - self.pos
        if extra:
            self.fail(f"{extra} trailing bytes after the payload at offset {self.pos}")


def _iq_pairs(z) -> np.ndarray:
    z = np.asarray(z, dtype=np.complex128)
    return np.stack([z.real, z.imag], axis=-1).astype("<f4")


def save_iq(path, samples) -> None:
    """Complex samples (T, M) -> IQ container."""
    rx = np.atleast_2d(np.asarray(samples, dtype=np.complex128))
    t, m = rx.shape
    if m < 1:
        raise ValueError("an IQ capture needs at least one antenna")
    if max(t, m) > _U32:
        raise ValueError("sample or antenna count does not fit the u32 header")
    head = np.array([(IQ_MAGIC, m, t)], dtype=_IQ_HEAD)
    with open(path, "wb") as fh:
        fh.write(head.tobytes() + _iq_pairs(rx).tobytes())


def load_iq(path) -> np.ndarray:
    """IQ container -> complex128 samples (T, M)."""
    r = _Reader(path, "IQ")
    h = r.header(_IQ_HEAD, IQ_MAGIC)
    m, t = int(h["m"]), int(h["t"])
    if m == 0:
        r.fail("IQ header declares M=0 antennas at offset 8")
    v = r.array("<f4", 2 * m * t, f"the payload of {t} samples x {m} antennas")
    r.finish()
    v = v.reshape(t, m, 2).astype(np.float64)
    return v[..., 0] + 1j * v[..., 1]


def save_model(path, f: FilterState, params: KernelParams) -> None:
    """Filter + kernel parameters -> model container."""
    if f.dim % 2:
        raise ValueError(f"filter dimension {f.dim} is odd: it must be 2M")
    if f.n_atoms > _U32:
        raise ValueError("atom count does not fit the u32 header")
    head = np.array([(MODEL_MAGIC, f.dim // 2, f.n_atoms, params.w_l, params.w_g,
                      params.sigma_sq)], dtype=_MODEL_HEAD)
    body = np.concatenate([np.ravel(f.theta), np.ravel(f.atoms), np.ravel(f.coeffs)])
    with open(path, "wb") as fh:
        fh.write(head.tobytes() + body.astype("<f8").tobytes())


def load_model(path) -> Tuple[FilterState, KernelParams]:
    """Model container -> (FilterState, KernelParams)."""
    r = _Reader(path, "model")
    h = r.header(_MODEL_HEAD, MODEL_MAGIC)
    m, a = int(h["m"]), int(h["a"])
    if m == 0:
        r.fail("model header declares M=0 antennas at offset 8")
    dim = 2 * m
    theta = r.array("<f8", dim, f"theta ({dim} f64)").astype(np.float64)
    atoms = r.array("<f8", a * dim, f"{a} atoms x {dim} f64").astype(np.float64).reshape(a, dim)
    coeffs = r.array("<f8", a, f"{a} coefficients").astype(np.float64)
    r.finish()
    try:
        params = KernelParams(float(h["w_l"]), float(h["w_g"]), float(h["sigma_sq"]))
    except ValueError as exc:
        raise FileFormatError(f"{path}: invalid kernel parameters in the header: {exc}") from exc
    return FilterState(theta, atoms, coeffs), params


def save_symbols(path, estimates) -> None:
    """Complex estimates -> raw float32 (I, Q) stream."""
    with open(path, "wb") as fh:
        fh.write(_iq_pairs(np.atleast_1d(estimates)).tobytes())


def load_symbols(path) -> np.ndarray:
    """Raw float32 (I, Q) stream -> complex128."""
    size = os.path.getsize(path)
    if size % 8:
        raise FileFormatError(f"{path}: symbol stream length {size} is not a multiple of 8 "
                              f"(truncated pair at offset {size - size % 8})")
    v = np.fromfile(path, dtype="<f4").astype(np.float64).reshape(-1, 2)
    return v[:, 0] + 1j * v[:, 1]
