"""Parallel live frame generation into pinned host memory.

The frames are the reference's seeded synthetic frames -- the generator is
the reference's host code (noma.py:195-246) called in run_trial's RNG order
(noma.py:265-269) with the acceptance-suite seeding (seeded_frame) -- so their
numpy PCG64 streams cannot be ported to the GPU without losing bit-identical
inputs.  Instead a pool of worker processes generates frames in parallel and
writes them, already in the device layout, straight into a shared-memory
ring that is registered with CUDA as pinned memory:

* rx      float32 (slots, F, T, M, 2)   interleaved (re, im), pilots first
* pilots  float32 (slots, F, K, n_train, 2)
* tx      uint8   (slots, F, K, n_data)  Gray labels of the payload symbols
* plab    uint8   (slots, F, K, n_train) labels of the pilot symbols

so a slot feeds ``FrameStream.submit`` (H2D by DMA) with no further copy.
``fill(slot, seeds)`` starts a slot asynchronously and returns a handle whose
``wait()`` blocks until the slot is complete; the host can overlap the next
slot's generation with the GPU work on the current one.
"""

from __future__ import annotations

import multiprocessing as mp
import os
from multiprocessing import shared_memory
from typing import Sequence

import numpy as np

__all__ = ["FrameGenerator"]


def _layout(slots, F, K, M, n_train, n_data):
    T = n_train + n_data
    parts = [("rx", (slots, F, T, M, 2), np.float32), ("pilots", (slots, F, K, n_train, 2), np.float32),
             ("tx", (slots, F, K, n_data), np.uint8), ("plab", (slots, F, K, n_train), np.uint8)]
    off, out = 0, {}
    for name, shape, dt in parts:
        nbytes = int(np.prod(shape)) * np.dtype(dt).itemsize
        out[name] = (off, shape, dt)
        off = (off + nbytes + 4095) // 4096 * 4096
    return out, off


def _views(buf, layout):
    return {k: np.ndarray(shape, dtype=dt, buffer=buf, offset=off)
            for k, (off, shape, dt) in layout.items()}


_W = {}


def _worker_init(name, slots, F, K, M, n_train, n_data, scheme, snr_db):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    shm = shared_memory.SharedMemory(name=name)
    layout, _ = _layout(slots, F, K, M, n_train, n_data)
    _W.update(shm=shm, views=_views(shm.buf, layout), K=K, M=M, n_train=n_train,
              n_data=n_data, scheme=scheme, snr_db=snr_db)


def _worker_frames(args):
    """Generate frames (slot, index, seed) into the shared ring."""
    from .noma import seeded_frame, symbol_labels
    w = _W
    v = w["views"]
    nt, nd = w["n_train"], w["n_data"]
    for slot, i, seed in args:
        fr = seeded_frame(int(seed), w["K"], w["M"], nt, nd, w["scheme"], w["snr_db"])
        k = fr["bps"]
        rx = fr["rx"]
        v["rx"][slot, i, ..., 0] = rx.real
        v["rx"][slot, i, ..., 1] = rx.imag
        pil = fr["symbols"][:, :nt]
        v["pilots"][slot, i, ..., 0] = pil.real
        v["pilots"][slot, i, ..., 1] = pil.imag
        v["tx"][slot, i] = symbol_labels(fr["bits"][:, nt * k:], k)
        v["plab"][slot, i] = symbol_labels(fr["bits"][:, :nt * k], k)
    return len(args)


class _Pending:
    def __init__(self, results):
        self._r = results

    def wait(self):
        for r in self._r:
            r.get()


class FrameGenerator:
    """A pool of ``workers`` processes filling ``slots`` batches of ``F`` frames
    in pinned shared memory (see the module docstring).  ``pin=True`` registers
    the ring with CUDA (needs a device); the tensors ``rx``/``pilots``/``tx``
    are torch views of it, indexed [slot]."""

    def __init__(self, F: int, K: int, M: int, n_train: int, n_data: int, scheme: str = "QPSK",
                 snr_db: float = 20.0, slots: int = 2, workers: int = 0, pin: bool = True):
        import torch
        self.F, self.slots = F, slots
        self.layout, nbytes = _layout(slots, F, K, M, n_train, n_data)
        self.shm = shared_memory.SharedMemory(create=True, size=nbytes)
        self.views = _views(self.shm.buf, self.layout)
        self.workers = workers if workers > 0 else max(1, (os.cpu_count() or 2) - 1)
        ctx = mp.get_context("spawn")          # the parent may hold a CUDA context
        self.pool = ctx.Pool(self.workers, initializer=_worker_init,
                             initargs=(self.shm.name, slots, F, K, M, n_train, n_data, scheme,
                                       snr_db))
        self.pinned = False
        if pin:
            ptr = np.frombuffer(self.shm.buf, dtype=np.uint8).ctypes.data
            err = torch.cuda.cudart().cudaHostRegister(ptr, nbytes, 0)
            if int(err) != 0:
                raise RuntimeError(f"cudaHostRegister failed ({err})")
            self._ptr = ptr
            self.pinned = True
        self.rx = torch.from_numpy(self.views["rx"])
        self.pilots = torch.from_numpy(self.views["pilots"])
        self.tx = torch.from_numpy(self.views["tx"])
        self.plab = torch.from_numpy(self.views["plab"])      # pilot labels (uint8)

    def fill(self, slot: int, seeds: Sequence[int]) -> _Pending:
        """Start generating ``len(seeds) == F`` frames into ``slot``."""
        if len(seeds) != self.F:
            raise ValueError(f"need {self.F} seeds, got {len(seeds)}")
        if not 0 <= slot < self.slots:
            raise ValueError(f"slot {slot} out of range")
        jobs = [(slot, i, s) for i, s in enumerate(seeds)]
        chunk = max(1, len(jobs) // (2 * self.workers))
        parts = [jobs[i:i + chunk] for i in range(0, len(jobs), chunk)]
        return _Pending([self.pool.apply_async(_worker_frames, (p,)) for p in parts])

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()
            self.pool = None
        if self.pinned:
            import torch
            torch.cuda.cudart().cudaHostUnregister(self._ptr)
            self.pinned = False
        self.rx = self.pilots = self.tx = self.plab = None
        self.views = None
        try:
            self.shm.close()
        except BufferError:          # a caller still holds a view of the ring
            pass
        self.shm.unlink()

    def __del__(self):
        try:
            if self.pool is not None:
                self.close()
        except Exception:
            pass
