"""Multi-GPU frame sharding (one process per GPU, torch.distributed over NCCL).

Frames are independent: every rank runs the whole K1 -> K2 ->
K3 pipeline on its own frames with no exchange during compute.  The only
collective step gathers the hard decisions and reduces the error counters:

* ``all_gather_into_tensor`` of the uint8 decision labels (F_local x K x n_data
  per rank),
* ``all_reduce(SUM)`` of the int64 per-user bit / symbol error counters.

The same functions run on the ``gloo`` backend with CPU tensors (tests).
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Optional, Sequence

import torch
import torch.distributed as tdist

__all__ = ["RankInfo", "init_from_env", "shard_frames", "gather_decisions", "reduce_counts",
           "BatchedExchange"]


@dataclass(frozen=True)
class RankInfo:
    rank: int
    world: int
    local_rank: int

    @property
    def is_root(self) -> bool:
        return self.rank == 0


def init_from_env(backend: Optional[str] = None) -> RankInfo:
    """Initialise the default process group from torchrun's environment
    (RANK, WORLD_SIZE, LOCAL_RANK, MASTER_ADDR/PORT).  Single process when the
    variables are absent."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not tdist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
            tdist.init_process_group(backend, device_id=torch.device("cuda", local))
        else:
            tdist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return RankInfo(rank, world, local)


def shard_frames(frame_ids: Sequence[int], rank: int, world: int) -> list:
    """Round-robin partition of independent frames over ranks (frame f -> rank
    f mod world); disjoint and covering."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    return [f for i, f in enumerate(frame_ids) if i % world == rank]


def gather_decisions(labels: torch.Tensor, group=None) -> torch.Tensor:
    """All ranks' decision tensors stacked along a new leading rank axis."""
    world = tdist.get_world_size(group) if tdist.is_initialized() else 1
    if world == 1:
        return labels.unsqueeze(0).clone()
    x = labels.contiguous()
    out = torch.empty((world * x.shape[0],) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    tdist.all_gather_into_tensor(out, x, group=group)
    return out.view((world,) + tuple(x.shape))


def reduce_counts(counts: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the per-user error counters over ranks (in place, returned)."""
    if tdist.is_initialized() and tdist.get_world_size(group) > 1:
        tdist.all_reduce(counts, op=tdist.ReduceOp.SUM, group=group)
    return counts


class BatchedExchange:
    """One exchange step per batch of frames: each rank stages
    its frames' decisions into a (batch, K, n_data) buffer and accumulates
    their error counters; every ``batch`` frames the buffer is all-gathered
    and the counters all-reduced (two collectives per batch instead of per
    frame).  Every rank must call ``add`` the same number of times.  Runs on
    the caller's current stream (CUDA) or on CPU tensors (gloo)."""

    def __init__(self, batch: int, labels_shape, device, group=None):
        if batch < 1:
            raise ValueError(f"batch must be >= 1, got {batch}")
        self.batch, self.group = batch, group
        self.buf = torch.zeros((batch,) + tuple(labels_shape), dtype=torch.uint8, device=device)
        self.acc = None
        self.n = 0
        self.gathered = None          # last batch: (world, batch, ...) decisions
        self.totals = None            # last batch: summed counters

    def add(self, labels: torch.Tensor, counts: torch.Tensor):
        k = self.n % self.batch
        self.buf[k].copy_(labels.reshape(self.buf.shape[1:]))
        if self.acc is None:
            self.acc = torch.zeros_like(counts)
        self.acc.add_(counts)
        self.n += 1
        if self.n % self.batch == 0:
            self._exchange(self.batch)
            return True
        return False

    @property
    def pending(self) -> int:
        """Frames added since the last exchange."""
        return self.n % self.batch

    def flush(self) -> bool:
        """Exchange a trailing partial batch (every rank must call it after
        the same number of ``add``s).  ``gathered`` then holds only the
        pending frames: shape (world, pending, ...)."""
        k = self.pending
        if k == 0:
            return False
        self._exchange(k)
        self.n += self.batch - k          # the next add starts a fresh batch
        return True

    def _exchange(self, k: int):
        self.gathered = gather_decisions(self.buf[:k].contiguous(), self.group)
        self.totals = reduce_counts(self.acc.clone(), self.group)
        self.acc.zero_()
