"""Multi-process (world_size 2, gloo, CPU) tests of the frame sharding and the
decision / error-count collectives used by the multi-GPU path."""

import os
import socket

import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

from paper_2201_05024_b200 import dist as D


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    try:
      try:
        info = D.init_from_env(backend="gloo")
        frames = D.shard_frames(list(range(10)), info.rank, info.world)
        K, nd = 3, 5
        labels = torch.full((len(frames), K, nd), rank + 1, dtype=torch.uint8)
        g = D.gather_decisions(labels)
        counts = torch.tensor([[rank, 10 * rank, 1]], dtype=torch.int64)
        D.reduce_counts(counts)
        # batched exchange: 5 frames per rank, batches of 2 -> 2 exchange steps
        ex = D.BatchedExchange(2, (K, nd), "cpu")
        steps = 0
        for fi in range(5):
            lab = torch.full((1, K, nd), 10 * rank + fi, dtype=torch.uint8)
            steps += ex.add(lab, torch.tensor([1, rank], dtype=torch.int64))
        bx = (steps, tuple(ex.gathered.shape), ex.gathered[:, :, 0, 0].tolist(), ex.totals.tolist())
        # the trailing partial batch (frame 4 of each rank) is exchanged by flush()
        fl = ex.flush()
        bx += (fl, tuple(ex.gathered.shape), ex.gathered[:, :, 0, 0].tolist(), ex.totals.tolist(),
               ex.flush(), ex.pending)
        q.put((rank, frames, tuple(g.shape), g[:, 0, 0, 0].tolist(), counts.tolist(), bx))
      except Exception as e:  # report instead of hanging the parent
        q.put((rank, "error", repr(e), None, None, None))
    finally:
        if tdist.is_initialized():
            tdist.destroy_process_group()


def test_shard_frames_partition():
    ids = list(range(13))
    parts = [D.shard_frames(ids, r, 4) for r in range(4)]
    assert sorted(sum(parts, [])) == ids
    assert all(set(a).isdisjoint(b) for i, a in enumerate(parts) for b in parts[i + 1:])
    with pytest.raises(ValueError):
        D.shard_frames(ids, 4, 4)


def test_gather_and_reduce_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, f0, s0, v0, c0, b0), (r1, f1, s1, v1, c1, b1) = res
    assert f0 == [0, 2, 4, 6, 8] and f1 == [1, 3, 5, 7, 9]
    assert tuple(s0) == (2, 5, 3, 5)
    assert v0 == [1, 2] and v1 == [1, 2]
    assert c0 == c1 == [[1, 10, 2]]
    # last exchanged batch = frames 2, 3 of each rank; counters summed over 2 frames x 2 ranks
    assert b0 == b1 == (2, (2, 2, 3, 5), [[2, 3], [12, 13]], [4, 2],
                        True, (2, 1, 3, 5), [[4], [14]], [2, 1], False, 0)
