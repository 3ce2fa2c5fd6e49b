"""CPU, world_size 2 (gloo): prompt sharding and the bench's cross-rank
reduction (max time, summed tokens) -- the multi-GPU host logic."""

from __future__ import annotations

import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2511_16193_b200.dist import reduce_step_stats, shard

    mine = shard(list(range(10)), rank, world)
    t, c = reduce_step_stats([10.0 + rank, 1.0], [100.0 * (rank + 1), len(mine)], dist)
    q.put((rank, mine, t, c))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_and_reduction():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 200
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert out[0][1] == [0, 2, 4, 6, 8] and out[1][1] == [1, 3, 5, 7, 9]
    for _, _, t, c in out:
        assert t == [11.0, 1.0]          # max over ranks
        assert c == [300.0, 10.0]        # sum over ranks


def test_shard_validation():
    from paper_2511_16193_b200.dist import shard

    with pytest.raises(ValueError):
        shard([1, 2], 2, 2)
    assert shard([1, 2, 3], 0, 1) == [1, 2, 3]
