"""Multi-process (world_size 2, gloo, CPU) tests of the batch-parallel host logic: sharding,
max-over-ranks timing and the token gather. The per-rank compute is independent (no per-step
collective), so a sequence's result cannot depend on which rank ran it."""
import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_08026_b200 import dist as pd


def test_shard_range_covers_batch_exactly():
    for gb in (1, 7, 16, 128):
        for world in (1, 2, 3, 8):
            rs = [pd.shard_range(gb, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == gb
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [hi - lo for lo, hi in rs]
            assert max(sizes) - min(sizes) <= 1


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gb, N = 5, 4
    lo, hi = pd.shard_range(gb, world, rank)
    toks = torch.arange(lo * N, hi * N, dtype=torch.int32).view(hi - lo, N)
    allt = pd.gather_tokens(toks, gb)
    mx = pd.max_over_ranks([float(rank + 1), 10.0 - rank])
    q.put((rank, allt.tolist(), mx))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_gather_and_max():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, allt, mx in res:
        assert allt == torch.arange(20, dtype=torch.int32).view(5, 4).tolist()
        assert mx == [2.0, 10.0]
