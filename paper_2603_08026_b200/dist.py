"""Batch-parallel multi-GPU plumbing: one process per GPU, every rank owns a
contiguous shard of the sequences and runs the whole DyLLM step on its own GPU with no per-step
collective. Only the bench timing (max over ranks) and the final token gather cross ranks.
torch.distributed (NCCL on GPUs, gloo in the CPU tests) is the transport."""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(global_batch: int, world: int, rank: int):
    """Sequences [lo, hi) owned by `rank`; shards differ in size by at most one sequence."""
    base, extra = divmod(global_batch, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def max_over_ranks(values, device=None):
    """Element-wise max of a list of floats over all ranks (device time of the slowest rank)."""
    t = torch.tensor(values, dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def gather_tokens(tokens: torch.Tensor, global_batch: int):
    """All-gather every rank's generated tokens [b_r][N] into [global_batch][N] (rank order)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return tokens
    world = dist.get_world_size()
    sizes = [shard_range(global_batch, world, r) for r in range(world)]
    bmax = max(hi - lo for lo, hi in sizes)
    pad = torch.zeros((bmax, tokens.shape[1]), dtype=tokens.dtype, device=tokens.device)
    pad[: tokens.shape[0]] = tokens
    out = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(out, pad)
    return torch.cat([o[: hi - lo] for o, (lo, hi) in zip(out, sizes)], dim=0)
