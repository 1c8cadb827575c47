"""Multi-GPU plumbing. Batch parallelism: one process per GPU, every rank owns a
contiguous shard of the sequences and runs the whole DyLLM step on its own GPU with no per-step
collective. Only the bench timing (max over ranks) and the final token gather cross ranks.
torch.distributed (NCCL on GPUs, gloo in the CPU tests) is the transport. Tensor parallelism
(include/dyllm.h dyllm_tp_*): shard_weights slices a model's weights into the head / FFN shards."""
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


def shard_weights(cfg, W, world: int, shard: int):
    """Tensor-parallel shard `shard` of `world` (include/dyllm.h): the local model cfg and the
    oracle-layout weights of its heads and FFN channels (embeddings, gains and LM head whole)."""
    from dataclasses import replace
    hd = cfg.head_dim
    Hl, KVl, Fl = cfg.n_heads // world, cfg.n_kv_heads // world, cfg.d_ff // world
    if Hl * world != cfg.n_heads or KVl * world != cfg.n_kv_heads or Fl * world != cfg.d_ff:
        raise ValueError("n_heads, n_kv_heads and d_ff must divide by the TP world size")
    lcfg = replace(cfg, n_heads=Hl, n_kv_heads=KVl, d_ff=Fl)
    q = slice(shard * Hl * hd, (shard + 1) * Hl * hd)
    kv = slice(shard * KVl * hd, (shard + 1) * KVl * hd)
    f = slice(shard * Fl, (shard + 1) * Fl)
    layers = []
    for lw in W["layers"]:
        sl = {"g_attn": lw["g_attn"], "wq": lw["wq"][q], "wk": lw["wk"][kv], "wv": lw["wv"][kv],
              "wo": lw["wo"][:, q], "g_ffn": lw["g_ffn"], "w_gate": lw["w_gate"][f], "w_up": lw["w_up"][f],
              "w_down": lw["w_down"][:, f]}
        if cfg.qkv_bias:
            sl.update(bq=lw["bq"][q], bk=lw["bk"][kv], bv=lw["bv"][kv])
        layers.append(sl)
    return lcfg, {"emb": W["emb"], "g_final": W["g_final"], "lm_head": W["lm_head"], "layers": layers}
