"""Shared helpers for the GPU parity tests: oracle state <-> libdyllm cache marshalling.

Inputs come from synth/ (seeded) and expected values from oracle/ only; the GPU receives the
oracle's bf16-rounded weights and cache state (teacher forcing).
"""
from __future__ import annotations

import copy

import numpy as np
import torch

import oracle as O
from synth import configs, gen


def bf16_round(a: np.ndarray) -> np.ndarray:
    return torch.tensor(np.asarray(a, dtype=np.float64)).to(torch.bfloat16).to(torch.float64).numpy()


def to_dev_bf16(a: np.ndarray) -> torch.Tensor:
    return torch.tensor(np.asarray(a, dtype=np.float32)).to(torch.bfloat16).cuda()


def f32_round(a: np.ndarray) -> np.ndarray:
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def storage_round(dtype: int):
    """The rounding of a value stored in the GPU caches: bf16 (product path) or fp32 (dtype 1)."""
    return f32_round if dtype == 1 else bf16_round


def to_dev(a: np.ndarray, dtype: int = 0) -> torch.Tensor:
    t = torch.tensor(np.asarray(a, dtype=np.float32))
    return (t if dtype == 1 else t.to(torch.bfloat16)).cuda()


def from_dev(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().numpy().astype(np.float64)


def row_rel_err(got: np.ndarray, ref: np.ndarray) -> np.ndarray:
    """Per-row ||got - ref||_inf / ||ref||_inf (the north_star metric)."""
    num = np.max(np.abs(got - ref), axis=-1)
    den = np.maximum(np.max(np.abs(ref), axis=-1), 1e-30)
    return num / den


class Model:
    """Oracle weights + the same weights uploaded to libdyllm."""

    def __init__(self, name: str, seed: int = 0, **over):
        from dataclasses import replace
        from paper_2603_08026_b200 import dyllm
        cfg, run = configs.preset(name)
        if over:
            cfg = replace(cfg, **{k: v for k, v in over.items() if hasattr(cfg, k)})
            run = replace(run, **{k: v for k, v in over.items() if hasattr(run, k) and not hasattr(cfg, k)})
        self.cfg, self.run = cfg, run
        self.W = gen.model_weights(cfg, seed)
        self.ctx = dyllm.Context(0)
        self.w = dyllm.Weights.from_blob(self.ctx, cfg, dyllm.blob_from_weights(cfg, self.W))
        self.dyllm = dyllm

    def new_cache(self, run=None):
        return self.dyllm.Cache(self.ctx, self.w, run or self.run)


def oracle_states(m: Model, prompts, steps: int, tau=0.999):
    """Run the oracle's Alg. 1 for `steps` steps from fresh prompts; return the states."""
    states = [O.init_state(p, m.cfg, m.run) for p in prompts]
    for st in states:
        for t in range(steps):
            O.denoise_step(st, m.W, m.cfg, m.run, t, tau)
    return states


def round_states(states, dtype: int = 0):
    rnd = storage_round(dtype)
    out = []
    for st in states:
        s2 = copy.deepcopy(st)
        for lc in s2.caches:
            lc.K, lc.V, lc.Q, lc.C, lc.H = (rnd(x) for x in (lc.K, lc.V, lc.Q, lc.C, lc.H))
        if s2.H0 is not None:
            s2.H0 = rnd(s2.H0)
        out.append(s2)
    return out


def import_states(m: Model, cache, states):
    """Write the oracle caches (all layers, all sequences) into the GPU cache."""
    dy = m.dyllm
    fields = [(dy.K, "K"), (dy.V, "V"), (dy.Q, "Q"), (dy.CTX, "C"), (dy.H, "H")]
    for l in range(m.cfg.n_layers):
        for which, f in fields:
            t = cache.tensor(l + 1 if which == dy.H else l, which)
            t.copy_(to_dev(np.stack([getattr(st.caches[l], f) for st in states]), m.cfg.dtype))
    cache.tensor(0, dy.H).copy_(to_dev(np.stack([st.H0 for st in states]), m.cfg.dtype))
    torch.cuda.synchronize()
    # mark initialised through the ABI import path
    buf = torch.empty_like(cache.tensor(0, dy.H))
    dy.lib().dyllm_cache_copy(m.ctx.h, cache.h, 0, dy.H, dy._ptr(buf), 1, 1)
    dy.lib().dyllm_cache_copy(m.ctx.h, cache.h, 0, dy.H, dy._ptr(buf), 1, 0)
    torch.cuda.synchronize()


def pack_lists(lists, N):
    """Per-sequence position lists -> (row ids int32 [cap], offsets int32 [b+1]) on the device."""
    rows, off = [], [0]
    for s, l in enumerate(lists):
        rows += [s * N + int(p) for p in l]
        off.append(len(rows))
    cap = max(len(lists) * N, 1)
    r = torch.zeros(cap, dtype=torch.int32)
    r[: len(rows)] = torch.tensor(rows, dtype=torch.int32)
    return r.cuda(), torch.tensor(off, dtype=torch.int32).cuda()


def unpack_lists(rows: torch.Tensor, off: torch.Tensor, N):
    off = off.cpu().numpy()
    rows = rows.cpu().numpy()
    return [rows[off[s]:off[s + 1]] - s * N for s in range(len(off) - 1)]
