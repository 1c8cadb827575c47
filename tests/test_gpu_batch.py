"""Batch-parallel invariants on one GPU (D16: every sequence is an
independent problem with its own caches and salient sets, so the batch shards across ranks with no
collective). Both checks run whole generations through Engine (dyllm_denoise_step every step) at
the LLaDA-8B layer shape (2 layers, vocab 126464, L_P 700, block 32) in fraction mode f = 0.1.

  - permuting the batch slots permutes the generated tokens and every cache row bit-for-bit
    (what makes the rank-sharded batch of bench.py --gpus N produce the single-GPU result);
  - two runs of the same generation are bit-identical.
"""
from dataclasses import replace

import numpy as np
import pytest
import torch

from synth import configs, gen

pytestmark = pytest.mark.gpu


def _generate(prompts, L_R=32, seed=5):
    from paper_2603_08026_b200 import dyllm as dy
    cfg, run = configs.preset("llada8b")
    cfg = replace(cfg, n_layers=2)
    run = replace(run, batch=len(prompts), L_R=L_R, select_mode=1)
    ctx = dy.Context(0)
    w = dy.Weights.random(ctx, cfg, seed=seed)
    eng = dy.Engine(ctx, w, run)
    out = eng.generate(torch.tensor(prompts, dtype=torch.int32).pin_memory(), np.full(cfg.n_layers, 0.1, np.float32))
    torch.cuda.synchronize()
    caches = {(l, k): eng.cache.export(l, k).cpu() for l in range(cfg.n_layers) for k in (dy.K, dy.V, dy.Q, dy.CTX)}
    caches.update({(l, dy.H): eng.cache.export(l, dy.H).cpu() for l in range(cfg.n_layers + 1)})
    counts = eng.sal_counts.cpu()
    return out.clone(), caches, counts


def test_batch_slot_permutation_invariance():
    cfg, run = configs.preset("llada8b")
    prompts = gen.prompt_tokens(17, 6, run.L_P, cfg.mask_id)
    perm = np.array([3, 0, 5, 1, 4, 2])
    tok_a, cache_a, cnt_a = _generate(prompts)
    tok_b, cache_b, cnt_b = _generate(prompts[perm])
    assert torch.equal(tok_b, tok_a[perm])
    for key, a in cache_a.items():
        assert torch.equal(cache_b[key], a[perm]), key
    assert torch.equal(cnt_b, cnt_a[:, :, perm])
    assert not torch.any(tok_a == cfg.mask_id)


def test_generation_is_bit_deterministic():
    cfg, run = configs.preset("llada8b")
    prompts = gen.prompt_tokens(18, 4, run.L_P, cfg.mask_id)
    tok_a, cache_a, cnt_a = _generate(prompts)
    tok_b, cache_b, cnt_b = _generate(prompts)
    assert torch.equal(tok_a, tok_b)
    assert torch.equal(cnt_a, cnt_b)
    for key, a in cache_a.items():
        assert torch.equal(cache_b[key], a), key
