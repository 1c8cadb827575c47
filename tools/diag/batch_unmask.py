"""Diagnostic: does every denoising step unmask n_u tokens per sequence at larger batches?"""
import os
import sys
from dataclasses import replace

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2603_08026_b200 import dyllm as dy  # noqa: E402
from synth import configs, gen  # noqa: E402

import sys as _s
LAYERS = int(_s.argv[1]) if len(_s.argv) > 1 else 2
BATCHES = [int(x) for x in _s.argv[2].split(',')] if len(_s.argv) > 2 else [16, 48, 64]
for b in BATCHES:
    cfg, run = configs.preset("llada8b")
    cfg = replace(cfg, n_layers=LAYERS)
    run = replace(run, select_mode=1, batch=b)
    ctx = dy.Context(0)
    w = dy.Weights.random(ctx, cfg, seed=0)
    eng = dy.Engine(ctx, w, run)
    eng.load_prompts(torch.tensor(gen.prompt_tokens(0, b, run.L_P, cfg.mask_id), dtype=torch.int32).cuda())
    taus = np.full(cfg.n_layers, 0.1, np.float32)
    prev = (eng.tokens[:, run.L_P:] == cfg.mask_id).sum(1)
    bad = None
    for t in range(run.T_total):
        eng.cache.denoise_step(t, taus, eng.tokens, eng.dec_pos, eng.dec_tok)
        cur = (eng.tokens[:, run.L_P:] == cfg.mask_id).sum(1)
        dec = (prev - cur).cpu().numpy()
        if bad is None and not np.all(dec == run.n_u):
            bad = (t, np.flatnonzero(dec != run.n_u)[:8].tolist(), dec[dec != run.n_u][:8].tolist(),
                   eng.dec_pos.cpu().numpy()[dec != run.n_u][:4].tolist())
        prev = cur
    ctx.sync()
    print(f"batch {b}: masked left {int(prev.sum())}; first bad step {bad}", flush=True)
    eng = None
    w.close()
    ctx.close()
