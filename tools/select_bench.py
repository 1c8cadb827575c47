"""Selection kernel at the bench shapes: fixed-tau mode through dyllm_select_salient vs the
fraction mode inside real denoising steps (per-launch CUDA events, ctx.profile).

    python tools/select_bench.py
"""
import os
import sys
from dataclasses import replace

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_08026_b200 import dyllm as dy  # noqa: E402
from synth import configs, gen  # noqa: E402

cfg, run = configs.preset("llada8b")
ctx = dy.Context(0)
b, N, qw = run.batch, run.N, cfg.q_width
cn = (torch.randn(b, N, qw, device="cuda") * 0.1).bfloat16()
cc = (torch.randn(b, N, qw, device="cuda") * 0.1).bfloat16()
cc0 = cc.clone()
idx = torch.zeros(b * N, dtype=torch.int32, device="cuda")
off = torch.zeros(b + 1, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for row_lo, name in [(run.L_P, "ro"), (0, "fi")]:
    ts = []
    for rep in range(12):
        cc.copy_(cc0)
        flush.fill_(rep)   # evict L2 (C rows come from HBM as in the step)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(ctx.stream)
        ctx.select_salient(cn, cc, row_lo, 0.5, 0, idx, off)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    L = N - row_lo
    byts = b * L * qw * 2 * 3
    t = np.median(ts[2:])
    print(f"tau mode {name}: {t:.1f} us  ({byts / t / 1e3:.0f} GB/s of {byts / 1e6:.0f} MB)")
# fraction mode inside real steps
run = replace(run, select_mode=1)
w = dy.Weights.random(ctx, cfg, seed=0)
eng = dy.Engine(ctx, w, run)
eng.tokens[:, : run.L_P].copy_(torch.tensor(gen.prompt_tokens(0, run.batch, run.L_P, cfg.mask_id), dtype=torch.int32))
eng.tokens[:, run.L_P:].fill_(cfg.mask_id)
taus = np.full(cfg.n_layers, 0.1, np.float32)
for t in range(10):
    if t in (8, 9):
        torch.cuda.synchronize()
        ctx.profile(True)
    eng.cache.denoise_step(t, taus, eng.tokens, eng.dec_pos, eng.dec_tok)
    if t in (8, 9):
        torch.cuda.synchronize()
        sel = ctx.profile_read(3)
        ctx.profile(False)
        print(f"fraction mode in step {t} ({'fi' if t % 4 == 0 else 'ro'}): select median {np.median(sel) * 1e3:.1f} us over {len(sel)} layers")
