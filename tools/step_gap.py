"""Device time of one denoising step vs the sum of its kernels' own durations (CUDA events
around every launch, ctx.profile): the difference is launch / dependency gaps between kernels.

    python tools/step_gap.py [--mode ro|fi]
"""
import argparse
import os
import sys
from dataclasses import replace

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_08026_b200 import dyllm as dy  # noqa: E402
from synth import configs, gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="ro")
ap.add_argument("--opt", default="", help="option=value[,option=value] set before the run (dy.OPT_* numbers)")
a = ap.parse_args()
for kv in filter(None, a.opt.split(",")):
    k, v = kv.split("=")
    dy.set_option(int(k), int(v))
cfg, run = configs.preset("llada8b")
run = replace(run, select_mode=1)
ctx = dy.Context(0)
w = dy.Weights.random(ctx, cfg, seed=0)
eng = dy.Engine(ctx, w, run)
eng.tokens[:, : run.L_P].copy_(torch.tensor(gen.prompt_tokens(0, run.batch, run.L_P, cfg.mask_id), dtype=torch.int32))
eng.tokens[:, run.L_P:].fill_(cfg.mask_id)
taus = np.full(cfg.n_layers, 0.1, np.float32)
want_fi = a.mode == "fi"
t = 0
res = []
while t < run.T_total and len(res) < 6:
    if t >= run.T_full + 4 and (t % run.full_period == 0) == want_fi:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(ctx.stream)
        eng.cache.denoise_step(t, taus, eng.tokens, eng.dec_pos, eng.dec_tok)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1))
    else:
        eng.cache.denoise_step(t, taus, eng.tokens, eng.dec_pos, eng.dec_tok)
    t += 1
# the next step of the same kind, with per-kernel events
while (t % run.full_period == 0) != want_fi:
    eng.cache.denoise_step(t, taus, eng.tokens, eng.dec_pos, eng.dec_tok)
    t += 1
torch.cuda.synchronize()
ctx.profile(True)
eng.cache.denoise_step(t, taus, eng.tokens, eng.dec_pos, eng.dec_tok)
torch.cuda.synchronize()
tot = sum(float(ctx.profile_read(i).sum()) for i in range(32))
ctx.profile(False)
print(f"{a.mode} step device time (no per-kernel events): {np.median(res):.3f} ms (n={len(res)})")
print(f"sum of per-kernel event durations: {tot:.3f} ms  -> gaps {np.median(res) - tot:.3f} ms")
