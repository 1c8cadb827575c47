"""Per-role mbarrier wait cycles of the fused attention kernel (debug hook, which = 1) for the last
layer of one denoising step of the bench workload.

    python tools/attn_trace.py --mode ro|fi|full
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
ap.add_argument("--frac", type=float, default=0.10)
a = ap.parse_args()
cfg, run = configs.preset("llada8b")
run = replace(run, select_mode=1)
ctx = dy.Context(0)
w = dy.Weights.random(ctx, cfg, seed=0)
eng = dy.Engine(ctx, w, run)
eng.tokens[:, : run.L_P].copy_(torch.tensor(gen.prompt_tokens(0, run.batch, run.L_P, cfg.mask_id), dtype=torch.int32))
eng.tokens[:, run.L_P:].fill_(cfg.mask_id)
taus = np.full(cfg.n_layers, a.frac, np.float32)
if a.mode == "full":
    target = 0
else:
    t0 = run.T_full + 8
    target = next(s for s in range(t0, run.T_total) if (s % run.full_period == 0) == (a.mode == "fi"))
for t in range(target):
    eng.cache.denoise_step(t, taus, eng.tokens, eng.dec_pos, eng.dec_tok)
tr = torch.zeros(148 * 32, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()
dy.lib().dyllm_debug_trace_buffer(1, tr.data_ptr())
eng.cache.denoise_step(target, taus, eng.tokens, eng.dec_pos, eng.dec_tok)
torch.cuda.synchronize()
dy.lib().dyllm_debug_trace_buffer(1, None)
t = tr.view(148, 32).cpu().numpy().astype(np.float64) / 1.9e3  # cycles -> us at ~1.9 GHz
names = ["prod k_empty", "prod q_empty", "vprod v_empty", "mma q_full", "mma s_empty", "mma k_full", "mma p_full",
         "mma v_full", "mma acc_empty", "smx s_full(S)", "smx s_full(P)", "smx p_empty", "smx acc_full", "total",
         "smx passS (incl wait)", "smx passP (incl wait)", "smx epilogue", "smx next_item", "mma next_item",
         "mma QK issue", "mma total", "mma PV issue", "smx passS tmem ld", "mma QK fence"]
print(f"mode {a.mode} step {target}: per-CTA wait time (us, median / max over CTAs)")
for i, n in enumerate(names):
    print(f"  {n:15s} {np.median(t[:, i]):8.1f} {t[:, i].max():8.1f}")
