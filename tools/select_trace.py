"""Phase timeline of the selection kernel (debug hook dyllm_debug_trace_buffer which = 3): per CTA
%globaltimer at start and after its rows; the last CTA's tail. One response-only and one full-input
layer step of the bench workload (fraction mode).

    python tools/select_trace.py
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
cfg = replace(cfg, n_layers=2)
run = replace(run, select_mode=1)
ctx = dy.Context(0)
w = dy.Weights.random(ctx, cfg, seed=0)
eng = dy.Engine(ctx, w, run)
eng.load_prompts(torch.tensor(gen.prompt_tokens(0, run.batch, run.L_P, cfg.mask_id), dtype=torch.int32).cuda())
taus = np.full(cfg.n_layers, 0.1, np.float32)
tr = torch.zeros(1024 * 64 * 4, dtype=torch.int64, device="cuda")
for t in range(14):
    traced = t in (12, 13)
    if traced:
        tr.zero_()
        torch.cuda.synchronize()
        dy.lib().dyllm_debug_trace_buffer(3, tr.data_ptr())
    eng.cache.denoise_step(t, taus, eng.tokens, eng.dec_pos, eng.dec_tok)
    if traced:
        torch.cuda.synchronize()
        dy.lib().dyllm_debug_trace_buffer(3, None)
        L = run.N - (0 if t % run.full_period == 0 else run.L_P)
        n = ((L + 31) // 32) * run.batch
        a = tr.view(-1, 4)[:n].cpu().numpy().astype(np.float64)   # last layer's launch
        t0 = a[:, 0][a[:, 0] > 0].min()
        start, rows = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
        last = a[np.argmax(a[:, 3])][None, :]        # the last CTA of this launch (latest tail end)
        print(f"step {t} ({'fi' if t % 4 == 0 else 'ro'}): {n} CTAs; start med {np.median(start):.2f} max {start.max():.2f} us; "
              f"rows done med {np.median(rows):.2f} max {rows.max():.2f} us; tail {(last[0, 2] - t0) / 1e3:.2f} -> "
              f"{(last[0, 3] - t0) / 1e3:.2f} us")
