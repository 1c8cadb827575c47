"""Run the bench workload up to one chosen denoising step and bracket exactly that step with
cudaProfilerStart/Stop, for `ncu --profile-from-start off` captures (B200_PROFILING.md).

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python tools/profile_step.py --mode ro
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from dataclasses import replace  # noqa: E402

from paper_2603_08026_b200 import dyllm as dy  # noqa: E402
from synth import configs, gen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llada8b")
    ap.add_argument("--mode", default="ro", choices=["ro", "fi", "full"])
    ap.add_argument("--frac", type=float, default=0.10)
    ap.add_argument("--warm-steps", type=int, default=8, help="sparse steps before the profiled one")
    a = ap.parse_args()
    cfg, run = configs.preset(a.config)
    run = replace(run, select_mode=1)
    ctx = dy.Context(0)
    w = dy.Weights.random(ctx, cfg, seed=0)
    eng = dy.Engine(ctx, w, run)
    prompts = torch.tensor(gen.prompt_tokens(0, run.batch, run.L_P, cfg.mask_id), dtype=torch.int32).cuda()
    eng.tokens[:, : run.L_P].copy_(prompts)
    eng.tokens[:, run.L_P:].fill_(cfg.mask_id)
    taus = np.full(cfg.n_layers, a.frac, np.float32)
    target = {"full": 0}[a.mode] if a.mode == "full" else None
    t = 0
    if target is None:
        want_fi = a.mode == "fi"
        t0 = run.T_full + a.warm_steps
        target = next(s for s in range(t0, run.T_total) if (s % run.full_period == 0) == want_fi)
    for t in range(target):
        eng.cache.denoise_step(t, taus, eng.tokens, eng.dec_pos, eng.dec_tok)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    eng.cache.denoise_step(target, taus, eng.tokens, eng.dec_pos, eng.dec_tok)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(f"profiled step t={target} mode={a.mode}")


if __name__ == "__main__":
    main()
