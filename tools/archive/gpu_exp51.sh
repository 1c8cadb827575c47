mkdir -p gpurun_out
python -m paper_2603_08026_b200.build > /dev/null 2>&1
timeout 120 python -u - > gpurun_out/exp51.log 2>&1 <<'PY'
import os, sys, numpy as np, torch
from dataclasses import replace
sys.path.insert(0, os.getcwd())
from paper_2603_08026_b200 import dyllm as dy
from synth import configs, gen
cfg, run = configs.preset("llada8b")
run = replace(run, select_mode=1)
ctx = dy.Context(0)
w = dy.Weights.random(ctx, cfg, seed=0)
eng = dy.Engine(ctx, w, run)
eng.tokens[:, : run.L_P].copy_(torch.tensor(gen.prompt_tokens(0, run.batch, run.L_P, cfg.mask_id), dtype=torch.int32))
eng.tokens[:, run.L_P:].fill_(cfg.mask_id)
taus = np.full(cfg.n_layers, 0.1, np.float32)
for t in range(12):
    print("step", t, flush=True)
    eng.cache.denoise_step(t, taus, eng.tokens, eng.dec_pos, eng.dec_tok)
    torch.cuda.synchronize()
    print("done", t, flush=True)
PY
echo "rc=$?" >> gpurun_out/exp51.log
