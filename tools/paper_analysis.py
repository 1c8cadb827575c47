"""Paper-analysis instrumentation on the GPU path, at random init:

  - per-layer histograms of the temporal cosine similarity s (Fig. 2), from the
    per-layer similarity trace of one response-only and one full-input denoising step;
  - salient counts per layer over the generation prefix (Fig. 6);
  - the approximation error of Alg. 4 against exact attention (Fig. 4): after a traced
    step, every input row's context C in the cache (exact for idx_in, C_cache + dC otherwise) is
    compared with softmax(Q K^T / sqrt(d_h)) V over the same step's Q / K / V caches (torch fp32
    SDPA, analysis only), i.e. the size of the term Eq. 3 drops (dS.V).

    python tools/paper_analysis.py [--config llada8b] [--frac 0.1] [--steps 12] [--out f4.json]

Everything the figures need comes from the library's own trace hooks (dyllm_cache_set_trace,
sal_counts) and read-only cache exports; torch is used only for the reference attention and the
histograms.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from dataclasses import replace

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_08026_b200 import dyllm as dy  # noqa: E402
from synth import configs, gen  # noqa: E402

BINS = np.concatenate([[-1.0, 0.0, 0.5, 0.8, 0.9], np.linspace(0.95, 1.0, 11)])


def exact_contexts(cache, cfg, run, layer, row_lo):
    """softmax(Q K^T / sqrt(d_h)) V of the input rows from the layer's current caches (fp32)."""
    b, N = run.batch, run.L_P + run.L_R
    H, KVH, hd = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    Q = cache.export(layer, dy.Q).float().view(b, N, H, hd).transpose(1, 2)[:, :, row_lo:]
    K = cache.export(layer, dy.K).float().view(b, N, KVH, hd).transpose(1, 2)
    V = cache.export(layer, dy.V).float().view(b, N, KVH, hd).transpose(1, 2)
    if KVH != H:
        K = K.repeat_interleave(H // KVH, dim=1)
        V = V.repeat_interleave(H // KVH, dim=1)
    C = torch.nn.functional.scaled_dot_product_attention(Q, K, V)
    return C.transpose(1, 2).reshape(b, N - row_lo, H * hd)


def approx_error(cache, cfg, run, layer, row_lo, lists, offs):
    """Per-row relative error of the cached contexts vs exact attention, split by row kind."""
    b, N = run.batch, run.L_P + run.L_R
    Cx = exact_contexts(cache, cfg, run, layer, row_lo)
    Cg = cache.export(layer, dy.CTX).float()[:, row_lo:]
    err = ((Cg - Cx).abs().amax(-1) / Cx.abs().amax(-1).clamp_min(1e-30)).cpu().numpy()   # [b][L]
    exact = np.zeros((b, N - row_lo), bool)
    for s in range(b):
        rows = lists[offs[s]:offs[s + 1]] - s * N - row_lo
        exact[s, rows[rows >= 0]] = True
    def stats(x):
        return {"n": int(x.size), "median": float(np.median(x)) if x.size else None,
                "p90": float(np.quantile(x, 0.9)) if x.size else None, "max": float(x.max()) if x.size else None}
    return {"exact_rows": stats(err[exact]), "approximate_rows": stats(err[~exact])}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llada8b")
    ap.add_argument("--layers", type=int, default=0, help="override n_layers (0 = config)")
    ap.add_argument("--frac", type=float, default=0.10)
    ap.add_argument("--steps", type=int, default=12, help="denoising steps after the FullSteps")
    ap.add_argument("--out", default="gpurun_out/paper_analysis.json")
    a = ap.parse_args()
    cfg, run = configs.preset(a.config)
    if a.layers:
        cfg = replace(cfg, n_layers=a.layers)
    run = replace(run, select_mode=1)
    ctx = dy.Context(0)
    w = dy.Weights.random(ctx, cfg, seed=0)
    eng = dy.Engine(ctx, w, run)
    prompts = torch.tensor(gen.prompt_tokens(0, run.batch, run.L_P, cfg.mask_id), dtype=torch.int32)
    eng.load_prompts(prompts.cuda())
    b, N, nl = run.batch, run.N, cfg.n_layers
    tr_lists = torch.zeros(nl * b * N, dtype=torch.int32, device="cuda")
    tr_offs = torch.zeros(nl * (b + 1), dtype=torch.int32, device="cuda")
    tr_sims = torch.zeros(nl * b * N, dtype=torch.float32, device="cuda")
    taus = np.full(nl, a.frac, np.float32)
    out = {"config": a.config, "n_layers": nl, "batch": b, "frac": a.frac, "bins": BINS.tolist(), "steps": {}}
    T = run.T_full + a.steps
    want = {}
    for t in range(run.T_full, T):
        kind = "fi" if t % run.full_period == 0 else "ro"
        if kind not in want.values() and t >= run.T_full + 4:
            want[t] = kind
    for t in range(T):
        traced = t in want
        eng.cache.set_trace(tr_lists, tr_offs, tr_sims) if traced else eng.cache.set_trace()
        eng.cache.denoise_step(t, taus, eng.tokens, eng.dec_pos, eng.dec_tok, eng.sal_counts[t])
        if not traced:
            continue
        torch.cuda.synchronize()
        row_lo = 0 if want[t] == "fi" else run.L_P
        lists = tr_lists.view(nl, b * N).cpu().numpy()
        offs = tr_offs.view(nl, b + 1).cpu().numpy()
        sims = tr_sims.view(nl, b, N).cpu().numpy()[:, :, row_lo:]
        rec = {"kind": want[t], "layers": []}
        for l in range(nl):
            # layer l's input list = layer l-1's output (D4); layer 0's is the carried set (not traced)
            src_l, src_o = (lists[l - 1], offs[l - 1]) if l else (None, None)
            entry = {"layer": l, "s_hist": np.histogram(sims[l].ravel(), BINS)[0].tolist(),
                     "salient": int(offs[l][-1])}
            if l:
                entry["approx_error"] = approx_error(eng.cache, cfg, run, l, row_lo, src_l, src_o)
            rec["layers"].append(entry)
        out["steps"][str(t)] = rec
    torch.cuda.synchronize()
    sal = eng.sal_counts[run.T_full:T].cpu().numpy().astype(np.float64)  # [steps][layers][b]
    rows_in = np.array([N if t % run.full_period == 0 else run.L_R for t in range(run.T_full, T)], np.float64)
    out["salient_fraction_per_layer"] = (sal.sum(axis=2) / (b * rows_in[:, None])).mean(axis=0).tolist()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f)
    for t, rec in out["steps"].items():
        print(f"step {t} ({rec['kind']}):")
        for e in rec["layers"][:4] + rec["layers"][-2:]:
            ae = e.get("approx_error", {})
            print(f"  layer {e['layer']:2d} salient {e['salient']:5d}  s-hist {e['s_hist']}  "
                  f"approx err (median/p90/max) {ae.get('approximate_rows', {})}  exact rows {ae.get('exact_rows', {})}")


if __name__ == "__main__":
    main()
