"""Derivation of the full-size context tolerance C_TOL (tests/test_gpu_fullsize.py; DESIGN.md §4
"tolerances") from the arithmetic, on the CPU: the fp64 oracle's contexts of one LLaDA-8B-shape
sequence are recomputed with the bf16 roundings the GPU path performs at fixed points, and the
row errors that the roundings alone produce are measured.

Rounding points (the GPU path, D12): the RMSNorm output fed to the QKV GEMM; the GEMM's Q / K / V
rows (bf16 output), then Q / K after RoPE; dV = V_new - V_cache; the probabilities P fed to the
P.V tensor-core product (bf16 operands; the normaliser sums the fp32 values); the exact rows' C
and the approximate rows' dC (bf16 stores); C_new = C_cache + dC rounded to bf16.

Inputs: the full-size GPU test's recipe (synth/gen.py IH4 tensors; score std ~2, cached contexts
whose row norms span 2^-4 .. 1), sequence 0, the same idx_in draw. The oracle steps used are
O.qkv / O.attention / O.approx_attention (Alg. 3 lines 4-11, Alg. 4); the FFN is not involved.
"""
import numpy as np
import pytest
import torch

import oracle as O
from synth import configs, gen

SEED = 3
STD = {"cK": 1.25, "cQ": 1.5, "cV": 1.25, "cC": 0.1, "cX": 1.0}
C_TOL = 4e-2     # tests/test_gpu_fullsize.py
TOL = 2e-2       # the north_star's hidden-state bar


def bf(a):
    return torch.tensor(np.asarray(a, dtype=np.float64)).to(torch.bfloat16).to(torch.float64).numpy()


def _inputs(mode, frac_in, s=0):
    cfg, run = configs.preset("llada8b")
    N, d, qw, kw = run.N, cfg.d_model, cfg.q_width, cfg.kv_width
    width = {"cK": kw, "cV": kw, "cQ": qw, "cC": qw, "cX": d}
    host = {k: gen.ih4_normal(SEED, gen.stream_id(0, k) + ((s + 1) << 32), (N, width[k]), sd, np.float32)
            for k, sd in STD.items()}
    kexp = np.random.default_rng(SEED).integers(0, 5, size=(run.batch, N, 1))[s]
    host["cC"] = host["cC"] * np.ldexp(np.float32(1.0), -kexp).astype(np.float32)
    W = {k: gen.ih4_normal(SEED, gen.stream_id(0, k), shape, cfg.qk_std or cfg.w_std if k != "wv" else cfg.w_std)
         for k, shape in (("wq", (qw, d)), ("wk", (kw, d)), ("wv", (kw, d)))}
    W["g_attn"] = np.ones(d)
    row_lo = 0 if mode == "fi" else run.L_P
    rows = np.arange(row_lo, N)
    rng = np.random.default_rng(17 + int(100 * frac_in))
    idx = [np.sort(rng.choice(rows, int(round(frac_in * len(rows))), replace=False)) for _ in range(run.batch)][s]
    return cfg, run, {k: v.astype(np.float64) for k, v in host.items()}, W, rows, idx


def _contexts(cfg, host, W, rows, idx, emulate):
    """New contexts of the input rows (Alg. 3 lines 4-11) in fp64, or with the GPU's roundings."""
    H, KVH, hd = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    r = bf if emulate else (lambda a: a)
    xn = r(O.rms_norm(host["cX"][idx], W["g_attn"], cfg.rms_eps))
    q_raw, k_raw, v = (r(xn @ W[w].T) for w in ("wq", "wk", "wv"))
    q = r(O.rope(q_raw, idx, cfg.rope_theta, hd))
    k = r(O.rope(k_raw, idx, cfg.rope_theta, hd))
    K, V, Q = host["cK"].copy(), host["cV"].copy(), host["cQ"].copy()
    dV = r(v - V[idx])
    K[idx], V[idx], Q[idx] = k, v, q
    A = O.attention_probs(Q[rows], K, H, KVH, hd)                       # [H][L][N], fp64
    grp = H // KVH
    Vh = np.repeat(V.reshape(-1, KVH, hd).transpose(1, 0, 2), grp, axis=0)
    dVh = np.repeat(dV.reshape(-1, KVH, hd).transpose(1, 0, 2), grp, axis=0)
    if emulate:
        # P = 2^(s - m) stored bf16 for the tensor-core product; l sums the unrounded values
        l = 1.0 / A.max(axis=-1, keepdims=True)                          # A = P / l with max P = 1
        P = bf(A * l)
        C_ex = bf((P @ Vh) / l).transpose(1, 0, 2).reshape(len(rows), -1)
        dC = bf((P[:, :, idx] @ dVh) / l).transpose(1, 0, 2).reshape(len(rows), -1)
        C = bf(host["cC"][rows] + dC)
    else:
        C_ex = (A @ Vh).transpose(1, 0, 2).reshape(len(rows), -1)
        C = host["cC"][rows] + (A[:, :, idx] @ dVh).transpose(1, 0, 2).reshape(len(rows), -1)
    pos = np.searchsorted(rows, idx)
    C[pos] = C_ex[pos]
    return C


def test_oracle_steps_reproduce_sparse_layer_contexts():
    """The fp64 reference below is the oracle's own Alg. 3 (sparse_layer) context, at a small size."""
    from dataclasses import replace
    cfg, run = configs.preset("small128")
    cfg = replace(cfg, n_layers=1)
    Wl = gen.layer_weights(cfg, 1, 0)
    rng = np.random.default_rng(0)
    N = run.N
    host = {"cX": rng.standard_normal((N, cfg.d_model)), "cK": rng.standard_normal((N, cfg.kv_width)),
            "cV": rng.standard_normal((N, cfg.kv_width)), "cQ": rng.standard_normal((N, cfg.q_width)),
            "cC": rng.standard_normal((N, cfg.q_width))}
    rows = np.arange(run.L_P, N)
    idx = np.sort(rng.choice(rows, 9, replace=False))
    lc = O.LayerCache(K=host["cK"].copy(), V=host["cV"].copy(), Q=host["cQ"].copy(), C=host["cC"].copy(),
                      H=np.zeros((N, cfg.d_model)))
    ref = O.sparse_layer(host["cX"], lc, Wl, cfg, idx, 0.5, rows, q_mode="cache")
    C = _contexts(cfg, host, Wl, rows, idx, emulate=False)
    assert np.abs(C - ref.C).max() < 1e-12


# (sequence 9 of the response-only case is the maximum over the 16 sequences of the bench batch:
# 3.02%, row 927; full-input sequences reach 2.2-2.8%)
@pytest.mark.parametrize("mode,frac_in,seq", [("fi", 0.06, 0), ("ro", 0.10, 0), ("ro", 0.10, 9)])
def test_bf16_roundings_alone_reach_the_context_tolerance(mode, frac_in, seq):
    cfg, run, host, W, rows, idx = _inputs(mode, frac_in, seq)
    ref = _contexts(cfg, host, W, rows, idx, emulate=False)
    emu = _contexts(cfg, host, W, rows, idx, emulate=True)
    num = np.abs(emu - ref).max(axis=1)
    err = num / np.maximum(np.abs(ref).max(axis=1), 1e-30)
    print(f"{mode} frac_in {frac_in}: max row error {err.max():.4f}, rows over 1e-2: {(err > 1e-2).sum()}/{len(err)}")
    # the roundings alone use most of the 2e-2 hidden-state bar on these contexts (approximate rows
    # whose new context is dominated by dC) and exceed it in some sequences, so the contexts get
    # their own bar with headroom for the kernels' summation orders
    assert err.max() < C_TOL
    assert err.max() > 0.5 * TOL
