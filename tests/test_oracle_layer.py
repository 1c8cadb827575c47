"""Pins of the oracle's layer steps and generation loop. CPU only.

- FullStep layer == an independent torch-fp64 transformer block (F.rms_norm, F.linear,
  complex-number RoPE, F.scaled_dot_product_attention, F.silu)
- all-salient SparseStep == full recompute (north_star), within 1e-10
- none-salient SparseStep leaves every cache bit-unchanged
- Q-cache variant == literal all-row Q (D6)
- Alg. 1 schedule pattern, unmask budget, prompt immutability, response-only locality
"""
import json
import os
from dataclasses import replace

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle as O
from synth import configs, gen

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _model(name="tiny", seed=0, **kw):
    cfg, run = configs.preset(name)
    cfg = replace(cfg, **kw) if kw else cfg
    return cfg, run, gen.model_weights(cfg, seed)


def _torch_block(x, w, cfg):
    """Independent torch-fp64 pre-norm block: complex RoPE, SDPA with repeated kv heads."""
    t = lambda a: torch.tensor(a, dtype=torch.float64)
    N, d, H, KVH, hd = x.shape[0], cfg.d_model, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    X = t(x)
    Xn = F.rms_norm(X, (d,), weight=t(w["g_attn"]), eps=cfg.rms_eps)
    q = F.linear(Xn, t(w["wq"]), t(w["bq"]) if cfg.qkv_bias else None)
    k = F.linear(Xn, t(w["wk"]), t(w["bk"]) if cfg.qkv_bias else None)
    v = F.linear(Xn, t(w["wv"]), t(w["bv"]) if cfg.qkv_bias else None)
    freqs = cfg.rope_theta ** (-torch.arange(0, hd, 2, dtype=torch.float64) / hd)
    rot = torch.polar(torch.ones(N, hd // 2, dtype=torch.float64),
                      torch.arange(N, dtype=torch.float64)[:, None] * freqs[None])

    def rope(z, nh):
        z = z.view(N, nh, hd)
        c = torch.complex(z[..., : hd // 2], z[..., hd // 2:]) * rot[:, None, :]
        return torch.cat([c.real, c.imag], -1).reshape(N, nh * hd)

    q, k = rope(q, H), rope(k, KVH)
    qh = q.view(N, H, hd).transpose(0, 1)
    kh = k.view(N, KVH, hd).transpose(0, 1).repeat_interleave(H // KVH, 0)
    vh = v.view(N, KVH, hd).transpose(0, 1).repeat_interleave(H // KVH, 0)
    C = F.scaled_dot_product_attention(qh, kh, vh).transpose(0, 1).reshape(N, H * hd)
    h = X + F.linear(C, t(w["wo"]))
    hn = F.rms_norm(h, (d,), weight=t(w["g_ffn"]), eps=cfg.rms_eps)
    out = h + F.linear(F.silu(F.linear(hn, t(w["w_gate"]))) * F.linear(hn, t(w["w_up"])), t(w["w_down"]))
    return q.numpy(), k.numpy(), v.numpy(), C.numpy(), out.numpy()


@pytest.mark.parametrize("name", ["tiny", "small128", "small128_gqa"])
def test_full_layer_vs_independent_torch(name):
    cfg, run, W = _model(name)
    toks = np.concatenate([gen.prompt_tokens(3, 1, run.L_P, cfg.mask_id)[0],
                           np.full(run.L_R, cfg.mask_id)])
    x = W["emb"][toks]
    lc = O.full_layer(x, W["layers"][0], cfg)
    q, k, v, C, out = _torch_block(x, W["layers"][0], cfg)
    for a, b in [(lc.Q, q), (lc.K, k), (lc.V, v), (lc.C, C), (lc.H, out)]:
        assert np.allclose(a, b, rtol=1e-10, atol=1e-12)


def test_full_step_zero_projections_uniform_attention():
    """zero projections + unit gains -> all scores equal -> attention weights 1/N."""
    cfg, run, W = _model("tiny")
    lw = {k: np.zeros_like(v) for k, v in W["layers"][0].items()}
    lw["g_attn"] = np.ones(cfg.d_model); lw["g_ffn"] = np.ones(cfg.d_model)
    rng = np.random.default_rng(0)
    k = rng.standard_normal((run.N, cfg.kv_width))
    a = O.attention_probs(np.zeros((run.N, cfg.q_width)), k, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim)
    assert np.allclose(a, 1.0 / run.N)
    lc = O.full_layer(rng.standard_normal((run.N, cfg.d_model)), lw, cfg)
    assert np.all(lc.C == 0)


def _warm_state(cfg, run, W, seed=0, decode_steps=2):
    """A sequence after FullSteps that decoded some tokens (caches filled, embeddings changed)."""
    prompt = gen.prompt_tokens(seed, 1, run.L_P, cfg.mask_id)[0]
    st = O.init_state(prompt, cfg, run)
    for t in range(decode_steps):
        O.denoise_step(st, W, cfg, run, t, None, force_full=True)
    return st


@pytest.mark.parametrize("name,mode", [("tiny", 0), ("tiny", 1), ("small128_gqa", 0)])
def test_all_salient_equals_full_recompute(name, mode):
    """S:337 / north_star: tau=+inf with idx_in = all input rows == full recompute (1e-10)."""
    cfg, run, W = _model(name, residual_mode=mode)
    st = _warm_state(cfg, run, W)
    # decode two more tokens WITHOUT refreshing caches: caches are now stale w.r.t. tokens
    st.tokens[run.L_P + 1] = 5; st.tokens[run.L_P + 2] = 6
    ref = O.init_state(st.tokens[: run.L_P], cfg, run)
    ref.tokens = st.tokens.copy()
    HL_ref = O.full_step(ref, W, cfg)
    st.idx_carried = np.arange(run.N)
    HL = O.sparse_step(st, W, cfg, run, O.MODE_FI, tau=2.0)
    assert np.allclose(HL, HL_ref, rtol=1e-10, atol=1e-10)
    for l in range(cfg.n_layers):
        for f in ("K", "V", "Q", "C", "H"):
            assert np.allclose(getattr(st.caches[l], f), getattr(ref.caches[l], f), rtol=1e-10, atol=1e-10)


def test_none_salient_leaves_caches_bit_unchanged():
    """tau = -inf selects nothing; with idx_in = {} everything is frozen; with
    idx_in != {} only K/V/Q/C of idx_in rows move, and every H is bit-unchanged."""
    cfg, run, W = _model("tiny")
    st = _warm_state(cfg, run, W)
    before = [c.copy() for c in st.caches]
    st.idx_carried = np.zeros(0, dtype=np.int64)
    st.decoded_prev = np.zeros(0, dtype=np.int64)
    run0 = replace(run, layer1_policy=0)
    O.sparse_step(st, W, cfg, run0, O.MODE_FI, tau=-2.0)
    for a, b in zip(st.caches, before):
        for f in ("K", "V", "Q", "C", "H"):
            assert np.array_equal(getattr(a, f), getattr(b, f))
    # idx_in non-empty at layer 1: H still bit-unchanged at every layer
    st.idx_carried = np.arange(run.L_P, run.N)
    O.sparse_step(st, W, cfg, run0, O.MODE_FI, tau=-2.0)
    for a, b in zip(st.caches, before):
        assert np.array_equal(a.H, b.H)
    assert st.idx_carried.size == 0


@pytest.mark.parametrize("policy", [0, 1])
def test_q_cache_equals_literal_q(policy):
    """D6: recomputing Q only for idx_in (and decoded rows under 'carried') reproduces P:876."""
    cfg, run, W = _model("small128")
    run = replace(run, layer1_policy=policy, L_R=32, block=16)
    prompts = gen.prompt_tokens(1, 1, run.L_P, cfg.mask_id)
    tau = 0.9995
    toks_c, st_c = O.generate(prompts, W, cfg, run, tau, q_mode="cache")
    toks_l, st_l = O.generate(prompts, W, cfg, run, tau, q_mode="literal")
    assert np.array_equal(toks_c, toks_l)
    for a, b in zip(st_c[0].caches, st_l[0].caches):
        for f in ("K", "V", "Q", "C", "H"):
            assert np.allclose(getattr(a, f), getattr(b, f), rtol=1e-12, atol=1e-13)


def test_schedule_pattern():
    g = json.load(open(os.path.join(GOLD, "schedule_pattern.json")))
    run = configs.RunCfg(batch=1, L_P=4, L_R=16, T_full=g["T_full"], full_period=g["period"])
    pat = " ".join("R" if O.step_mode(t, run) == O.MODE_RO else "F" for t in range(16))
    assert pat == g["pattern"]
    assert [O.step_mode(t, run) for t in range(5)] == ["full"] * 4 + ["fi"]


def test_generation_invariants():
    """Budget, semi-AR order, prompt immutability, RO locality."""
    cfg, run, W = _model("small128")
    run = replace(run, L_R=64, block=32)
    prompt = gen.prompt_tokens(2, 1, run.L_P, cfg.mask_id)[0]
    st = O.init_state(prompt, cfg, run)
    for t in range(run.T_total):
        masked_before = int(np.sum(st.tokens == cfg.mask_id))
        snap = [c.copy() for c in st.caches] if st.caches else None
        mode = O.step_mode(t, run)
        pos, tok = O.denoise_step(st, W, cfg, run, t, 0.9995)
        assert len(pos) == min(run.n_u, masked_before)
        assert np.all(pos >= run.L_P + (t // run.block) * run.block)
        assert np.all(pos < run.L_P + (t // run.block + 1) * run.block)
        assert np.array_equal(st.tokens[: run.L_P], prompt)
        if mode == O.MODE_RO:
            for a, b in zip(st.caches, snap):
                for f in ("K", "V", "Q", "C", "H"):
                    assert np.array_equal(getattr(a, f)[: run.L_P], getattr(b, f)[: run.L_P])
    assert not np.any(st.tokens == cfg.mask_id)


@pytest.mark.parametrize("name", ["tiny", "small128_gqa"])
def test_all_salient_generation_equals_generate_full(name):
    """all-salient + full input every step (+ idx initialised to all rows) reproduces
    the full-recompute generation token for token."""
    cfg, run, W = _model(name)
    run = replace(run, full_period=1)
    if name != "tiny":
        run = replace(run, L_R=32, block=16)
    prompts = gen.prompt_tokens(4, run.batch, run.L_P, cfg.mask_id)
    ref, _ = O.generate_full(prompts, W, cfg, run)
    states = [O.init_state(p, cfg, run) for p in prompts]
    for st in states:
        for t in range(run.T_total):
            if t == run.T_full:
                st.idx_carried = np.arange(run.N)
            O.denoise_step(st, W, cfg, run, t, 2.0)
    assert np.array_equal(np.stack([s.tokens for s in states]), ref)


def test_saliency_monotone_in_tau():
    cfg, run, W = _model("tiny")
    counts = []
    for tau in (0.9, 0.99, 0.999, 0.99999):
        st = _warm_state(cfg, run, W)
        O.sparse_step(st, W, cfg, run, O.MODE_FI, tau)
        counts.append(st.sal_counts[-1][0])
    assert counts == sorted(counts)


def test_fraction_mode_generation_counts():
    """select_mode=1: every sparse layer selects round(f * L) rows of each sequence (no ties)."""
    cfg, run, W = _model("small128", qk_std=0.09)
    run = replace(run, L_R=32, block=16, select_mode=1)
    prompts = gen.prompt_tokens(5, 1, run.L_P, cfg.mask_id)
    _, states = O.generate(prompts, W, cfg, run, 0.25)
    for t, counts in zip(range(run.T_full, run.T_total), states[0].sal_counts):
        L = run.N if O.step_mode(t, run) == O.MODE_FI else run.L_R
        assert counts == [int(np.floor(0.25 * L + 0.5))] * cfg.n_layers
