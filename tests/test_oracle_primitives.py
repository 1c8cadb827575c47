"""Pins of the oracle's primitives against closed forms, special cases, independent torch-fp64
routines and SPEC/paper examples. CPU only."""
import json
import math
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle as O
from synth import gen

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- generator (synth) pins

def test_splitmix64_reference_values():
    g = _gold("splitmix64.json")
    got = [format(gen._mix64_py(x), "016x") for x in g["mix64_of"]]
    assert got == g["expected_hex"]
    arr = gen._mix64_np(np.asarray(g["mix64_of"], dtype=np.uint64))
    assert [format(int(v), "016x") for v in arr] == g["expected_hex"]


def test_ih4_moments_and_bf16():
    v = gen.ih4_normal(seed=1, stream=7, shape=(200000,), std=0.02)
    assert abs(v.mean()) < 2e-4
    assert abs(v.std() - 0.02) < 3e-4
    assert np.abs(v).max() <= 0.02 * math.sqrt(12) + 1e-6           # Irwin-Hall(4) support
    bits = gen.f32_to_bf16_bits(v.astype(np.float32))
    assert np.array_equal(gen.bf16_bits_to_f32(bits).astype(np.float64), v)   # already bf16
    # element-wise addressable: a slice regenerates identically
    part = gen.ih4_normal_bf16_bits(1, 7, 100, 0.02, start=5000)
    assert np.array_equal(part, gen.ih4_normal_bf16_bits(1, 7, 200000, 0.02)[5000:5100])


def test_bf16_rounding_is_rne():
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -2.5, 1.0 + 2 ** -9], dtype=np.float32)
    got = gen.bf16_bits_to_f32(gen.f32_to_bf16_bits(x))
    ref = torch.tensor(x).to(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(got, ref)


# ---------------------------------------------------------------- numerics pins

def test_rmsnorm_closed_forms():
    assert np.allclose(O.rms_norm(np.ones((1, 4)), np.ones(4), 0.0), 1.0, atol=0, rtol=0)
    rng = np.random.default_rng(0)
    x = rng.standard_normal((5, 33))
    g = rng.standard_normal(33)
    ref = F.rms_norm(torch.tensor(x), (33,), weight=torch.tensor(g), eps=1e-6).numpy()
    assert np.allclose(O.rms_norm(x, g, 1e-6), ref, rtol=1e-13, atol=1e-14)


@pytest.mark.parametrize("alpha", [0.5, 3.7, 100.0])
def test_prop1_scale_invariance(alpha):
    """Prop. 1: RMSNorm((alpha C) W_o) = RMSNorm(C W_o), exact for eps = 0."""
    rng = np.random.default_rng(1)
    C = rng.standard_normal((4, 16))
    Wo = rng.standard_normal((16, 16))
    g = np.ones(16)
    assert np.allclose(O.rms_norm((alpha * C) @ Wo, g, 0.0), O.rms_norm(C @ Wo, g, 0.0),
                       rtol=1e-9, atol=1e-12)


def test_rope_special_cases():
    # S:69 single pair (1,0), pos=1, theta=1 -> (cos 1, sin 1)
    out = O.rope(np.array([[1.0, 0.0]]), np.array([1]), 1.0, 2)
    assert np.allclose(out, [[math.cos(1.0), math.sin(1.0)]], atol=1e-15)
    rng = np.random.default_rng(2)
    x = rng.standard_normal((3, 32))
    assert np.array_equal(O.rope(x, np.zeros(3), 1e4, 16), x)                  # position 0 = identity
    # norm per rotated pair preserved
    y = O.rope(x, np.array([5, 17, 900]), 1e4, 16)
    xr, yr = x.reshape(3, 2, 16), y.reshape(3, 2, 16)
    nx = xr[..., :8] ** 2 + xr[..., 8:] ** 2
    ny = yr[..., :8] ** 2 + yr[..., 8:] ** 2
    assert np.allclose(nx, ny, rtol=1e-12)


def test_rope_matches_complex_rotation_and_is_relative():
    """Independent formulation: pair (x_k, x_{k+h/2}) as a complex number times e^{i pos w_k}."""
    rng = np.random.default_rng(3)
    hd, theta = 16, 5e5
    x = rng.standard_normal((4, 2 * hd))
    pos = np.array([0, 3, 100, 955])
    w = theta ** (-(np.arange(hd // 2) * 2.0) / hd)
    xr = x.reshape(4, 2, hd)
    z = (xr[..., : hd // 2] + 1j * xr[..., hd // 2:]) * np.exp(1j * pos[:, None, None] * w)
    ref = np.concatenate([z.real, z.imag], axis=-1).reshape(4, 2 * hd)
    assert np.allclose(O.rope(x, pos, theta, hd), ref, rtol=1e-12, atol=1e-12)
    # <rope(q,p), rope(k,p')> depends only on p - p'
    q, k = rng.standard_normal((1, hd)), rng.standard_normal((1, hd))
    d1 = O.rope(q, [10], theta, hd) @ O.rope(k, [4], theta, hd).T
    d2 = O.rope(q, [106], theta, hd) @ O.rope(k, [100], theta, hd).T
    assert np.allclose(d1, d2, rtol=1e-10)


def test_softmax_special_cases():
    assert np.allclose(O.softmax_rows(np.zeros((1, 4))), 0.25)
    assert np.allclose(O.softmax_rows(np.array([[1000.0, 0.0]])), [[1.0, 0.0]], atol=1e-12)
    s = np.random.default_rng(4).standard_normal((3, 5))
    assert np.allclose(O.softmax_rows(s).sum(1), 1.0, atol=1e-12)


@pytest.mark.parametrize("H,KVH", [(4, 4), (4, 1), (6, 2)])
def test_attention_vs_torch_sdpa(H, KVH):
    rng = np.random.default_rng(5)
    hd, Lq, N = 16, 7, 11
    q = rng.standard_normal((Lq, H * hd))
    k = rng.standard_normal((N, KVH * hd))
    v = rng.standard_normal((N, KVH * hd))
    tq = torch.tensor(q).view(Lq, H, hd).transpose(0, 1)
    tk = torch.tensor(k).view(N, KVH, hd).transpose(0, 1).repeat_interleave(H // KVH, 0)
    tv = torch.tensor(v).view(N, KVH, hd).transpose(0, 1).repeat_interleave(H // KVH, 0)
    ref = F.scaled_dot_product_attention(tq, tk, tv, is_causal=False).transpose(0, 1).reshape(Lq, -1)
    got = O.attention(q, k, v, H, KVH, hd)
    assert np.allclose(got, ref.numpy(), rtol=1e-12, atol=1e-12)


def test_attention_saturation():
    """one key equal to the (scaled) query, others orthogonal -> context ~ that value row."""
    hd = 16
    q = np.zeros((1, hd)); q[0, 0] = 60.0
    k = np.zeros((3, hd)); k[1, 0] = 60.0; k[0, 1] = 1.0; k[2, 2] = 1.0
    v = np.arange(3 * hd, dtype=np.float64).reshape(3, hd)
    assert np.allclose(O.attention(q, k, v, 1, 1, hd), v[1:2], atol=1e-9)


def test_cosine_special_cases():
    rng = np.random.default_rng(6)
    a = rng.standard_normal((50, 64))
    assert np.all(O.cosine_rows(a, a) == 1.0)                                   # exactly 1 (D9)
    b = a.astype(np.float32).astype(np.float64)
    assert np.all(O.cosine_rows(b, b) == 1.0)
    assert np.allclose(O.cosine_rows(a, -a), -1.0, atol=1e-15)
    e1, e2 = np.eye(2, 4)[0:1], np.eye(2, 4)[1:2]
    assert O.cosine_rows(e1, e2)[0] == 0.0
    z = np.zeros((1, 4))
    assert O.cosine_rows(z, z)[0] == 1.0 and O.cosine_rows(z, e1)[0] == 0.0
    s = O.cosine_rows(a, rng.standard_normal((50, 64)))
    assert np.all(np.abs(s) <= 1 + 1e-12)


def test_prop2_exact_component():
    """P:1073 / S:643: for unit vectors, |u - v| = sqrt(2 (1 - s))."""
    rng = np.random.default_rng(7)
    u = rng.standard_normal((20, 32)); u /= np.linalg.norm(u, axis=1, keepdims=True)
    v = u + 0.1 * rng.standard_normal((20, 32)); v /= np.linalg.norm(v, axis=1, keepdims=True)
    s = O.cosine_rows(u, v)
    assert np.allclose(np.linalg.norm(u - v, axis=1), np.sqrt(2 * (1 - s)), rtol=1e-9, atol=1e-12)


def test_select_salient_worked_example():
    g = _gold("select_example.json")
    pos = g["offset"] + np.arange(len(g["s"]))
    assert O.select_salient(g["s"], g["tau"], pos).tolist() == g["expected"]
    assert O.select_salient(g["s"], g["tau_all"], pos).tolist() == pos.tolist()
    assert O.select_salient(g["s"], g["tau_none"], pos).tolist() == []
    # ties: '<' excludes s == tau, '<=' includes it (D1)
    assert O.select_salient([0.99], 0.99, [3], cmp=0).tolist() == []
    assert O.select_salient([0.99], 0.99, [3], cmp=1).tolist() == [3]


def test_select_salient_brute_force_and_monotone():
    rng = np.random.default_rng(8)
    s = rng.uniform(0.9, 1.0, 300)
    pos = np.arange(100, 400)
    prev = set()
    for tau in np.linspace(0.9, 1.0, 21):
        got = O.select_salient(s, tau, pos)
        assert got.tolist() == [p for p, v in zip(pos, s) if v < tau]
        assert prev <= set(got.tolist())
        prev = set(got.tolist())


# ---------------------------------------------------------------- Alg. 4 and Eq. 3

def test_approx_attention_dense_zero_padded():
    rng = np.random.default_rng(9)
    H, KVH, hd, L, N = 4, 2, 16, 9, 13
    q = rng.standard_normal((L, H * hd))
    k = rng.standard_normal((N, KVH * hd))
    idx = np.array([1, 4, 5, 12])
    dv = rng.standard_normal((len(idx), KVH * hd))
    pad = np.zeros((N, KVH * hd)); pad[idx] = dv
    dense = O.attention(q, k, pad, H, KVH, hd)                                 # A · dV_padded
    assert np.allclose(O.approx_attention(q, k, dv, idx, H, KVH, hd), dense, rtol=1e-12, atol=1e-13)
    assert np.all(O.approx_attention(q, k, np.zeros_like(dv), idx, H, KVH, hd) == 0)   # dV = 0
    assert np.all(O.approx_attention(q, k, dv[:0], idx[:0], H, KVH, hd) == 0)          # idx = {}
    full = rng.standard_normal((N, KVH * hd))                                          # idx = all
    assert np.allclose(O.approx_attention(q, k, full, np.arange(N), H, KVH, hd),
                       O.attention(q, k, full, H, KVH, hd), rtol=1e-12, atol=1e-13)


def test_eq3_identity():
    rng = np.random.default_rng(10)
    S0 = O.softmax_rows(rng.standard_normal((6, 8)))
    S1 = O.softmax_rows(rng.standard_normal((6, 8)))
    V0, V1 = rng.standard_normal((8, 5)), rng.standard_normal((8, 5))
    lhs, rhs = O.eq3_terms(S0, S1, V0, V1)
    assert np.allclose(lhs, rhs, atol=1e-10)


# ---------------------------------------------------------------- unmasking (D13)

def test_process_logit_brute_force():
    rng = np.random.default_rng(11)
    for trial in range(20):
        n, V = int(rng.integers(1, 9)), 7
        pos = np.sort(rng.choice(np.arange(50, 90), n, replace=False))
        z = rng.standard_normal((n, V))
        if trial % 3 == 0:
            z[1 % n] = z[0]                              # tie in confidence
        n_u = int(rng.integers(1, 4))
        p, t, _ = O.process_logit(pos, z, n_u)
        probs = np.exp(z) / np.exp(z).sum(1, keepdims=True)
        conf = probs.max(1)
        brute = sorted(range(n), key=lambda i: (-round(conf[i], 12), pos[i]))[:n_u]
        assert p.tolist() == [pos[i] for i in brute]
        assert t.tolist() == [int(np.argmax(z[i])) for i in brute]


def test_process_logit_never_commits_the_mask_token():
    """D22: even when [M] has the largest logit, the committed token is the best other one and its
    confidence is its probability over the whole vocabulary (brute force)."""
    rng = np.random.default_rng(5)
    V, mask = 9, 8
    pos = np.arange(30, 36)
    z = rng.standard_normal((6, V))
    z[:, mask] = z.max(axis=1) + 1.0 + rng.random(6)          # the mask logit dominates every row
    p, t, c = O.process_logit(pos, z, 3, mask_id=mask)
    probs = np.exp(z) / np.exp(z).sum(1, keepdims=True)
    best = np.argmax(np.where(np.arange(V) == mask, -np.inf, z), axis=1)
    conf = probs[np.arange(6), best]
    brute = sorted(range(6), key=lambda i: (-round(conf[i], 12), pos[i]))[:3]
    assert mask not in t.tolist()
    assert p.tolist() == [pos[i] for i in brute]
    assert t.tolist() == [int(best[i]) for i in brute]
    assert np.allclose(c, conf[brute], rtol=1e-12)


def test_generation_unmasks_exactly_n_u_per_step_with_a_dominant_mask_logit():
    """S:347 budget under D22: a model whose LM head favours [M] still unmasks min(n_u, remaining)
    positions every step and never writes the mask id."""
    from dataclasses import replace
    from synth import configs, gen
    cfg, run = configs.preset("tiny")
    W = gen.model_weights(cfg, 1)
    # [M]'s embedding and LM-head row share a direction that the residual stream of every masked
    # row carries: [M] wins every masked row's logits
    u = np.random.default_rng(0).standard_normal(cfg.d_model)
    u /= np.linalg.norm(u)
    W["emb"], W["lm_head"] = W["emb"].copy(), W["lm_head"].copy()
    W["emb"][cfg.mask_id], W["lm_head"][cfg.mask_id] = 5.0 * u, 2.0 * u
    st0 = O.init_state(gen.prompt_tokens(2, run.batch, run.L_P, cfg.mask_id)[0], cfg, run)
    HL = O.full_step(st0, W, cfg)
    cand = O.candidate_rows(st0.tokens, cfg, run)
    assert np.all(O.lm_logits(HL[cand], W, cfg).argmax(1) == cfg.mask_id)
    prompts = gen.prompt_tokens(2, run.batch, run.L_P, cfg.mask_id)
    st = O.init_state(prompts[0], cfg, run)
    left = run.L_R
    for t in range(run.T_total):
        pos, tok = O.denoise_step(st, W, cfg, run, t, 0.99)
        assert len(pos) == min(run.n_u, left) and cfg.mask_id not in tok.tolist()
        left -= len(pos)
    assert not np.any(st.tokens == cfg.mask_id)


def test_process_logit_all_equal_picks_lowest_positions():
    pos = np.array([40, 41, 42, 43])
    p, t, _ = O.process_logit(pos, np.zeros((4, 5)), 2)
    assert p.tolist() == [40, 41] and t.tolist() == [0, 0]


# ---------------------------------------------------------------- paper's printed arithmetic

def test_cost_example_from_paper():
    g = _gold("cost_example.json")
    assert O.fastdllm_computed_tokens(g["L_P"], g["L_R"], g["B"], g["n_u"], dual=False) == g["prefix_per_step"]
    assert O.fastdllm_computed_tokens(g["L_P"], g["L_R"], g["B"], g["n_u"], dual=True) == g["dual_per_step"]
    assert (g["prefix_avg_block_tokens"] * 31 + g["refresh_tokens"]) / 32 == g["prefix_per_step"]


# ---------------------------------------------------------------- fraction-controlled threshold (D19)

def test_quantile_threshold_brute_force():
    rng = np.random.default_rng(12)
    for n in (1, 5, 64, 257):
        s = rng.uniform(0.5, 1.0, n)
        for f in (0.0, 0.05, 0.1, 0.37, 0.5, 1.0):
            tau = O.quantile_threshold(s, f)
            k = int(np.floor(f * n + 0.5))
            got = O.select_salient(s, tau, np.arange(n))
            assert sorted(got.tolist()) == sorted(np.argsort(s)[:k].tolist())


def test_quantile_threshold_ties_select_fewer():
    s = np.array([0.9, 1.0, 1.0, 1.0])           # identical rows give s == 1 exactly (D9)
    assert O.select_salient(s, O.quantile_threshold(s, 0.75), np.arange(4)).tolist() == [0]
