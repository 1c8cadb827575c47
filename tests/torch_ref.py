"""Independent torch-fp64 transformer pieces used to PIN the oracle (tests only).

Written without reference to oracle/: complex-number RoPE (torch.polar), F.rms_norm, F.linear,
F.scaled_dot_product_attention with repeated kv heads, F.silu. Each function restates the
passage it follows:
  - pre-norm residual block (D2 primary, LLaDA/Dream): h = x + C W_o ; out = h + FFN(RMSNorm(h))
  - paper_literal block (Alg. 2/3 lines 'x <- LN(OutProj(C)); x <- FFN(x)')
  - LM head after the final RMSNorm (Alg. 2 line 10)
"""
from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F


def t64(a):
    return torch.as_tensor(np.asarray(a, dtype=np.float64))


def rope(z, pos, n_heads, hd, theta):
    """Rotate-half RoPE as a complex multiplication: (x_k + i x_{k+hd/2}) * e^{i pos theta^(-2k/hd)}."""
    z = t64(z)
    n = z.shape[0]
    freqs = theta ** (-torch.arange(0, hd, 2, dtype=torch.float64) / hd)
    rot = torch.polar(torch.ones(n, hd // 2, dtype=torch.float64), t64(pos)[:, None] * freqs[None])
    z = z.view(n, n_heads, hd)
    c = torch.complex(z[..., : hd // 2], z[..., hd // 2:]) * rot[:, None, :]
    return torch.cat([c.real, c.imag], -1).reshape(n, n_heads * hd)


def qkv(x, pos, w, cfg):
    """RMSNorm(x) then Q/K/V projections (+bias), RoPE on Q and K at global positions."""
    X = t64(x)
    Xn = F.rms_norm(X, (cfg.d_model,), weight=t64(w["g_attn"]), eps=cfg.rms_eps)
    b = (lambda k: t64(w[k])) if cfg.qkv_bias else (lambda k: None)
    q = F.linear(Xn, t64(w["wq"]), b("bq"))
    k = F.linear(Xn, t64(w["wk"]), b("bk"))
    v = F.linear(Xn, t64(w["wv"]), b("bv"))
    return (rope(q, pos, cfg.n_heads, cfg.head_dim, cfg.rope_theta),
            rope(k, pos, cfg.n_kv_heads, cfg.head_dim, cfg.rope_theta), v)


def sdpa(q, k, v, cfg):
    """softmax(q k^T / sqrt(hd)) v per head, non-causal, kv heads repeated for GQA."""
    q, k, v = t64(q), t64(k), t64(v)
    H, KVH, hd = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    if q.shape[0] == 0:
        return torch.zeros(0, H * hd, dtype=torch.float64)
    qh = q.view(-1, H, hd).transpose(0, 1)
    kh = k.view(-1, KVH, hd).transpose(0, 1).repeat_interleave(H // KVH, 0)
    vh = v.view(-1, KVH, hd).transpose(0, 1).repeat_interleave(H // KVH, 0)
    return F.scaled_dot_product_attention(qh, kh, vh).transpose(0, 1).reshape(q.shape[0], H * hd)


def post_attention(x, c, w, cfg, residual_mode):
    """Returns (h, out) of the O-projection + FFN part of the block."""
    X, Cc = t64(x), t64(c)
    o = F.linear(Cc, t64(w["wo"]))
    ffn = lambda z: F.linear(F.silu(F.linear(z, t64(w["w_gate"]))) * F.linear(z, t64(w["w_up"])), t64(w["w_down"]))
    if residual_mode == 0:
        h = X + o
        return h, h + ffn(F.rms_norm(h, (cfg.d_model,), weight=t64(w["g_ffn"]), eps=cfg.rms_eps))
    h = F.rms_norm(o, (cfg.d_model,), weight=t64(w["g_ffn"]), eps=cfg.rms_eps)
    return h, ffn(h)


def block(x, w, cfg, residual_mode=0):
    """A whole layer over all rows; returns numpy (Q, K, V, C, out)."""
    n = x.shape[0]
    q, k, v = qkv(x, np.arange(n), w, cfg)
    C = sdpa(q, k, v, cfg)
    _, out = post_attention(x, C, w, cfg, residual_mode)
    return q.numpy(), k.numpy(), v.numpy(), C.numpy(), out.numpy()


def lm_logits(h, W, cfg):
    return F.linear(F.rms_norm(t64(h), (cfg.d_model,), weight=t64(W["g_final"]), eps=cfg.rms_eps),
                    t64(W["lm_head"])).numpy()
