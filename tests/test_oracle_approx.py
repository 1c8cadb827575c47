"""Pins of the oracle's APPROXIMATE-row path of SparseStep (Alg. 3 lines 5-11, P:879-889;
Alg. 4), its LM head and the paper_literal block, against independent torch-fp64
arithmetic (tests/torch_ref.py). CPU only.

The cache is filled with the torch block's own K/V/Q/C (C exact for the old keys), the layer
input changes on a strict subset idx_in of the input rows, and the oracle's sparse_layer must
satisfy, on the rows OUTSIDE idx_in (q unchanged there, D6):
  (i)   C_new - C_cache = softmax(Q K_new^T / sqrt(hd)) . dV_pad           (Alg. 4;
        dV_pad = V_new - V_old, zero outside idx_in; K_new = K merged at idx_in)
  (ii)  C_exact(K_new, V_new) - C_new = (A_new - A_old) . V_old             (Eq. 3's dropped
        term dS V_{t-1}, with A = softmax(Q K^T / sqrt(hd)))
and on idx_in: C_new = softmax(Q_new K_new^T) V_new, new K/V/Q rows, dV = V_new - V_old
(captured before the overwrite), and the post-attention rows of the block
in both residual readings (D2). Each plausible slip in the oracle — a flipped dV, C_cache - dC,
a scaled dC, the pre-merge K in ApproxAttn, a missing final or FFN RMSNorm — breaks one of them.
"""
from dataclasses import replace

import numpy as np
import pytest

import oracle as O
import torch_ref as T
from synth import configs, gen

TOL = 1e-9


def _model(name, **kw):
    cfg, run = configs.preset(name)
    cfg = replace(cfg, **kw)
    return cfg, run, gen.model_weights(cfg, 0)


def _close(a, b, tol=TOL):
    a, b = np.asarray(a), np.asarray(b)
    scale = max(np.abs(b).max(), 1e-30)
    err = np.abs(a - b).max() / scale
    assert err < tol, err


def _setup(name, mode, residual_mode, seed=0):
    cfg, run, W = _model(name, qk_std=0.09 if name != "tiny" else 0.18, residual_mode=residual_mode)
    lw = W["layers"][0]
    N = run.N
    rng = np.random.default_rng(seed)
    toks = np.concatenate([gen.prompt_tokens(seed, 1, run.L_P, cfg.mask_id)[0], np.full(run.L_R, cfg.mask_id)])
    x_old = W["emb"][toks]
    q0, k0, v0, c0, h0 = T.block(x_old, lw, cfg, residual_mode)
    cache = O.LayerCache(K=k0.copy(), V=v0.copy(), Q=q0.copy(), C=c0.copy(), H=h0.copy())
    input_rows = np.arange(N) if mode == "fi" else np.arange(run.L_P, N)
    idx_in = np.sort(rng.choice(input_rows, max(2, len(input_rows) // 3), replace=False))
    x_new = x_old.copy()
    x_new[idx_in] += rng.standard_normal((len(idx_in), cfg.d_model)) * np.abs(x_old).max()
    return cfg, run, lw, cache, x_new, idx_in, input_rows, (q0, k0, v0, c0, h0)


@pytest.mark.parametrize("name", ["tiny", "small128", "small128_gqa"])
@pytest.mark.parametrize("mode", ["fi", "ro"])
@pytest.mark.parametrize("residual_mode", [0, 1])
def test_sparse_layer_rows_against_independent_attention(name, mode, residual_mode):
    cfg, run, lw, cache, x_new, idx, rows, (q0, k0, v0, c0, h0) = _setup(name, mode, residual_mode)
    lc = cache.copy()
    r = O.sparse_layer(x_new, lc, lw, cfg, idx, 2.0, rows, q_mode="cache")   # tau > 1: all rows selected
    # independent reference
    qn, kn, vn = (t.numpy() for t in T.qkv(x_new[idx], idx, lw, cfg))
    K_new, V_new, Q = k0.copy(), v0.copy(), q0.copy()
    K_new[idx], V_new[idx], Q[idx] = kn, vn, qn
    dV_pad = V_new - v0
    apx = np.setdiff1d(rows, idx)
    at_apx = np.searchsorted(rows, apx)
    at_idx = np.searchsorted(rows, idx)
    assert len(apx) and len(idx)
    # (i) approximate rows: C_new - C_cache = A_new . dV_pad
    _close(r.C[at_apx] - c0[apx], T.sdpa(Q[apx], K_new, dV_pad, cfg).numpy())
    # (ii) the dropped term of Eq. 3: C_exact - C_new = (A_new - A_old) . V_old
    dropped = T.sdpa(Q[apx], K_new, v0, cfg).numpy() - T.sdpa(Q[apx], k0, v0, cfg).numpy()
    _close(T.sdpa(Q[apx], K_new, V_new, cfg).numpy() - r.C[at_apx], dropped)
    assert np.abs(dropped).max() > 1e3 * TOL * np.abs(c0).max()     # the pin is not vacuous
    # exact rows, dV, cache writes
    _close(r.C[at_idx], T.sdpa(qn, K_new, V_new, cfg).numpy())
    _close(r.dV, vn - v0[idx])
    _close(lc.K, K_new)
    _close(lc.V, V_new)
    _close(lc.Q, Q)
    _close(lc.C[rows], r.C)
    # post-attention rows (all input rows selected at tau > 1)
    assert np.array_equal(r.idx_out, rows)
    h, out = (t.numpy() for t in T.post_attention(x_new[rows], r.C, lw, cfg, residual_mode))
    _close(r.h, h)
    _close(r.out, out)
    _close(lc.H[rows], out)


@pytest.mark.parametrize("residual_mode", [0, 1])
def test_sparse_layer_partial_selection_keeps_cached_rows(residual_mode):
    """Rows outside idx_out keep FFN_OUT_cache bit-for-bit; selected rows get the block."""
    cfg, run, lw, cache, x_new, idx, rows, (q0, k0, v0, c0, h0) = _setup("small128", "fi", residual_mode, seed=3)
    lc = cache.copy()
    r0 = O.sparse_layer(x_new, cache.copy(), lw, cfg, idx, 2.0, rows, q_mode="cache")
    tau = float(np.median(r0.s))
    r = O.sparse_layer(x_new, lc, lw, cfg, idx, tau, rows, q_mode="cache")
    sel = rows[r.s < tau]
    assert np.array_equal(r.idx_out, sel) and 0 < len(sel) < len(rows)
    _, out = (t.numpy() for t in T.post_attention(x_new[sel], r0.C[np.searchsorted(rows, sel)], lw, cfg,
                                                    residual_mode))
    _close(lc.H[sel], out)
    rest = np.setdiff1d(np.arange(run.N), sel)
    assert np.array_equal(lc.H[rest], h0[rest])


@pytest.mark.parametrize("name", ["tiny", "small128_gqa"])
def test_full_layer_paper_literal_vs_independent_torch(name):
    """residual_mode 1 (paper_literal): h = RMSNorm(C W_o) ; out = FFN(h)."""
    cfg, run, W = _model(name, residual_mode=1)
    toks = np.concatenate([gen.prompt_tokens(1, 1, run.L_P, cfg.mask_id)[0], np.full(run.L_R, cfg.mask_id)])
    x = W["emb"][toks]
    lc = O.full_layer(x, W["layers"][0], cfg)
    q, k, v, c, out = T.block(x, W["layers"][0], cfg, residual_mode=1)
    for a, b in [(lc.Q, q), (lc.K, k), (lc.V, v), (lc.C, c), (lc.H, out)]:
        _close(a, b, 1e-10)


@pytest.mark.parametrize("name", ["tiny", "small128"])
def test_lm_logits_vs_independent_torch(name):
    """logits = RMSNorm_f(H_L) W_lm^T (Alg. 2 line 10), on rows of any scale."""
    cfg, run, W = _model(name)
    rng = np.random.default_rng(7)
    h = rng.standard_normal((9, cfg.d_model)) * np.array([1e-3, 1, 30, 1, 1, 1, 1, 1, 5])[:, None]
    _close(O.lm_logits(h, W, cfg), T.lm_logits(h, W, cfg), 1e-12)


def test_generate_with_approximate_rows_decodes_like_a_pinned_path():
    """End-to-end Alg. 1 on tiny with a real partial selection: every step's H_L for the
    candidate rows equals an independent recomputation of the oracle state's last layer."""
    cfg, run, W = _model("tiny")
    st = O.init_state(gen.prompt_tokens(2, 1, run.L_P, cfg.mask_id)[0], cfg, run)
    for t in range(run.T_total):
        O.denoise_step(st, W, cfg, run, t, 0.995)
        lc = st.caches[-1]
        # the last layer's H rows that were selected this step must be the block applied to the
        # cached contexts and the previous layer's hidden rows (post-attention is row-local)
        x_prev = st.caches[-2].H
        if O.step_mode(t, run) != O.MODE_FULL and st.idx_carried.size:
            sel = st.idx_carried
            _, out = T.post_attention(x_prev[sel], lc.C[sel], W["layers"][-1], cfg, 0)
            _close(lc.H[sel], out.numpy(), 1e-10)
