"""GPU-vs-oracle parity of the Alg. 1 loop body, dyllm_denoise_step (
P:804-823), resynchronised from the oracle state at every step.

Each step t: the oracle's (bf16-rounded) state — tokens, every layer's K/V/Q/C/H, H_0, the carried
salient set and the rows decoded at t-1 (D5) — is imported into the GPU cache, and the GPU
runs dyllm_denoise_step(t) with a per-layer trace of its selected lists and similarities. Every
layer of that step is then re-run by the oracle from the layer's own GPU input (teacher forcing
inside the step: H_l as the GPU's previous layer left it, and idx_in = the GPU's previous list, or
for layer 1 the oracle's own layer1_idx of the carried set and decoded rows), so that bf16 errors
do not accumulate across layers and a near-tie that went the other way at one layer does not
poison the next. Compared (north_star bars):
  - sparse layers: the selected set, bit-exact outside |s - tau| < 1e-3; s of every input row;
    the new context rows C of every input row; K/V/Q rows of idx_in (and, under the literal
    layer-1 policy, the Q-only refresh of decoded rows); the hidden rows H_{l+1} of the rows both
    sides selected (2e-2 max row-relative error); rows neither selected keep H bit-unchanged;
  - FullSteps: K, V, Q, C, H of every row of every layer;
  - unmasking: process_logit on the GPU's own H_L (positions and tokens exact unless a near-tie)
    and H_0 of the decoded rows (= E[token], bit-exact).
The next step resynchronises from the oracle's own, free-running Alg. 1 step.
Head_dim-128 configs run the response tiles with incremental softmax statistics (SURVEY §8f1,
D20): after the import the statistics are recomputed densely from the imported K and Q, so the
step updates them by the changed keys' old and new terms exactly as in a free-running generation.
"""
import copy
from dataclasses import replace

import numpy as np
import pytest
import torch

import oracle as O
from synth import gen
from gpu_helpers import Model, bf16_round, from_dev, import_states, row_rel_err, storage_round

pytestmark = pytest.mark.gpu
TOL = 2e-2
BAND = 1e-3
S_TOL = 5e-3
TOL_F32 = 1e-4      # north_star: hidden states within 1e-4 max relative error in fp32 mode
S_TOL_F32 = 1e-5
CONF_RTOL = 1e-4    # near-tie margins of process_logit on the same bf16 H_L rows (fp32 LM head vs fp64)
LOGIT_ATOL = 1e-3
QK = {"tiny": 0.18, "small128": 0.09, "small128_gqa": 0.09, "small64": 0.08}
LM_STD = {"tiny": 1.0}   # LM-head std (default 0.25): distinct unmasking confidences


def _calibrated_taus(m, states, frac):
    """Fixed-tau mode (the paper's rule): one tau per layer, calibrated once from the ORACLE at the
    first sparse step as the mean over sequences of the per-layer frac-quantile."""
    cp = copy.deepcopy(states)
    run1 = replace(m.run, select_mode=1)
    for st in cp:
        O.denoise_step(st, m.W, m.cfg, run1, m.run.T_full, frac)
    return np.array([np.mean([O.quantile_threshold(st.layer_results[l].s, frac) for st in cp])
                     for l in range(m.cfg.n_layers)], dtype=np.float64)


def _rows(lists, off, s, N):
    return set((lists[off[s]:off[s + 1]] - s * N).tolist())


def _check_decode(gp, gt, HL_rows, cand, W, cfg, n_u, rnd=bf16_round):
    """Unmasking parity (D13) on the GPU's own last-layer rows. The decision is taken in the
    precision the GPU path defines (its LM-head GEMM reads the RMSNorm_f output rounded to bf16,
    D12), so the reference logits are fp64 products of those bf16 rows. Returns False (not
    compared) when the choice is a near-tie at that precision; else positions and tokens match."""
    if len(cand) == 0:
        return len(gp) == 0
    z = rnd(O.rms_norm(HL_rows, W["g_final"], cfg.rms_eps)) @ W["lm_head"].T
    pos, tok, conf = O.process_logit(cand, z, n_u, cfg.mask_id)
    k = len(pos)
    zn = z.copy()
    zn[:, cfg.mask_id] = -np.inf                     # D22: [M] is never a prediction
    allc = np.sort(1.0 / np.exp(z - zn.max(axis=1, keepdims=True)).sum(axis=1))[::-1]
    chosen = np.searchsorted(cand, pos)
    top2 = np.sort(zn[chosen], axis=1)[:, -2:]
    if (len(allc) > k and allc[k - 1] - allc[k] < CONF_RTOL * allc[k - 1]) or np.any(top2[:, 1] - top2[:, 0] < LOGIT_ATOL):
        return False
    assert sorted(gp.tolist()) == sorted(pos.tolist()), (gp, pos)
    assert dict(zip(gp.tolist(), gt.tolist())) == dict(zip(pos.tolist(), tok.tolist()))
    return True


def _denoise_parity(name, select_mode, policy, residual_mode=0, cmp=0, steps=12, seed=0, frac=0.1,
                    inc=True, empty_seq_at=None, n_u=4, qk=None, dtype=0):
    """dtype 1: the fp32-parity mode (D12), compared at the north_star's fp32 bar (TOL_F32)."""
    m = Model(name, seed=seed, qk_std=qk or QK[name], lm_std=LM_STD.get(name, 0.25), select_mode=select_mode,
              layer1_policy=policy, residual_mode=residual_mode, cmp=cmp, n_u=n_u, dtype=dtype)
    rnd = storage_round(dtype)
    tol, s_tol = (TOL, S_TOL) if dtype == 0 else (TOL_F32, S_TOL_F32)
    cfg, run, dy = m.cfg, m.run, m.dyllm
    N, b, nl = run.N, run.batch, cfg.n_layers
    steps = min(steps, run.T_total)
    prompts = gen.prompt_tokens(seed + 31, b, run.L_P, cfg.mask_id)
    states = [O.init_state(p, cfg, run) for p in prompts]
    cache = m.new_cache()
    dev = "cuda"
    tr_lists = torch.zeros(nl * b * N, dtype=torch.int32, device=dev)
    tr_offs = torch.zeros(nl * (b + 1), dtype=torch.int32, device=dev)
    tr_sims = torch.zeros(nl * b * N, dtype=torch.float32, device=dev)
    cache.set_trace(tr_lists, tr_offs, tr_sims)
    dec_pos = torch.full((b, run.n_u), -1, dtype=torch.int32, device=dev)
    dec_tok = torch.full((b, run.n_u), -1, dtype=torch.int32, device=dev)
    emb_bf = bf16_round(m.W["emb"])
    taus = None
    stats = dict(steps=0, band=0, compared_rows=0, disagreed=0, seq_layers=0, decode_checked=0, decode_ties=0)
    for t in range(steps):
        mode = O.step_mode(t, run)
        if mode != O.MODE_FULL and taus is None:
            taus = (np.full(nl, frac) if select_mode == 1 else _calibrated_taus(m, states, frac))
        if t == empty_seq_at and b > 1:      # a sequence with an empty layer-1 idx_in (fixed-tau mode)
            states[1].idx_carried = np.zeros(0, dtype=np.int64)
            states[1].decoded_prev = np.zeros(0, dtype=np.int64)
        # ---- resynchronise the GPU from the (bf16-rounded) oracle state
        pre = [copy.deepcopy(st) for st in states]
        for st in pre:
            if st.caches:                    # the embeddings of the current tokens (Alg. 3 line 1)
                st.H0 = m.W["emb"][st.tokens]
            for lc in st.caches:
                lc.K, lc.V, lc.Q, lc.C, lc.H = (rnd(x) for x in (lc.K, lc.V, lc.Q, lc.C, lc.H))
            if st.H0 is not None:
                st.H0 = rnd(st.H0)
        if pre[0].caches:
            import_states(m, cache, pre)
            if inc and cfg.head_dim == 128:
                for l in range(nl):
                    cache.refresh_stats(l)
        toks = torch.tensor(np.stack([st.tokens for st in pre]), dtype=torch.int32, device=dev)
        if pre[0].idx_carried is None:
            cache.set_carried(None)
        else:
            rows = [s * N + int(p) for s, st in enumerate(pre) for p in st.idx_carried]
            off = np.cumsum([0] + [len(st.idx_carried) for st in pre]).astype(np.int32)
            buf = torch.zeros(max(b * N, 1), dtype=torch.int32)
            buf[: len(rows)] = torch.tensor(rows, dtype=torch.int32)
            cache.set_carried(buf.to(dev), torch.tensor(off, device=dev))
        if t == 0:
            cache.set_decoded(None)
        else:
            d = np.full((b, run.n_u), -1, np.int32)
            for s, st in enumerate(pre):
                d[s, : len(st.decoded_prev)] = s * N + st.decoded_prev
            cache.set_decoded(torch.tensor(d, device=dev))
        # ---- the GPU step
        rc = cache.denoise_step(t, taus if taus is not None else np.zeros(nl), toks, dec_pos, dec_tok)
        assert rc == 0
        torch.cuda.synchronize()
        stats["steps"] += 1
        G = {w: [from_dev(cache.export(l, w)) for l in range(nl)] for w in (dy.K, dy.V, dy.Q, dy.CTX)}
        st_tok = [st.tokens for st in pre]
        Hg = [from_dev(cache.export(l, dy.H)) for l in range(nl + 1)]
        # ---- every layer re-run by the oracle from the GPU's own layer input
        if mode == O.MODE_FULL:
            for s in range(b):
                for l in range(nl):
                    x_in = emb_bf[st_tok[s]] if l == 0 else Hg[l][s]    # H_0: before this step's commit
                    lc = O.full_layer(x_in, m.W["layers"][l], cfg)
                    for w, f in ((dy.K, "K"), (dy.V, "V"), (dy.Q, "Q"), (dy.CTX, "C")):
                        assert row_rel_err(G[w][l][s], getattr(lc, f)).max() < tol, (t, l, s, f)
                    assert row_rel_err(Hg[l + 1][s], lc.H).max() < tol, (t, l, s)
        else:
            lists = tr_lists.view(nl, b * N).cpu().numpy()
            offs = tr_offs.view(nl, b + 1).cpu().numpy()
            sims = tr_sims.view(nl, b, N).cpu().numpy()
            rows_in = np.arange(N) if mode == O.MODE_FI else np.arange(run.L_P, N)
            for s, st in enumerate(pre):
                idx = O.layer1_idx(copy.deepcopy(st), run, rows_in)
                q_extra = np.intersect1d(st.decoded_prev, rows_in) if policy == 0 else ()
                for l in range(nl):
                    lc = st.caches[l].copy()
                    thr = (lambda sv, f=taus[l]: O.quantile_threshold(sv, f)) if select_mode == 1 else taus[l]
                    x_in = emb_bf[st.tokens] if l == 0 else Hg[l][s]      # H_0: before this step's commit
                    r = O.sparse_layer(x_in, lc, m.W["layers"][l], cfg, idx, thr, rows_in, cmp,
                                       q_mode="cache", q_extra=q_extra if l == 0 else ())
                    tau_sl = O.quantile_threshold(r.s, taus[l]) if select_mode == 1 else taus[l]
                    band = set(rows_in[np.abs(r.s - tau_sl) < BAND].tolist())
                    got, ref = _rows(lists[l], offs[l], s, N), set(r.idx_out.tolist())
                    assert got - band == ref - band, (t, l, s, sorted(got ^ ref))
                    assert np.abs(sims[l, s, rows_in] - r.s).max() < s_tol, (t, l, s)
                    assert row_rel_err(G[dy.CTX][l][s, rows_in], r.C).max() < tol, (t, l, s)
                    rec = np.union1d(idx, q_extra if l == 0 else []).astype(np.int64)
                    for w, f in ((dy.K, "K"), (dy.V, "V"), (dy.Q, "Q")):
                        if len(rec):
                            assert row_rel_err(G[w][l][s, rec], getattr(lc, f)[rec]).max() < tol, (t, l, s, f)
                    both = np.array(sorted(got & ref), dtype=np.int64)
                    if len(both):
                        assert row_rel_err(Hg[l + 1][s, both], lc.H[both]).max() < tol, (t, l, s)
                    untouched = np.array(sorted(set(range(N)) - got - ref), dtype=np.int64)
                    assert np.array_equal(Hg[l + 1][s, untouched], st.caches[l].H[untouched]), (t, l, s)
                    stats["band"] += len(band)
                    stats["compared_rows"] += len(rows_in)
                    stats["seq_layers"] += 1
                    stats["disagreed"] += int(got != ref)
                    idx = np.array(sorted(got), dtype=np.int64)      # the GPU's list feeds the next layer
        # ---- unmasking on the GPU's H_L, and the H_0 refresh of the decoded rows
        dp, dt = dec_pos.cpu().numpy(), dec_tok.cpu().numpy()
        H0 = from_dev(cache.export(0, dy.H))
        for s, st in enumerate(pre):
            gp = dp[s][dp[s] >= 0] - s * N
            gt = dt[s][: len(gp)]
            assert np.array_equal(H0[s, gp], emb_bf[gt])
            cand = O.candidate_rows(st.tokens, cfg, run)
            if _check_decode(gp, gt, Hg[nl][s, cand], cand, m.W, cfg, run.n_u, rnd):
                stats["decode_checked"] += 1
            else:
                stats["decode_ties"] += 1
        # ---- the next step starts from the oracle's own free-running step
        for st in pre:
            O.denoise_step(st, m.W, cfg, run, t, taus if taus is not None else 0.0)
        states = pre
    if stats["seq_layers"]:
        assert stats["band"] <= 0.05 * stats["compared_rows"] + (2 * stats["seq_layers"] if select_mode == 1 else 0), stats
    assert stats["decode_checked"] >= stats["steps"] * b // 2, stats
    print(name, stats)
    return stats


@pytest.mark.parametrize("select_mode,policy,residual_mode,cmp", [
    (0, 1, 0, 0), (1, 1, 0, 0), (0, 0, 0, 0), (0, 1, 1, 0), (1, 1, 0, 1)])
def test_denoise_tiny(select_mode, policy, residual_mode, cmp):
    _denoise_parity("tiny", select_mode, policy, residual_mode, cmp)


# fraction mode (D19) is run with the carried-and-decoded policy only: under the literal policy the
# decoded rows never enter idx_in, every context barely moves, and the rank-k threshold falls inside
# a cluster of similarities within 1e-3 of each other (a vacuous comparison)
@pytest.mark.parametrize("select_mode,policy", [(0, 1), (1, 1), (0, 0)])
def test_denoise_small128(select_mode, policy):
    _denoise_parity("small128", select_mode, policy)


@pytest.mark.parametrize("select_mode,policy", [(1, 1), (0, 0)])
def test_denoise_small128_gqa(select_mode, policy):
    _denoise_parity("small128_gqa", select_mode, policy)


@pytest.mark.parametrize("select_mode,policy", [(0, 1), (1, 1)])
def test_denoise_head_dim_64(select_mode, policy):
    _denoise_parity("small64", select_mode, policy)


def test_denoise_paper_literal_block_and_le_rule():
    # no residual stream in this block: a softer attention keeps bf16 Q/K within the 2e-2 H bar
    _denoise_parity("small128", 1, 1, residual_mode=1, cmp=1, qk=0.07)


def test_denoise_dense_statistics():
    """The same loop with every tile's normaliser computed densely (no statistics refresh)."""
    _denoise_parity("small128", 0, 1, inc=False)


def test_denoise_empty_layer1_list_in_batch():
    """Fixed-tau mode, literal policy: sequence 1 enters a sparse step with an empty idx_in while
    sequence 0 does not (nothing recomputed for it, its caches stay)."""
    _denoise_parity("small128", 0, 0, empty_seq_at=6)


@pytest.mark.parametrize("select_mode", [0, 1])
def test_denoise_fused_similarity_partials(select_mode):
    """SURVEY §8f3 variant (DYLLM_OPT_ATTN_COS = 1): C_new, its commit and the cosine partials in the
    attention epilogue; the selection kernel only sums the partials over the heads."""
    from paper_2603_08026_b200 import dyllm as dy
    prev = dy.set_option(dy.OPT_ATTN_COS, 1)
    try:
        _denoise_parity("small128", select_mode, 1)
    finally:
        dy.set_option(dy.OPT_ATTN_COS, prev)


def test_denoise_two_kernel_attention_path():
    """head_dim 128 through the two-kernel attention of attn.cu (statistics, then P.V:
    DYLLM_OPT_ATTN_FUSED = 0), the path of every other head dim (dense Alg. 4, no incremental
    statistics)."""
    from paper_2603_08026_b200 import dyllm as dy
    prev = dy.set_option(dy.OPT_ATTN_FUSED, 0)
    try:
        _denoise_parity("small128", 1, 1)
    finally:
        dy.set_option(dy.OPT_ATTN_FUSED, prev)
