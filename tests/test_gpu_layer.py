"""GPU parity of FullStep and the teacher-forced per-layer SparseStep against the oracle
(north_star bars: salient sets bit-exact outside |s - tau| < 1e-3, hidden
states / contexts within 2e-2 max relative error per row in bf16)."""
import numpy as np
import pytest
import torch

import oracle as O
from synth import gen
from gpu_helpers import (Model, bf16_round, from_dev, import_states, oracle_states, pack_lists,
                               round_states, row_rel_err, to_dev_bf16, unpack_lists)

pytestmark = pytest.mark.gpu
TOL = 2e-2
S_TOL = 1e-2   # similarities: bf16 contexts, fp32 sums (overflow-fixup rows reach 5.2e-3)
BAND = 1e-3


@pytest.mark.parametrize("name", ["tiny", "small128", "small128_gqa"])
def test_full_step_caches_match_oracle(name):
    m = Model(name)
    run = m.run
    prompts = gen.prompt_tokens(11, run.batch, run.L_P, m.cfg.mask_id)
    states = [O.init_state(p, m.cfg, run) for p in prompts]
    for st in states:
        st.tokens[run.L_P + 3] = 17                       # a few decoded tokens
        O.full_step(st, m.W, m.cfg)
    cache = m.new_cache()
    toks = torch.tensor(np.stack([st.tokens for st in states]), dtype=torch.int32).cuda()
    cache.init(toks)
    torch.cuda.synchronize()
    dy = m.dyllm
    for l in range(m.cfg.n_layers):
        for which, f in [(dy.K, "K"), (dy.V, "V"), (dy.Q, "Q"), (dy.CTX, "C"), (dy.H, "H")]:
            got = from_dev(cache.tensor(l + 1 if which == dy.H else l, which))
            ref = np.stack([getattr(st.caches[l], f) for st in states])
            err = row_rel_err(got, ref).max()
            assert err < TOL, (l, f, err)


QK_STD = {"tiny": 0.18, "small128": 0.09, "small128_gqa": 0.09, "small64": 0.09}   # sharper attention


def _teacher_forced_layer(name, layer, mode, frac_in=0.4, seed=0, select_mode=0, frac=0.3, refresh=False,
                          dominate=False, overflow=False, tau_q=0.5, **over):
    """refresh: recompute the layer's softmax statistics on the GPU from the imported caches before
    the step, so that response tiles take the incremental path — as in every
    denoising step after the FullSteps. dominate: make one approximate row of sequence 0 attend
    (head 0) almost only to a salient key whose old value is overwritten, so its incremental
    normaliser cancels and its tile goes through the dense fixup launch. overflow: give one exact
    row of sequence 0 a key, in its second key tile, scoring ~88 nats above everything else, so that
    the single-pass softmax of exact rows hands its item to the two-pass fixup."""
    m = Model(name, seed=seed, qk_std=QK_STD[name], select_mode=select_mode, **over)
    cfg, run = m.cfg, m.run
    N = run.N
    prompts = gen.prompt_tokens(seed + 5, run.batch, run.L_P, cfg.mask_id)
    states = round_states(oracle_states(m, prompts, steps=max(run.T_full, 1)))
    rng = np.random.default_rng(seed + 99)
    row_lo = 0 if mode == "fi" else run.L_P
    input_rows = np.arange(row_lo, N)
    idx_lists = [np.sort(rng.choice(input_rows, max(1, int(frac_in * len(input_rows))), replace=False))
                 for _ in range(run.batch)]
    # the previous layer changed the idx_in rows: perturb H_{layer} there (same values to both sides)
    for st, idx in zip(states, idx_lists):
        x = st.H0 if layer == 0 else st.caches[layer - 1].H
        noise = rng.standard_normal((len(idx), cfg.d_model)) * 0.5 * np.abs(x[idx]).max(axis=1, keepdims=True)
        x[idx] = bf16_round(x[idx] + noise)
    if overflow:
        st, idx = states[0], idx_lists[0]
        r = int(idx[0])
        x_all = st.H0 if layer == 0 else st.caches[layer - 1].H
        xn = O.rms_norm(x_all, m.W["layers"][layer]["g_attn"], cfg.rms_eps)
        q_new = O.qkv(xn[[r]], m.W["layers"][layer], cfg, np.array([r]))[0][0]
        hd = cfg.head_dim
        j = next(q for q in range(N - 1, 127, -1) if q not in set(idx.tolist()))
        lc = st.caches[layer]
        lc.K[j, :hd] = bf16_round(q_new[:hd] * (1000.0 / float(q_new[:hd] @ q_new[:hd])))
    if dominate:
        st, idx = states[0], idx_lists[0]
        r = next(q for q in input_rows if q not in set(idx.tolist()))
        j, hd = int(idx[0]), cfg.head_dim
        lc = st.caches[layer]
        lc.K[j, :hd] = bf16_round(lc.Q[r, :hd] * (24.0 / max(np.linalg.norm(lc.Q[r, :hd]) ** 2, 1e-12)) * np.sqrt(hd))
    cache = m.new_cache()
    import_states(m, cache, states)
    if refresh:
        cache.refresh_stats(layer)
    h_before = from_dev(cache.tensor(layer + 1, m.dyllm.H))
    # oracle reference from the same (rounded) state
    refs = []
    for st, idx in zip(states, idx_lists):
        x_all = st.H0 if layer == 0 else st.caches[layer - 1].H
        lc = st.caches[layer].copy()
        r = O.sparse_layer(x_all, lc, m.W["layers"][layer], cfg, idx, np.inf, input_rows,
                           q_mode="cache")
        refs.append((r, lc))
    s_all = np.concatenate([r.s for r, _ in refs])
    tau = float(np.quantile(s_all, tau_q))
    # rerun the oracle with the chosen tau (tau only affects selection and the FFN rows);
    # in fraction mode every sequence thresholds at its own quantile (D19)
    first, refs, taus = refs, [], []
    for st, idx, (r0, _) in zip(states, idx_lists, first):
        x_all = st.H0 if layer == 0 else st.caches[layer - 1].H
        lc = st.caches[layer].copy()
        t_seq = O.quantile_threshold(r0.s, frac) if select_mode == 1 else tau
        r = O.sparse_layer(x_all, lc, m.W["layers"][layer], cfg, idx, t_seq, input_rows, q_mode="cache")
        refs.append((r, lc))
        taus.append(t_seq)
    idx_d, off_d = pack_lists(idx_lists, N)
    out_d = torch.zeros(run.batch * N, dtype=torch.int32, device="cuda")
    oof_d = torch.zeros(run.batch + 1, dtype=torch.int32, device="cuda")
    sim_d = torch.full((run.batch * N,), -9.0, device="cuda")
    cache.layer_step(layer, 0 if mode == "fi" else 1, idx_d, off_d, frac if select_mode == 1 else tau,
                     out_d, oof_d, sim_d)
    torch.cuda.synchronize()
    got_lists = unpack_lists(out_d, oof_d, N)
    sim = sim_d.cpu().numpy().reshape(run.batch, N)
    dy = m.dyllm
    C_gpu = from_dev(cache.tensor(layer, dy.CTX))
    H_gpu = from_dev(cache.tensor(layer + 1, dy.H))
    K_gpu = from_dev(cache.tensor(layer, dy.K))
    V_gpu = from_dev(cache.tensor(layer, dy.V))
    n_band = 0
    for s, ((r, lc), idx) in enumerate(zip(refs, idx_lists)):
        assert np.abs(sim[s, row_lo:] - r.s).max() < S_TOL
        band = set(input_rows[np.abs(r.s - taus[s]) < BAND].tolist())
        n_band += len(band)
        got, ref = set(got_lists[s].tolist()), set(r.idx_out.tolist())
        assert got - band == ref - band, (s, sorted(got ^ ref))
        # contexts of all input rows
        assert row_rel_err(C_gpu[s, row_lo:], r.C).max() < TOL
        # K/V rows of idx_in
        assert row_rel_err(K_gpu[s, idx], lc.K[idx]).max() < TOL
        assert row_rel_err(V_gpu[s, idx], lc.V[idx]).max() < TOL
        # hidden rows: recomputed for the agreed selection, bit-unchanged elsewhere
        agreed = sorted((got & ref))
        sel = np.searchsorted(r.idx_out, agreed)
        if len(agreed):
            assert row_rel_err(H_gpu[s, agreed], r.out[sel]).max() < TOL
        untouched = sorted(set(range(N)) - got)
        assert np.array_equal(H_gpu[s, untouched], h_before[s, untouched])
    # the excluded band must stay small, else the comparison is vacuous (in fraction mode tau* is
    # itself one of the similarities, so its row and a neighbour are always in the band)
    assert n_band <= 0.05 * run.batch * len(input_rows) + (2 * run.batch if select_mode == 1 else 1)
    return m


@pytest.mark.parametrize("name", ["tiny", "small128", "small128_gqa"])
@pytest.mark.parametrize("layer", [0, 1])
@pytest.mark.parametrize("mode", ["fi", "ro"])
def test_layer_step_teacher_forced(name, layer, mode):
    _teacher_forced_layer(name, layer, mode)


@pytest.mark.parametrize("name", ["small128", "small128_gqa"])
@pytest.mark.parametrize("mode", ["fi", "ro"])
@pytest.mark.parametrize("select_mode", [0, 1])
def test_layer_step_incremental_statistics(name, mode, select_mode):
    """Response tiles with current statistics: incremental normaliser == Alg. 4's dense one."""
    _teacher_forced_layer(name, 1, mode, select_mode=select_mode, refresh=True)


@pytest.mark.parametrize("name", ["small128", "small128_gqa"])
@pytest.mark.parametrize("mode", ["fi", "ro"])
@pytest.mark.parametrize("t4", [0, 32])
def test_layer_step_exact_rows_transposed_option(name, mode, t4):
    """Exact-row tiles of <= 32 rows: with a -DDYLLM_FA_T4=1 build they run transposed (type 4:
    S^T = K Q^T, O^T = V^T P^T) at DYLLM_OPT_ATTN_T4 = 32 and take the 128-row type-2 path at 0;
    the default build compiles type 4 out and both settings take type 2. Every form matches
    Alg. 3/4."""
    from paper_2603_08026_b200 import dyllm as dyl
    prev = dyl.set_option(dyl.OPT_ATTN_T4, t4)
    try:
        _teacher_forced_layer(name, 1, mode, refresh=True)
    finally:
        dyl.set_option(dyl.OPT_ATTN_T4, prev)


@pytest.mark.parametrize("mode", ["fi", "ro"])
def test_layer_step_single_pass_overflow_fixup(mode):
    """An exact row whose later key outscores its first key tile by ~2^127: two-pass fixup."""
    _teacher_forced_layer("small128", 1, mode, refresh=True, overflow=True)


@pytest.mark.parametrize("mode", ["fi", "ro"])
def test_layer_step_incremental_cancellation_fixup(mode):
    """A row whose attention sat on an overwritten key: its tile is recomputed densely."""
    _teacher_forced_layer("small128", 1, mode, refresh=True, dominate=True)


def test_incremental_statistics_match_dense_over_steps():
    """Denoising steps with incremental statistics vs the same steps with dense normalisers
    (DYLLM_OPT_ATTN_INC = 0), run in lockstep from the same prompts: the same decoded tokens and
    hidden states / contexts within the bf16 bar, step by step. Free-running bf16 trajectories may
    part at a near-tie of the unmasking rule; the comparison then stops, but only
    after at least 8 sparse steps agreed — two full-input and six response-only ones (the full-size
    test checks the statistics themselves over 64 steps without that caveat). With the FullStep's
    fused a2 + a3 (no bf16 QKV scratch) the two runs part at step 14, where they agreed over all 24
    steps with the unfused FullStep: the trajectory moved, not the statistics."""
    m = Model("small128", qk_std=QK_STD["small128"], select_mode=1)
    dy = m.dyllm
    run = m.run
    prompts = gen.prompt_tokens(21, run.batch, run.L_P, m.cfg.mask_id)
    sides = []
    for _ in range(2):
        toks = torch.tensor(np.stack([np.concatenate([p, np.full(run.L_R, m.cfg.mask_id)]) for p in prompts]),
                            dtype=torch.int32).cuda()
        dec_pos = torch.zeros(run.batch * run.n_u, dtype=torch.int32, device="cuda")
        sides.append((m.new_cache(), toks, dec_pos, torch.zeros_like(dec_pos)))
    tau = np.full(m.cfg.n_layers, 0.25, np.float32)   # salient fraction per layer (D19)
    prev = dy.set_option(dy.OPT_ATTN_INC, 1)
    agreed = 0
    try:
        for t in range(24):
            for inc, (cache, toks, dp, dt) in zip((1, 0), sides):
                dy.set_option(dy.OPT_ATTN_INC, inc)
                cache.denoise_step(t, tau, toks, dp, dt)
            torch.cuda.synchronize()
            (ca, ta, _, _), (cb, tb, _, _) = sides
            if not torch.equal(ta, tb):
                break
            assert row_rel_err(from_dev(ca.tensor(m.cfg.n_layers, dy.H)), from_dev(cb.tensor(m.cfg.n_layers, dy.H))).max() < TOL
            assert row_rel_err(from_dev(ca.tensor(1, dy.CTX)), from_dev(cb.tensor(1, dy.CTX))).max() < TOL
            agreed = t + 1
    finally:
        dy.set_option(dy.OPT_ATTN_INC, prev)
    assert agreed >= run.T_full + 8, agreed


@pytest.mark.parametrize("name", ["tiny", "small128_gqa"])
@pytest.mark.parametrize("mode", ["fi", "ro"])
@pytest.mark.parametrize("frac", [0.1, 0.5])
def test_layer_step_fraction_mode(name, mode, frac):
    _teacher_forced_layer(name, 1, mode, select_mode=1, frac=frac)


def test_layer_step_all_salient_equals_full(name="small128"):
    """tau > 1 and idx_in = all input rows -> the layer reproduces full recompute (GPU path)."""
    m = Model(name)
    cfg, run = m.cfg, m.run
    N = run.N
    prompts = gen.prompt_tokens(3, run.batch, run.L_P, cfg.mask_id)
    toks = np.stack([np.concatenate([p, np.full(run.L_R, cfg.mask_id)]) for p in prompts])
    cache = m.new_cache()
    cache.init(torch.tensor(toks, dtype=torch.int32).cuda())
    # change two tokens, refresh H0 rows, run all-salient layer steps, compare with a fresh full step
    toks2 = toks.copy()
    toks2[:, run.L_P + 1] = 5
    H0 = cache.tensor(0, m.dyllm.H)
    emb = to_dev_bf16(m.W["emb"])
    H0.copy_(emb[torch.tensor(toks2, dtype=torch.long).cuda()])
    idx, off = pack_lists([np.arange(N)] * run.batch, N)
    outs = [(torch.zeros_like(idx), torch.zeros_like(off)) for _ in range(cfg.n_layers)]
    cur = (idx, off)
    for l in range(cfg.n_layers):
        cache.layer_step(l, 0, cur[0], cur[1], 2.0, outs[l][0], outs[l][1])
        cur = outs[l]
    torch.cuda.synchronize()
    assert int(cur[1][-1]) == run.batch * N
    HL = from_dev(cache.tensor(cfg.n_layers, m.dyllm.H))
    ref = m.new_cache()
    ref.init(torch.tensor(toks2, dtype=torch.int32).cuda())
    torch.cuda.synchronize()
    HR = from_dev(ref.tensor(cfg.n_layers, m.dyllm.H))
    assert row_rel_err(HL, HR).max() < TOL


def test_layer_step_none_salient_keeps_hidden():
    m = Model("small128")
    cfg, run = m.cfg, m.run
    N = run.N
    prompts = gen.prompt_tokens(4, run.batch, run.L_P, cfg.mask_id)
    toks = np.stack([np.concatenate([p, np.full(run.L_R, cfg.mask_id)]) for p in prompts])
    cache = m.new_cache()
    cache.init(torch.tensor(toks, dtype=torch.int32).cuda())
    torch.cuda.synchronize()
    before = [cache.tensor(l + 1, m.dyllm.H).clone() for l in range(cfg.n_layers)]
    idx, off = pack_lists([np.arange(run.L_P, N)] * run.batch, N)
    o_idx, o_off = torch.zeros_like(idx), torch.zeros_like(off)
    for l in range(cfg.n_layers):
        cache.layer_step(l, 1, idx, off, -2.0, o_idx, o_off)
        torch.cuda.synchronize()
        assert int(o_off[-1]) == 0
        idx, off = o_idx.clone(), o_off.clone()
    for l in range(cfg.n_layers):
        assert torch.equal(cache.tensor(l + 1, m.dyllm.H), before[l])


@pytest.mark.parametrize("select_mode", [0, 1])
def test_layer_step_long_input(select_mode):
    """More than 1024 input rows per sequence (the paper's L_P = 1024 setting): the selection
    kernel's fraction mode streams the similarities from L2 instead of registers."""
    _teacher_forced_layer("small128", 1, "fi", select_mode=select_mode, frac=0.1, refresh=True, L_P=1100)


@pytest.mark.parametrize("mode", ["fi", "ro"])
@pytest.mark.parametrize("layer", [0, 1])
def test_layer_step_head_dim_64(mode, layer):
    """head_dim 64 (GQA 4/2): the tcgen05 statistics + mma.sync P.V attention of the other head
    dims. tau nearer 1 than the median (the paper's regime is tau = 0.99): at the full-input
    median (s ~ 0.83) the bf16 rounding of C_new alone moves s by ~1e-3, the width of the band;
    the quantiles keep the excluded band under 5% of the rows (checked on the oracle alone)."""
    _teacher_forced_layer("small64", layer, mode, tau_q={"fi": 0.95, "ro": 0.5}[mode])


@pytest.mark.parametrize("mode", ["fi", "ro"])
def test_layer_step_paper_literal_block(mode):
    """residual_mode 1 (paper_literal): h = RMSNorm(C W_o), out = FFN(h)."""
    _teacher_forced_layer("small128", 1, mode, residual_mode=1)


@pytest.mark.parametrize("name", ["small128", "small128_gqa"])
@pytest.mark.parametrize("mode", ["fi", "ro"])
def test_layer_step_qkv_unfused(name, mode):
    """a3 as its own kernel in every step kind (DYLLM_OPT_QKV_FUSED = 0: the projection writes a bf16
    QKV scratch, qkv_post applies bias / RoPE / dV / cache writes) against the oracle's Alg. 3 layer
    (by default full-input steps and FullSteps run a2 + a3 in the projection's epilogue)."""
    from paper_2603_08026_b200 import dyllm as dy
    prev = dy.set_option(dy.OPT_QKV_FUSED, 0)
    try:
        _teacher_forced_layer(name, 1, mode)
    finally:
        dy.set_option(dy.OPT_QKV_FUSED, prev)
