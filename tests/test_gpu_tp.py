"""Tensor parallelism over heads / FFN, on one GPU with the loopback backend
(SURVEY §4(ii)): the G shards of a group run one after another on the device and their partial
sums are added in shard order. The group must reproduce the TP = 1 path (and the oracle).

  - FullStep: every shard's K / V / Q / C caches are the head slices of the oracle's, its hidden
    states the oracle's (2e-2), bit-identical across shards;
  - denoising steps, resynchronised from the TP = 1 cache before each step: per layer the salient
    lists agree outside |s - tau| < 1e-3 (tau from the TP = 1 trace), the hidden rows both sides
    recomputed agree within 2e-2, the decoded tokens agree (the shards' H_L is bit-identical, so
    every shard decides the same), and the shards hold bit-identical hidden states.
"""
import numpy as np
import pytest
import torch

import oracle as O
from synth import gen
from gpu_helpers import Model, from_dev, row_rel_err

pytestmark = pytest.mark.gpu
TOL = 2e-2
BAND = 1e-3


def _group(m, world, run=None):
    dy = m.dyllm
    run = run or m.run
    tp = dy.TensorParallel(m.ctx, world)
    ws, caches = [], []
    for g in range(world):
        lcfg, lW = dy.shard_weights(m.cfg, m.W, world, g)
        w = dy.Weights.from_blob(m.ctx, lcfg, dy.blob_from_weights(lcfg, lW))
        c = dy.Cache(m.ctx, w, run)
        tp.attach(g, c)
        ws.append(w)
        caches.append(c)
    return tp, ws, caches


def _slices(cfg, world, g):
    hd = cfg.head_dim
    Hl, KVl = cfg.n_heads // world, cfg.n_kv_heads // world
    return slice(g * Hl * hd, (g + 1) * Hl * hd), slice(g * KVl * hd, (g + 1) * KVl * hd), slice(g * Hl, (g + 1) * Hl)


@pytest.mark.parametrize("name,residual_mode", [("small128", 0), ("small128", 1), ("small64", 0)])
def test_tp_full_step_matches_oracle(name, residual_mode):
    world = 2
    m = Model(name, residual_mode=residual_mode)
    cfg, run, dy = m.cfg, m.run, m.dyllm
    prompts = gen.prompt_tokens(11, run.batch, run.L_P, cfg.mask_id)
    states = [O.init_state(p, cfg, run) for p in prompts]
    for st in states:
        st.tokens[run.L_P + 3] = 17
        O.full_step(st, m.W, cfg)
    tp, ws, caches = _group(m, world)
    toks = torch.tensor(np.stack([st.tokens for st in states]), dtype=torch.int32).cuda()
    tp.init(ws, toks)
    torch.cuda.synchronize()
    for l in range(cfg.n_layers):
        Hs = [from_dev(c.export(l + 1, dy.H)) for c in caches]
        assert all(np.array_equal(Hs[0], h) for h in Hs[1:])          # replicated, bit-identical
        ref = np.stack([st.caches[l].H for st in states])
        assert row_rel_err(Hs[0], ref).max() < TOL, l
        for g, c in enumerate(caches):
            qs, kvs, _ = _slices(cfg, world, g)
            for which, f, sl in ((dy.K, "K", kvs), (dy.V, "V", kvs), (dy.Q, "Q", qs), (dy.CTX, "C", qs)):
                got = from_dev(c.export(l, which))
                want = np.stack([getattr(st.caches[l], f)[:, sl] for st in states])
                assert row_rel_err(got, want).max() < TOL, (l, g, f)


def _sync_group(m, src, caches, world, dec_pos):
    """Copy the TP = 1 cache state into the shards (head slices; hidden states whole)."""
    dy, cfg = m.dyllm, m.cfg
    for g, c in enumerate(caches):
        qs, kvs, hs = _slices(cfg, world, g)
        for l in range(cfg.n_layers):
            for which, sl in ((dy.K, kvs), (dy.V, kvs), (dy.Q, qs), (dy.CTX, qs)):
                c.import_(l, which, src.export(l, which)[:, :, sl])
            c.import_(l + 1, dy.H, src.export(l + 1, dy.H))
            if cfg.head_dim == 128:
                c.import_(l, dy.STATS, src.export(l, dy.STATS)[:, :, hs])
        c.import_(0, dy.H, src.export(0, dy.H))
        c.set_decoded(dec_pos)


@pytest.mark.parametrize("name,residual_mode", [("small128", 0), ("small128", 1), ("small64", 0)])
def test_tp_denoise_steps_match_tp1(name, residual_mode, select_mode=1):
    world = 2
    m = Model(name, qk_std=0.09, lm_std=0.25, select_mode=select_mode, residual_mode=residual_mode)
    cfg, run, dy = m.cfg, m.run, m.dyllm
    b, N, nl = run.batch, run.N, cfg.n_layers
    prompts = gen.prompt_tokens(23, b, run.L_P, cfg.mask_id)
    toks = torch.tensor(np.stack([np.concatenate([p, np.full(run.L_R, cfg.mask_id)]) for p in prompts]),
                        dtype=torch.int32).cuda()
    ref = m.new_cache()
    tp, ws, caches = _group(m, world)
    dec_pos = torch.full((b, run.n_u), -1, dtype=torch.int32, device="cuda")
    dec_tok = torch.full((b, run.n_u), -1, dtype=torch.int32, device="cuda")
    tau = np.full(nl, 0.2, np.float32)                 # salient fraction per layer (D19)
    for t in range(run.T_full):
        ref.denoise_step(t, tau, toks, dec_pos, dec_tok)
    tr_lists = torch.zeros(nl * b * N, dtype=torch.int32, device="cuda")
    tr_offs = torch.zeros(nl * (b + 1), dtype=torch.int32, device="cuda")
    tr_sims = torch.zeros(nl * b * N, dtype=torch.float32, device="cuda")
    ref.set_trace(tr_lists, tr_offs, tr_sims)
    tp_lists, tp_offs, tp_sims = torch.zeros_like(tr_lists), torch.zeros_like(tr_offs), torch.zeros_like(tr_sims)
    caches[0].set_trace(tp_lists, tp_offs, tp_sims)
    sal_tp = torch.zeros(nl * b, dtype=torch.int32, device="cuda")
    compared = band_n = 0
    for t in range(run.T_full, run.T_full + 6):
        for l in range(nl):                     # current statistics on both sides (D20, D21)
            ref.refresh_stats(l)
        _sync_group(m, ref, caches, world, dec_pos)
        if t > run.T_full:                      # carried list = the TP = 1 last layer's output
            lst = tr_lists.view(nl, b * N)[nl - 1].contiguous()
            off = tr_offs.view(nl, b + 1)[nl - 1].contiguous()
            for c in caches:
                c.set_carried(lst, off)
        toks_tp = toks.clone()
        dp_tp, dt_tp = dec_pos.clone(), dec_tok.clone()
        torch.cuda.synchronize()
        tp.denoise_step(ws, t, tau, toks_tp, dp_tp, dt_tp, sal_tp)
        ref.denoise_step(t, tau, toks, dec_pos, dec_tok)
        torch.cuda.synchronize()
        mode_fi = t % run.full_period == 0
        row_lo = 0 if mode_fi else run.L_P
        lists = tr_lists.view(nl, b * N).cpu().numpy()
        offs = tr_offs.view(nl, b + 1).cpu().numpy()
        sims = tr_sims.view(nl, b, N).cpu().numpy()
        HL_ref = [from_dev(ref.export(l + 1, dy.H)) for l in range(nl)]
        HL_tp = [[from_dev(c.export(l + 1, dy.H)) for c in caches] for l in range(nl)]
        sal = sal_tp.view(nl, b).cpu().numpy()
        tl = tp_lists.view(nl, b * N).cpu().numpy()
        to = tp_offs.view(nl, b + 1).cpu().numpy()
        ts = tp_sims.view(nl, b, N).cpu().numpy()
        for l in range(nl):
            assert all(np.array_equal(HL_tp[l][0], h) for h in HL_tp[l][1:])
            for s in range(b):
                got_ref = set((lists[l][offs[l][s]:offs[l][s + 1]] - s * N).tolist())
                got_tp = set((tl[l][to[l][s]:to[l][s + 1]] - s * N).tolist())
                assert len(got_tp) == int(sal[l, s])
                sv = sims[l, s, row_lo:]
                # the similarities the two sides threshold: equal up to the rounding of the paths
                # (bf16 hidden rows summed in another order; the paper_literal block has no residual
                # stream to damp it: the denoise parity tests' bars)
                ds = np.abs(ts[l, s, row_lo:] - sv).max()
                assert ds < (5e-3 if residual_mode == 0 else 2e-2), (t, l, s, ds)
                # the group's list is exactly its own rule on its own (all-reduced) similarities
                st = ts[l, s, row_lo:].astype(np.float64)
                thr_tp = O.quantile_threshold(st, tau[l]) if select_mode == 1 else tau[l]
                assert got_tp == set((np.flatnonzero(st < thr_tp) + row_lo).tolist()), (t, l, s)
                thr = O.quantile_threshold(sv, tau[l]) if select_mode == 1 else tau[l]
                # rows whose order against the threshold the measured difference can flip
                band = set((np.flatnonzero(np.abs(sv - thr) < max(BAND, 2 * ds)) + row_lo).tolist())
                band_n += len(band)
                assert got_tp - band == got_ref - band, (t, l, s, sorted(got_tp ^ got_ref))
                rows = np.array(sorted((got_ref & got_tp) - band), dtype=np.int64)
                if len(rows):
                    # two bf16 paths against each other (the oracle bar applies to each): 2x the bar
                    # for the block without a residual stream
                    tol = TOL if residual_mode == 0 else 2 * TOL
                    assert row_rel_err(HL_tp[l][0][s, rows], HL_ref[l][s, rows]).max() < tol, (t, l, s)
                compared += N - row_lo
        assert torch.equal(dp_tp, dec_pos) and torch.equal(dt_tp, dec_tok), t
        assert torch.equal(toks_tp, toks), t
    # most similarities lie within a few 1e-3 of each other at this state, so two bf16 paths may
    # order many of them differently against the threshold; the list comparison must still cover
    # a fifth of the rows (the group's own rule is checked on every row above)
    print(f"{name}: band {band_n} of {compared} rows")
    assert band_n <= 0.8 * compared


def test_tp_nccl_backend_single_rank_equals_plain_path():
    """The NCCL backend (dlopen'd libnccl, ncclCommInitRank, ncclAllReduce with the list length read
    back) with one rank: the group path — partial similarities, thresholding of the reduced sums,
    O / down projections into scratch, all-reduce, scatter-back — reproduces the plain single-GPU
    path bit for bit (a one-rank all-reduce is the identity)."""
    m = Model("small128", qk_std=0.09, lm_std=0.25, select_mode=1)
    cfg, run, dy = m.cfg, m.run, m.dyllm
    b, N, nl = run.batch, run.N, cfg.n_layers
    try:
        uid = dy.TensorParallel.unique_id()
    except dy.DyllmError as e:
        pytest.skip(f"NCCL unavailable: {e}")
    tp = dy.TensorParallel(m.ctx, 1, 0, uid)
    c_tp = m.new_cache()
    tp.attach(0, c_tp)
    c_ref = m.new_cache()
    prompts = gen.prompt_tokens(29, b, run.L_P, cfg.mask_id)
    toks = torch.tensor(np.stack([np.concatenate([p, np.full(run.L_R, cfg.mask_id)]) for p in prompts]),
                        dtype=torch.int32).cuda()
    toks_tp = toks.clone()
    dp, dt = (torch.full((b, run.n_u), -1, dtype=torch.int32, device="cuda") for _ in range(2))
    dp2, dt2 = dp.clone(), dt.clone()
    tau = np.full(nl, 0.25, np.float32)
    for t in range(run.T_full + 8):
        c_ref.denoise_step(t, tau, toks, dp, dt)
        tp.denoise_step([m.w], t, tau, toks_tp, dp2, dt2)
        torch.cuda.synchronize()
        assert torch.equal(toks, toks_tp), t
        for l in range(nl):
            assert torch.equal(c_ref.export(l + 1, dy.H), c_tp.export(l + 1, dy.H)), (t, l)
            assert torch.equal(c_ref.export(l, dy.CTX), c_tp.export(l, dy.CTX)), (t, l)
    tp.close()
