"""Host-side tests of the tensor-parallel decomposition (include/dyllm.h dyllm_tp_*):
the head / FFN shards produced by shard_weights sum to the full layer (single process), and a
world-size-2 gloo run of one Alg. 3 sparse layer split into shards — per-shard Q/K/V, attention and
Alg. 4 on the shard's heads, all-reduced similarity partials, all-reduced O projection (rank 0 adds
the residual) and FFN — reproduces the oracle's sparse_layer (the same collectives the CUDA group
performs). The computation here is the oracle's own primitives (oracle/), fp64."""
import os
from dataclasses import replace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from synth import configs, gen
from paper_2603_08026_b200.dist import shard_weights


def _layer(name, residual_mode=0):
    cfg, run = configs.preset(name)
    cfg = replace(cfg, n_layers=1, residual_mode=residual_mode)
    return cfg, run, gen.model_weights(cfg, 7)


@pytest.mark.parametrize("name", ["small128", "small64", "small128_gqa"])
def test_shards_sum_to_the_full_layer(name):
    cfg, run, W = _layer(name)
    world = 2 if cfg.n_kv_heads % 2 == 0 else 1
    lw = W["layers"][0]
    rng = np.random.default_rng(0)
    C = rng.standard_normal((9, cfg.q_width))
    Cold = rng.standard_normal((9, cfg.q_width))
    xn = rng.standard_normal((9, cfg.d_model))
    o_full, f_full = C @ lw["wo"].T, O.ffn(xn, lw)
    o_sum, f_sum = np.zeros_like(o_full), np.zeros_like(f_full)
    part = np.zeros((9, 3))
    for g in range(world):
        lcfg, lW = shard_weights(cfg, W, world, g)
        sw = lW["layers"][0]
        q = slice(g * lcfg.q_width, (g + 1) * lcfg.q_width)
        o_sum += C[:, q] @ sw["wo"].T
        f_sum += O.ffn(xn, sw)
        part += np.stack([(C[:, q] * Cold[:, q]).sum(1), (C[:, q] ** 2).sum(1), (Cold[:, q] ** 2).sum(1)], 1)
    assert np.abs(o_sum - o_full).max() < 1e-12
    assert np.abs(f_sum - f_full).max() < 1e-12
    s = part[:, 0] / np.sqrt(part[:, 1] * part[:, 2])
    assert np.abs(s - O.cosine_rows(C, Cold)).max() < 1e-12


def test_shard_weights_rejects_indivisible_heads():
    cfg, _, W = _layer("small128_gqa")   # one kv head
    with pytest.raises(ValueError):
        shard_weights(cfg, W, 2, 0)


def _sparse_layer_tp(rank, world, cfg, W, x_all, cache, idx_in, tau, rows):
    """One Alg. 3 layer on shard `rank` (heads / FFN channels of shard_weights), with all-reduces."""
    lcfg, lW = shard_weights(cfg, W, world, rank)
    w = lW["layers"][0]
    hd = cfg.head_dim
    q = slice(rank * lcfg.q_width, (rank + 1) * lcfg.q_width)
    kv = slice(rank * lcfg.kv_width, (rank + 1) * lcfg.kv_width)
    lc = O.LayerCache(K=cache.K[:, kv].copy(), V=cache.V[:, kv].copy(), Q=cache.Q[:, q].copy(),
                      C=cache.C[:, q].copy(), H=cache.H.copy())
    xn = O.rms_norm(x_all, w["g_attn"], cfg.rms_eps)
    qn, kn, vn = O.qkv(xn[idx_in], w, lcfg, idx_in)
    K, V = lc.K.copy(), lc.V.copy()
    K[idx_in], V[idx_in] = kn, vn
    dV = V[idx_in] - lc.V[idx_in]
    Q = lc.Q.copy()
    Q[idx_in] = qn
    C = lc.C[rows] + O.approx_attention(Q[rows], K, dV, idx_in, lcfg.n_heads, lcfg.n_kv_heads, hd)
    pos = np.searchsorted(rows, idx_in)
    C[pos] = O.attention(Q[idx_in], K, V, lcfg.n_heads, lcfg.n_kv_heads, hd)
    part = torch.tensor(np.stack([(C * lc.C[rows]).sum(1), (C * C).sum(1), (lc.C[rows] ** 2).sum(1)], 1))
    dist.all_reduce(part)                                       # similarity partials over the shards
    p = part.numpy()
    s = p[:, 0] / np.sqrt(p[:, 1] * p[:, 2])
    idx_out = O.select_salient(s, tau, rows)
    sel = np.searchsorted(rows, idx_out)
    o = torch.tensor(C[sel] @ w["wo"].T)
    dist.all_reduce(o)                                          # O projection (row-parallel)
    if cfg.residual_mode == 0:
        h = x_all[idx_out] + o.numpy()
        f = torch.tensor(O.ffn(O.rms_norm(h, w["g_ffn"], cfg.rms_eps), w))
        dist.all_reduce(f)                                      # FFN down projection (row-parallel)
        out = h + f.numpy()
    else:
        h = O.rms_norm(o.numpy(), w["g_ffn"], cfg.rms_eps)
        f = torch.tensor(O.ffn(h, w))
        dist.all_reduce(f)
        out = f.numpy()
    return idx_out, s, C, out


def _tp_worker(rank, world, port, q, name, residual_mode, tau):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.set_num_threads(1)
    cfg, run, W = _layer(name, residual_mode)
    rng = np.random.default_rng(3)
    N = run.N
    x_all = rng.standard_normal((N, cfg.d_model))
    cache = O.full_layer(x_all, W["layers"][0], cfg)
    rows = np.arange(run.L_P, N)
    idx_in = np.sort(rng.choice(rows, 12, replace=False))
    x2 = x_all.copy()
    x2[idx_in] += rng.standard_normal((12, cfg.d_model))
    idx_out, s, C, out = _sparse_layer_tp(rank, world, cfg, W, x2, cache, idx_in, tau, rows)
    q.put((rank, idx_out.tolist(), s.tolist(), out.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,residual_mode", [("small128", 0), ("small64", 1)])
def test_two_rank_gloo_tp_layer_matches_the_oracle(name, residual_mode):
    cfg, run, W = _layer(name, residual_mode)
    rng = np.random.default_rng(3)
    N = run.N
    x_all = rng.standard_normal((N, cfg.d_model))
    cache = O.full_layer(x_all, W["layers"][0], cfg)
    rows = np.arange(run.L_P, N)
    idx_in = np.sort(rng.choice(rows, 12, replace=False))
    x2 = x_all.copy()
    x2[idx_in] += rng.standard_normal((12, cfg.d_model))
    s0 = O.sparse_layer(x2, cache.copy(), W["layers"][0], cfg, idx_in, 2.0, rows, q_mode="cache").s
    ss = np.sort(s0)
    tau = float(0.5 * (ss[len(ss) // 2 - 1] + ss[len(ss) // 2]))   # between two similarities: no tie
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 1000 + residual_mode
    ps = [ctx.Process(target=_tp_worker, args=(r, 2, port, q, name, residual_mode, tau)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    r = O.sparse_layer(x2, cache, W["layers"][0], cfg, idx_in, tau, rows, q_mode="cache")
    assert 0 < len(r.idx_out) < len(rows)
    for rank, idx_out, s, out in res:
        assert idx_out == r.idx_out.tolist()
        assert np.abs(np.array(s) - r.s).max() < 1e-12
        assert np.abs(np.array(out) - r.out).max() < 1e-10
