"""GPU unit parity of individual kernels through the C ABI (pytest -m gpu)."""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dy():
    from paper_2603_08026_b200 import dyllm
    return dyllm


@pytest.fixture(scope="module")
def ctx(dy):
    return dy.Context(0)


# ------------------------------------------------------------------ tcgen05 GEMM
@pytest.mark.parametrize("M_cap,M,N,K", [
    (128, 128, 128, 64),        # one tile
    (300, 300, 384, 256),       # ragged M
    (1000, 613, 4096, 512),     # device M < capacity, BN=128 path
    (512, 77, 12288, 4096),     # weight-streaming shape, BN=256 path
    (2048, 2048, 1024, 1024),   # many tiles per CTA (persistent loop, TMEM double buffer)
    (64, 0, 256, 128),          # empty row set
])
def test_gemm_vs_torch(dy, ctx, M_cap, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M_cap + N + K)
    A = (torch.randn(M_cap, K, device="cuda", generator=g) * 0.5).bfloat16()
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
    D = torch.full((M_cap, N), 7.0, device="cuda").bfloat16()
    Md = torch.tensor([M], dtype=torch.int32, device="cuda")
    ctx.gemm_bf16(A, W, D, M_dev=Md)
    torch.cuda.synchronize()
    ref = A[:M].float() @ W.float().T
    got = D[:M].float()
    if M:
        err = ((got - ref).abs().amax(1) / ref.abs().amax(1).clamp_min(1e-30)).max().item()  # per row
        assert err < 1e-2, err
    assert torch.all(D[M:] == 7.0)            # rows beyond the device count untouched


@pytest.mark.parametrize("skinny", [1, 0])
@pytest.mark.parametrize("M_cap,M,N,K", [
    (512, 16, 256, 64),         # one activation MMA, one weight pair
    (512, 205, 4096, 4096),     # f = 5% row count
    (512, 410, 12288, 4096),    # two activation MMAs (256 + 160)
    (512, 512, 512, 12288),     # maximum skinny M, long K (dozens of split-K contributors per block)
    (512, 300, 4096, 12288),    # FFN-down shape: 16 weight blocks split over all SM pairs
    (512, 100, 24576, 4096),    # gate/up width, M <= 256 (double-buffered TMEM accumulator)
    (1024, 700, 1024, 256),     # M > 512: three activation chunks of <= 256 rows
    (2048, 1530, 4096, 4096),   # full-input O-proj row count: 6 chunks x 16 weight blocks, ragged last chunk
    (2048, 2048, 512, 12288),   # maximum skinny M, long K
    (4096, 2500, 512, 256),     # 10 activation chunks
    (17000, 16500, 256, 128),   # device M > 16384: skinny exits, standard kernel computes
])
def test_gemm_skinny_vs_torch(dy, ctx, skinny, M_cap, M, N, K):
    prev = dy.set_option(dy.OPT_SKINNY_GEMM, skinny)
    try:
        g = torch.Generator(device="cuda").manual_seed(M + N + K)
        A = (torch.randn(M_cap, K, device="cuda", generator=g) * 0.5).bfloat16()
        W = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
        R = torch.randn(M_cap, N, device="cuda", generator=g).bfloat16()
        B = torch.randn(N, device="cuda", generator=g).bfloat16()
        Md = torch.tensor([M], dtype=torch.int32, device="cuda")
        for resid in (None, R):
            D = torch.full((M_cap, N), 7.0, device="cuda").bfloat16()
            ctx.gemm_bf16(A, W, D, M_dev=Md, resid=resid, bias=B)
            torch.cuda.synchronize()
            ref = A[:M].float() @ W.float().T + B.float()
            if resid is not None:
                ref = ref + R[:M].float()
            err = ((D[:M].float() - ref).abs().amax(1) / ref.abs().amax(1).clamp_min(1e-30)).max().item()
            assert err < 1e-2, (resid is not None, err)
            assert torch.all(D[M:] == 7.0)
            # split-K partials are reduced in a fixed contributor order: bit-identical reruns
            D2 = torch.full((M_cap, N), 7.0, device="cuda").bfloat16()
            ctx.gemm_bf16(A, W, D2, M_dev=Md, resid=resid, bias=B)
            torch.cuda.synchronize()
            assert torch.equal(D, D2)
    finally:
        dy.set_option(dy.OPT_SKINNY_GEMM, prev)


@pytest.mark.parametrize("M,N,K", [(4608, 12288, 512), (15296, 512, 256)])
def test_gemm_host_known_rows(dy, ctx, M, N, K):
    """Host-known row counts (the FullStep's GEMMs, M up to 16384) on the CTA-pair kernel."""
    g = torch.Generator(device="cuda").manual_seed(M + N)
    A = (torch.randn(M, K, device="cuda", generator=g) * 0.5).bfloat16()
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
    D = torch.empty((M, N), device="cuda").bfloat16()
    ctx.gemm_bf16(A, W, D)
    torch.cuda.synchronize()
    ref = A.float() @ W.float().T
    err = ((D.float() - ref).abs().amax(1) / ref.abs().amax(1).clamp_min(1e-30)).max().item()
    assert err < 1e-2, err


@pytest.mark.parametrize("S", [1, 2, 3, 4, 16, 64])
@pytest.mark.parametrize("M,N,K", [(410, 4096, 4096), (100, 12288, 4096), (257, 512, 1024), (1530, 4096, 4096)])
def test_gemm_skinny_split_granularity(dy, ctx, S, M, N, K):
    """Every split-K granularity gives the same result (fixed-order fp32 reduction)."""
    prev = dy.set_option(dy.OPT_SKINNY_SPLIT, S)
    try:
        g = torch.Generator(device="cuda").manual_seed(S * 7 + M)
        cap = 2048
        A = (torch.randn(cap, K, device="cuda", generator=g) * 0.5).bfloat16()
        W = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
        R = torch.randn(cap, N, device="cuda", generator=g).bfloat16()
        Md = torch.tensor([M], dtype=torch.int32, device="cuda")
        D = torch.full((cap, N), 7.0, device="cuda").bfloat16()
        ctx.gemm_bf16(A, W, D, M_dev=Md, resid=R)
        torch.cuda.synchronize()
        ref = A[:M].float() @ W.float().T + R[:M].float()
        err = ((D[:M].float() - ref).abs().amax(1) / ref.abs().amax(1).clamp_min(1e-30)).max().item()
        assert err < 1e-2, err
        assert torch.all(D[M:] == 7.0)
    finally:
        dy.set_option(dy.OPT_SKINNY_SPLIT, prev)


def test_gemm_residual_and_bias(dy, ctx):
    M, N, K = 200, 256, 192
    A = torch.randn(M, K, device="cuda").bfloat16()
    W = (torch.randn(N, K, device="cuda") * 0.1).bfloat16()
    R = torch.randn(M, N, device="cuda").bfloat16()
    B = torch.randn(N, device="cuda").bfloat16()
    D = torch.empty(M, N, device="cuda").bfloat16()
    ctx.gemm_bf16(A, W, D, resid=R, bias=B)
    torch.cuda.synchronize()
    ref = A.float() @ W.float().T + R.float() + B.float()
    assert ((D.float() - ref).abs().max() / ref.abs().max()).item() < 1e-2


# ------------------------------------------------------------------ K1 cosine / threshold / compaction
@pytest.mark.parametrize("b,N,row_lo,width", [(1, 32, 16, 64), (2, 160, 96, 256), (3, 200, 0, 512),
                                              (16, 956, 700, 4096)])
def test_select_salient_vs_oracle(dy, ctx, b, N, row_lo, width):
    rng = np.random.default_rng(b * 1000 + N)
    old = rng.standard_normal((b, N, width))
    new = old + rng.standard_normal((b, N, width)) * rng.uniform(0.0, 1.5, (b, N, 1))
    new[:, row_lo::7] = old[:, row_lo::7]                     # identical rows -> s == 1 exactly
    new_d = torch.tensor(new, dtype=torch.float32).bfloat16().cuda()
    old_d = torch.tensor(old, dtype=torch.float32).bfloat16().cuda()
    new_q = new_d.double().cpu().numpy()
    old_q = old_d.double().cpu().numpy()
    cache = old_d.clone()
    pos = np.arange(row_lo, N)
    s_ref = np.concatenate([O.cosine_rows(new_q[s, row_lo:], old_q[s, row_lo:]) for s in range(b)])
    tau = float(np.median(s_ref))
    idx = torch.zeros(b * N, dtype=torch.int32, device="cuda")
    off = torch.zeros(b + 1, dtype=torch.int32, device="cuda")
    sim = torch.full((b * N,), -9.0, device="cuda")
    ctx.select_salient(new_d, cache, row_lo, tau, 0, idx, off, sim)
    torch.cuda.synchronize()
    offs = off.cpu().numpy()
    rows = idx.cpu().numpy()
    sim_h = sim.cpu().numpy().reshape(b, N)
    excluded = 0
    for s in range(b):
        s_o = O.cosine_rows(new_q[s, row_lo:], old_q[s, row_lo:])
        assert np.abs(sim_h[s, row_lo:] - s_o).max() < 1e-5
        assert np.all(sim_h[s, row_lo:][::7] == 1.0)          # D9: identical -> exactly 1
        ref = set(O.select_salient(s_o, tau, pos).tolist())
        got = set((rows[offs[s]:offs[s + 1]] - s * N).tolist())
        assert list(rows[offs[s]:offs[s + 1]]) == sorted(rows[offs[s]:offs[s + 1]])
        band = set(pos[np.abs(s_o - tau) < 1e-3].tolist())
        excluded += len(band)
        assert (got - band) == (ref - band)
    assert excluded < 0.05 * b * (N - row_lo) + 2
    # commit: C_cache <- C_new on the input rows, prompt rows untouched
    assert torch.equal(cache[:, row_lo:], new_d[:, row_lo:])
    assert torch.equal(cache[:, :row_lo], old_d[:, :row_lo])
    # threshold extremes
    for t, expect in ((2.0, N - row_lo), (-2.0, 0)):
        c2 = old_d.clone()
        ctx.select_salient(new_d, c2, row_lo, t, 0, idx, off)
        torch.cuda.synchronize()
        assert int(off[-1]) == b * expect


def test_select_salient_worked_example(dy, ctx):
    """s = [1.0, 0.9, 0.995], tau = 0.99 -> {offset + 1} (built from exact unit vectors)."""
    w = 64
    old = np.zeros((1, 3, w)); old[0, :, 0] = 1.0
    new = np.zeros((1, 3, w))
    for i, s in enumerate([1.0, 0.9, 0.995]):
        new[0, i, 0], new[0, i, 1] = s, np.sqrt(1 - s * s)
    # bf16-exact construction is not possible for 0.995; check with the similarity the kernel reports
    new_d = torch.tensor(new, dtype=torch.float32).bfloat16().cuda()
    old_d = torch.tensor(old, dtype=torch.float32).bfloat16().cuda()
    idx = torch.zeros(3, dtype=torch.int32, device="cuda")
    off = torch.zeros(2, dtype=torch.int32, device="cuda")
    ctx.select_salient(new_d, old_d.clone(), 0, 0.99, 0, idx, off)
    torch.cuda.synchronize()
    assert idx[: int(off[1])].tolist() == [1]
