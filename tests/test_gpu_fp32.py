"""fp32-parity mode (dyllm_model_cfg.dtype = 1, DESIGN D12): the same ABI calls and the same step
structure as the bf16 product path, with fp32 storage and SIMT fp32 arithmetic (csrc/fp32.cu),
compared with the fp64 oracle at the north_star's fp32 bar: 1e-4 max row-relative error for
hidden states (and every cache row), salient sets bit-exact outside |s - tau| < 1e-3.

The protocol is the bf16 one (tests/test_gpu_denoise.py: resynchronised per step, teacher-forced
per layer) with the imported state rounded to fp32 instead of bf16."""
import numpy as np
import pytest
import torch

import oracle as O
from synth import gen
from gpu_helpers import Model, from_dev, row_rel_err
from test_gpu_denoise import TOL_F32, _denoise_parity

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["tiny", "small128", "small128_gqa", "small64"])
def test_fp32_full_step_caches(name):
    """FullStep (Alg. 2): K, V, Q, C, H of every row of every layer at 1e-4."""
    m = Model(name, dtype=1)
    run = m.run
    prompts = gen.prompt_tokens(11, run.batch, run.L_P, m.cfg.mask_id)
    states = [O.init_state(p, m.cfg, run) for p in prompts]
    for st in states:
        st.tokens[run.L_P + 3] = 17
        O.full_step(st, m.W, m.cfg)
    cache = m.new_cache()
    cache.init(torch.tensor(np.stack([st.tokens for st in states]), dtype=torch.int32).cuda())
    torch.cuda.synchronize()
    dy = m.dyllm
    assert cache.tensor(0, dy.H).dtype == torch.float32
    for l in range(m.cfg.n_layers):
        for which, f in [(dy.K, "K"), (dy.V, "V"), (dy.Q, "Q"), (dy.CTX, "C"), (dy.H, "H")]:
            got = from_dev(cache.export(l + 1 if which == dy.H else l, which))
            ref = np.stack([getattr(st.caches[l], f) for st in states])
            err = row_rel_err(got, ref).max()
            assert err < TOL_F32, (l, f, err)


@pytest.mark.parametrize("select_mode,policy,residual_mode,cmp", [
    (0, 1, 0, 0), (1, 1, 0, 0), (0, 0, 0, 0), (0, 1, 1, 0), (1, 1, 0, 1)])
def test_fp32_denoise_tiny(select_mode, policy, residual_mode, cmp):
    _denoise_parity("tiny", select_mode, policy, residual_mode, cmp, dtype=1)


@pytest.mark.parametrize("name,select_mode,policy", [
    ("small128", 0, 1), ("small128", 1, 1), ("small128", 0, 0), ("small128_gqa", 1, 1),
    ("small128_gqa", 0, 0), ("small64", 0, 1)])
def test_fp32_denoise_small(name, select_mode, policy):
    _denoise_parity(name, select_mode, policy, dtype=1)


def test_fp32_denoise_paper_literal():
    _denoise_parity("small128", 1, 1, residual_mode=1, cmp=1, qk=0.07, dtype=1)


def test_fp32_all_salient_equals_full_path():
    """tau = +inf and idx_in = every input row: the sparse layer reproduces the fp32
    FullStep of the same tokens (K, V, Q, C, H of every row)."""
    m = Model("small128", dtype=1)
    run, dy = m.run, m.dyllm
    N, b = run.N, run.batch
    prompts = gen.prompt_tokens(3, b, run.L_P, m.cfg.mask_id)
    toks = np.full((b, N), m.cfg.mask_id, np.int32)
    toks[:, : run.L_P] = prompts
    a = m.new_cache()
    a.init(torch.tensor(toks).cuda())
    toks[:, run.L_P + 5] = 42       # one decoded token
    t_dev = torch.tensor(toks).cuda()
    ref = m.new_cache()
    ref.init(t_dev)
    # layer by layer with every row salient: layer 0 input = the new embeddings
    a.tensor(0, dy.H).copy_(ref.tensor(0, dy.H))
    idx = torch.arange(b * N, dtype=torch.int32, device="cuda")
    off = torch.tensor([s * N for s in range(b + 1)], dtype=torch.int32, device="cuda")
    out = torch.zeros(b * N, dtype=torch.int32, device="cuda")
    oof = torch.zeros(b + 1, dtype=torch.int32, device="cuda")
    for l in range(m.cfg.n_layers):
        a.layer_step(l, dy.INPUT_FULL, idx, off, float("inf"), out, oof)
        torch.cuda.synchronize()
        assert int(oof[-1]) == b * N
        for which in (dy.K, dy.V, dy.Q, dy.CTX):
            err = row_rel_err(from_dev(a.export(l, which)), from_dev(ref.export(l, which))).max()
            assert err < 1e-5, (l, which, err)
        err = row_rel_err(from_dev(a.export(l + 1, dy.H)), from_dev(ref.export(l + 1, dy.H))).max()
        assert err < 1e-5, (l, err)
