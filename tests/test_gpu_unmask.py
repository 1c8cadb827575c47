"""GPU parity of the unmasking rule (Alg. 1 lines 20-21, P:822-823, P:202-206;
D13) through the C ABI (dyllm_unmask): final RMSNorm + LM head on the masked rows of the active
semi-AR block, confidence = max softmax probability, argmax token, top n_u positions (ties to the
lowest position), commit into the token array and the embedding cache H_0.

Positions and tokens are integers decided by floating point (bf16 LM head with fp32 accumulation
on the GPU, fp64 in the oracle): they are compared exactly except where the oracle's decision
sits on a near-tie (the n_u-th / (n_u+1)-th confidences within 1e-3 relative, or the top two
logits within 2e-2), which is excluded and counted (it must stay rare)."""
import numpy as np
import pytest
import torch

import oracle as O
from synth import gen
from gpu_helpers import Model, from_dev

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_u", [1, 2, 4])
def test_unmask_matches_oracle(n_u):
    # lm_head std 0.2: logits of std ~3, so that confidences are spread (at std 0.02 they are all
    # ~1/vocab and every ranking would be a near-tie)
    m = Model("small128", w_std=0.2, n_u=n_u)
    cfg, run = m.cfg, m.run
    dy = m.dyllm
    b, N = run.batch, run.N
    rng = np.random.default_rng(7 + n_u)
    prompts = gen.prompt_tokens(13, b, run.L_P, cfg.mask_id)
    toks = np.full((b, N), cfg.mask_id, dtype=np.int32)
    toks[:, : run.L_P] = prompts
    # block 0 of the response partly decoded (a different number per sequence)
    for s in range(b):
        done = rng.choice(run.block, size=5 + 7 * s, replace=False)
        toks[s, run.L_P + done] = rng.integers(0, cfg.mask_id, size=len(done))
    HL = gen.cache_tensor(5, cfg.n_layers, "cH", b, N, cfg.d_model, 1.0)
    cache = m.new_cache()
    cache.tensor(cfg.n_layers, dy.H).copy_(torch.from_numpy(HL).to(torch.bfloat16))
    torch.cuda.synchronize()
    buf = torch.empty_like(cache.tensor(0, dy.H))     # mark initialised through the ABI import
    dy.lib().dyllm_cache_copy(m.ctx.h, cache.h, 0, dy.H, dy._ptr(buf), 1, 1)
    dy.lib().dyllm_cache_copy(m.ctx.h, cache.h, 0, dy.H, dy._ptr(buf), 1, 0)
    t_d = torch.tensor(toks, dtype=torch.int32).cuda()
    pos_d = torch.full((b * n_u,), -7, dtype=torch.int32, device="cuda")
    tok_d = torch.full((b * n_u,), -7, dtype=torch.int32, device="cuda")
    cache.unmask(t_d, pos_d, tok_d)
    torch.cuda.synchronize()
    t_gpu = t_d.cpu().numpy()
    pos_gpu = pos_d.cpu().numpy().reshape(b, n_u)
    tok_gpu = tok_d.cpu().numpy().reshape(b, n_u)
    H0 = from_dev(cache.tensor(0, dy.H))
    excluded = 0
    for s in range(b):
        cand = O.candidate_rows(toks[s], cfg, run)
        z = O.lm_logits(HL[s, cand].astype(np.float64), m.W, cfg)
        pos_ref, tok_ref, conf_ref = O.process_logit(cand, z, n_u, cfg.mask_id)
        k = len(pos_ref)
        zn = z.copy()
        zn[:, cfg.mask_id] = -np.inf                 # D22: [M] is never a prediction
        # ranking near-tie at the cut: the oracle's choice of positions is not decidable in bf16
        conf_all = np.sort(1.0 / np.exp(z - zn.max(axis=1, keepdims=True)).sum(axis=1))[::-1]
        cut_tie = k < len(cand) and abs(conf_all[k - 1] - conf_all[k]) <= 1e-3 * conf_all[k - 1]
        got_pos = pos_gpu[s][pos_gpu[s] >= 0] - s * N   # decoded row ids -> positions
        assert len(got_pos) == len(pos_ref)
        if cut_tie:
            excluded += 1
        else:
            assert sorted(got_pos.tolist()) == sorted(pos_ref.tolist()), (s, got_pos, pos_ref)
        for p, t in zip(pos_ref, tok_ref):
            zz = np.sort(zn[list(cand).index(p)])[::-1]
            if zz[0] - zz[1] <= 2e-2:
                excluded += 1
                continue
            if p in set(got_pos.tolist()):
                assert t_gpu[s, p] == t, (s, p, t_gpu[s, p], t)
                # the decoded row's embedding was committed into H_0
                assert np.array_equal(H0[s, p], gen.bf16_bits_to_f32(gen.f32_to_bf16_bits(
                    m.W["emb"][t].astype(np.float32))).astype(np.float64))
        # every other position is unchanged (prompt immutable, masks stay masks)
        keep = np.ones(N, dtype=bool)
        keep[list(got_pos)] = False
        assert np.array_equal(t_gpu[s, keep], toks[s, keep])
    assert excluded <= b * (n_u + 1) // 2


def test_mask_token_never_committed_on_gpu():
    """D22 on the GPU (LM-head epilogue leaves the mask column out of the max / argmax, keeps it in
    the normaliser): a model whose masked rows all score [M] highest still unmasks min(n_u,
    remaining) positions per step, never writes the mask id, and finishes the generation."""
    m = Model("tiny")
    cfg, run, dy = m.cfg, m.run, m.dyllm
    u = np.random.default_rng(0).standard_normal(cfg.d_model)
    u /= np.linalg.norm(u)
    W = dict(m.W)
    W["emb"], W["lm_head"] = m.W["emb"].copy(), m.W["lm_head"].copy()
    W["emb"][cfg.mask_id], W["lm_head"][cfg.mask_id] = 5.0 * u, 2.0 * u
    w = dy.Weights.from_blob(m.ctx, cfg, dy.blob_from_weights(cfg, W))
    eng = dy.Engine(m.ctx, w, run)
    prompts = torch.tensor(gen.prompt_tokens(2, run.batch, run.L_P, cfg.mask_id), dtype=torch.int32)
    eng.load_prompts(prompts.cuda())
    left = run.L_R
    for t in range(run.T_total):
        eng.cache.denoise_step(t, np.full(cfg.n_layers, 0.99, np.float32), eng.tokens, eng.dec_pos, eng.dec_tok)
        torch.cuda.synchronize()
        n_dec = int((eng.dec_pos >= 0).sum())
        assert n_dec == run.batch * min(run.n_u, left), t
        assert cfg.mask_id not in eng.dec_tok.cpu().numpy().ravel().tolist()
        left -= min(run.n_u, left)
    assert not bool((eng.tokens[:, run.L_P:] == cfg.mask_id).any())
