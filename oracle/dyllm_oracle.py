"""DyLLM CPU oracle — plain, slow, fp64 NumPy. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) may import this module; the CUDA product path never does.
It shares no code with paper_2603_08026_b200/ (only the seeded generators in
synth/ serve both).

Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
Dn = a reading listed in DESIGN.md §2 (and SURVEY.md §8c.2).

What it follows, step by step:
  Alg. 1  DyLLM generation loop ............ P:794-826   -> denoise_step / generate
  Alg. 2  FullStep ......................... P:834-852   -> full_layer / full_step
  Alg. 3  SparseStep ....................... P:866-904   -> sparse_layer
  Alg. 4  ApproximateAttention ............. P:917-934   -> approx_attention
  §3.1    temporal cosine similarity ....... P:259-261   -> cosine_rows
  §3.2    salient set (strict '<', D1) ..... P:269, P:891 -> select_salient
  §2.2    confidence-based unmasking ....... P:202-206   -> process_logit
  Eq. 3   delta decomposition .............. P:328-335   -> eq3_terms (self-check only)

Parity pins: every function here is pinned by tests/test_oracle_*.py against
closed forms, special cases, brute force, independent torch-fp64 routines or
the paper's printed cost example — see DESIGN.md §4. Accuracy/salient-fraction
statistics of the paper (Tables 1-2, Figs. 2/4/6) are "parity unpinned": they
need trained weights.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

MODE_FULL, MODE_FI, MODE_RO = "full", "fi", "ro"


# --------------------------------------------------------------------------- primitives

def rms_norm(x, g, eps):
    """RMSNorm (D3): y = x / sqrt(mean(x^2) + eps) * g, per row."""
    x = np.asarray(x, dtype=np.float64)
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * g


def rope(x, pos, theta, head_dim):
    """Rotate-half RoPE at GLOBAL positions (D10).

    Pair k of each head (x[k], x[k+hd/2]) is rotated by angle pos * theta^(-2k/hd).
    """
    x = np.asarray(x, dtype=np.float64)
    rows = x.shape[0]
    half = head_dim // 2
    nh = x.shape[1] // head_dim
    inv = theta ** (-(np.arange(half, dtype=np.float64) * 2.0) / head_dim)
    ang = np.asarray(pos, dtype=np.float64)[:, None] * inv[None, :]
    c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    xr = x.reshape(rows, nh, head_dim)
    x1, x2 = xr[..., :half], xr[..., half:]
    out = np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)
    return out.reshape(rows, nh * head_dim)


def softmax_rows(s):
    """Row softmax with max subtraction (Alg. 4 line 2)."""
    s = np.asarray(s, dtype=np.float64)
    if s.shape[-1] == 0:
        return s.copy()
    m = np.max(s, axis=-1, keepdims=True)
    e = np.exp(s - m)
    return e / np.sum(e, axis=-1, keepdims=True)


def silu(x):
    return x / (1.0 + np.exp(-x))


def _heads(x, nh, hd):
    return np.asarray(x, dtype=np.float64).reshape(x.shape[0], nh, hd).transpose(1, 0, 2)


def attention_probs(q, k, n_heads, n_kv_heads, head_dim):
    """A = softmax(Q K^T / sqrt(d_h)) per head, non-causal (Alg. 4 lines 1-2).

    GQA: query head h reads kv head h // (n_heads / n_kv_heads). Returns [H][Lq][N].
    """
    g = n_heads // n_kv_heads
    qh = _heads(q, n_heads, head_dim)
    kh = _heads(k, n_kv_heads, head_dim)
    kh = np.repeat(kh, g, axis=0)
    s = qh @ kh.transpose(0, 2, 1) / np.sqrt(head_dim)
    return softmax_rows(s)


def attention(q, k, v, n_heads, n_kv_heads, head_dim):
    """C = softmax(Q K^T / sqrt(d_h)) V, concatenated heads (Alg. 2 line 5; Alg. 3 line 8)."""
    lq = q.shape[0]
    if lq == 0:
        return np.zeros((0, n_heads * head_dim))
    g = n_heads // n_kv_heads
    a = attention_probs(q, k, n_heads, n_kv_heads, head_dim)
    vh = np.repeat(_heads(v, n_kv_heads, head_dim), g, axis=0)
    return (a @ vh).transpose(1, 0, 2).reshape(lq, n_heads * head_dim)


def approx_attention(q, k, dv, idx_cols, n_heads, n_kv_heads, head_dim):
    """Alg. 4 ApproximateAttention, literally:

    S = Q K^T ; A = Softmax(S) ; A_sal = A[:, idx_sal] ; dC = A_sal dV.
    `idx_cols` are key positions (0-based, into K's rows); dv has |idx_cols| rows.
    """
    lq = q.shape[0]
    qw = n_heads * head_dim
    if lq == 0:
        return np.zeros((0, qw))
    if len(idx_cols) == 0:
        return np.zeros((lq, qw))
    g = n_heads // n_kv_heads
    a = attention_probs(q, k, n_heads, n_kv_heads, head_dim)          # [H][L][N]
    a_sal = a[:, :, np.asarray(idx_cols)]                              # [H][L][m]
    dvh = np.repeat(_heads(dv, n_kv_heads, head_dim), g, axis=0)       # [H][m][hd]
    return (a_sal @ dvh).transpose(1, 0, 2).reshape(lq, qw)


def cosine_rows(a, b):
    """Temporal cosine similarity s = <C_t, C_{t-1}> / (|C_t| |C_{t-1}|) per row.

    Zero-norm policy (D9): both norms < 1e-12 -> 1; exactly one -> 0.
    Evaluated as dot / sqrt(|a|^2 |b|^2) (D9): for identical rows the three sums are the same
    numbers, and sqrt(fl(x*x)) == |x| in IEEE arithmetic, so s == 1 exactly.
    """
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    dot = np.sum(a * b, axis=-1)
    na2 = np.sum(a * a, axis=-1)
    nb2 = np.sum(b * b, axis=-1)
    out = np.empty(a.shape[0])
    for i in range(a.shape[0]):
        za, zb = na2[i] < 1e-24, nb2[i] < 1e-24
        if za and zb:
            out[i] = 1.0
        elif za or zb:
            out[i] = 0.0
        else:
            out[i] = dot[i] / np.sqrt(na2[i] * nb2[i])
    return out


def select_salient(s, tau, positions, cmp=0):
    """idx_sal = Where(CosSim(C, C_cache) < tau) (Alg. 3 line 12); cmp=1 gives '<=' (D1).

    Returns the global positions (ascending if `positions` is) of the selected rows.
    """
    s = np.asarray(s)
    sel = (s <= tau) if cmp else (s < tau)
    return np.asarray(positions, dtype=np.int64)[sel]


def ffn(x, w):
    """Gated SiLU FFN (D11): W_down( SiLU(x W_gate^T) * (x W_up^T) )."""
    return (silu(x @ w["w_gate"].T) * (x @ w["w_up"].T)) @ w["w_down"].T


def qkv(xn, w, cfg, pos):
    """Q/K/V projections with optional bias, RoPE on Q and K at global positions."""
    q = xn @ w["wq"].T
    k = xn @ w["wk"].T
    v = xn @ w["wv"].T
    if cfg.qkv_bias:
        q, k, v = q + w["bq"], k + w["bk"], v + w["bv"]
    return rope(q, pos, cfg.rope_theta, cfg.head_dim), rope(k, pos, cfg.rope_theta, cfg.head_dim), v


def post_attention(x, c, w, cfg):
    """Alg. 2/3 'x <- LN(OutProj(C)); x <- FFN(x)' under the residual reading D2.

    residual_mode 0 (LLaDA/Dream pre-norm block): h = x + C W_o ; out = h + FFN(RMSNorm(h)).
    residual_mode 1 (paper_literal):    h = RMSNorm(C W_o) ; out = FFN(h).
    Returns (h, out).
    """
    o = c @ w["wo"].T
    if cfg.residual_mode == 0:
        h = x + o
        return h, h + ffn(rms_norm(h, w["g_ffn"], cfg.rms_eps), w)
    h = rms_norm(o, w["g_ffn"], cfg.rms_eps)
    return h, ffn(h, w)


def lm_logits(h, wg, cfg):
    """logits = LMHead(RMSNorm_f(x)) (Alg. 2 line 10; D3)."""
    return rms_norm(h, wg["g_final"], cfg.rms_eps) @ wg["lm_head"].T


# --------------------------------------------------------------------------- layer steps

@dataclass
class LayerCache:
    """Per-layer activation caches: K, V, C, FFN_OUT(=H), plus the Q cache (D6)."""
    K: np.ndarray
    V: np.ndarray
    Q: np.ndarray
    C: np.ndarray
    H: np.ndarray

    def copy(self):
        return LayerCache(self.K.copy(), self.V.copy(), self.Q.copy(), self.C.copy(), self.H.copy())


def full_layer(x, w, cfg):
    """One layer of FullStep (Alg. 2 lines 3-8) over all N rows; returns its LayerCache."""
    n = x.shape[0]
    pos = np.arange(n)
    xn = rms_norm(x, w["g_attn"], cfg.rms_eps)
    q, k, v = qkv(xn, w, cfg, pos)
    c = attention(q, k, v, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim)
    _, out = post_attention(x, c, w, cfg)
    return LayerCache(K=k, V=v, Q=q, C=c, H=out)


@dataclass
class SparseLayerResult:
    idx_out: np.ndarray          # selected global positions (ascending)
    s: np.ndarray                # cosine similarity per input row
    C: np.ndarray                # new context rows for the input rows [L][qw]
    h: np.ndarray                # post-attention rows for idx_out [M_out][d]
    out: np.ndarray              # new H rows for idx_out [M_out][d]
    dV: np.ndarray               # V_new[idx_in] - V_cache[idx_in]


def quantile_threshold(s_all, frac):
    """Fraction-controlled threshold (DESIGN D19, the bench's stand-in for a calibrated tau):
    tau* = the (k+1)-th smallest similarity with k = round(frac * n), so that the strict rule
    s < tau* selects exactly the k least similar rows when there are no ties (+inf if k >= n)."""
    s_all = np.sort(np.asarray(s_all, dtype=np.float64).ravel())
    n = s_all.size
    k = int(np.floor(frac * n + 0.5))
    return np.inf if k >= n else float(s_all[k])


def sparse_layer(x_all, cache, w, cfg, idx_in, tau, input_rows, cmp=0, q_mode="literal",
                 q_extra=()):
    """One layer of SparseStep (Alg. 3 lines 3-17), in Alg. 3's order.

    x_all      : current H_{l-1} for all N positions (the layer input; only input rows are used)
    cache      : LayerCache of this layer; UPDATED IN PLACE
    idx_in     : salient positions produced by the previous layer (D4), subset of input_rows
    input_rows : global positions that form this step's input (all N, or the response)
    q_mode     : "literal" -> Q for all input rows;
                 "cache"   -> Q recomputed only for idx_in ∪ q_extra, rest from the Q cache (D6)
    tau        : a float, or a callable s -> tau (used by the fraction-controlled mode)
    """
    input_rows = np.asarray(input_rows, dtype=np.int64)
    idx_in = np.asarray(idx_in, dtype=np.int64)
    H, KVH, hd = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    x = x_all[input_rows]
    # line 3: x <- LayerNorm(x)
    xn_all = rms_norm(x_all, w["g_attn"], cfg.rms_eps)
    # line 4: Q <- QProj(x) for every input row
    if q_mode == "literal":
        q_in, _, _ = qkv(xn_all[input_rows], w, cfg, input_rows)
    else:
        q_in = cache.Q[input_rows].copy()
        rec = np.union1d(idx_in, np.asarray(q_extra, dtype=np.int64))
        if len(rec):
            qr, _, _ = qkv(xn_all[rec], w, cfg, rec)
            where = np.searchsorted(input_rows, rec)
            q_in[where] = qr
    # lines 5-6: K, V <- cache; K[idx], V[idx] <- KProj/VProj(x[idx])
    K = cache.K.copy()
    V = cache.V.copy()
    if len(idx_in):
        _, k_new, v_new = qkv(xn_all[idx_in], w, cfg, idx_in)
        K[idx_in] = k_new
        V[idx_in] = v_new
    # line 7: dV <- V[idx] - V_cache[idx]   (before the cache is overwritten)
    dV = V[idx_in] - cache.V[idx_in]
    # line 8: C_sal <- Attention(Q[idx], K, V)
    pos_in_input = np.searchsorted(input_rows, idx_in)
    c_sal = attention(q_in[pos_in_input], K, V, H, KVH, hd)
    # line 9: dC <- ApproxAttn(Q, K, dV)
    dC = approx_attention(q_in, K, dV, idx_in, H, KVH, hd)
    # lines 10-11: C <- C_cache + dC ; C[idx] <- C_sal
    C = cache.C[input_rows] + dC
    C[pos_in_input] = c_sal
    # line 12: idx <- Where(CosSim(C, C_cache) < tau)
    s = cosine_rows(C, cache.C[input_rows])
    if callable(tau):
        tau = tau(s)
    idx_out = select_salient(s, tau, input_rows, cmp)
    # lines 13-15: x <- LN(OutProj(C)); x[idx] <- FFN(x[idx]); x[~idx] <- FFN_OUT_cache[~idx]
    #  (D8: OutProj / FFN evaluated only on the rows whose result is used)
    sel = np.searchsorted(input_rows, idx_out)
    h, out = post_attention(x[sel], C[sel], w, cfg)
    # line 16: caches <- K, V, C, x   (rows outside idx_out keep FFN_OUT_cache: x[~idx] = cache)
    cache.K = K
    cache.V = V
    cache.C[input_rows] = C
    cache.Q[input_rows] = q_in
    cache.H[idx_out] = out
    return SparseLayerResult(idx_out=idx_out, s=s, C=C, h=h, out=out, dV=dV)


def eq3_terms(S_prev, S_new, V_prev, V_new):
    """Eq. 3: dC = (S + dS) dV + dS V_{t-1}; returns (lhs, rhs) for the identity check."""
    dS = S_new - S_prev
    dV = V_new - V_prev
    return S_new @ V_new - S_prev @ V_prev, (S_prev + dS) @ dV + dS @ V_prev


# --------------------------------------------------------------------------- unmasking

def active_block(tokens, cfg, run):
    """First semi-AR block (size B) of the response that still holds a mask token; None if done."""
    for k in range(run.L_R // run.block):
        lo = run.L_P + k * run.block
        if np.any(tokens[lo:lo + run.block] == cfg.mask_id):
            return k
    return None


def candidate_rows(tokens, cfg, run):
    """Masked positions of the active block (D13): the only rows whose logits are needed."""
    k = active_block(tokens, cfg, run)
    if k is None:
        return np.zeros(0, dtype=np.int64)
    lo = run.L_P + k * run.block
    blk = np.arange(lo, lo + run.block)
    return blk[tokens[blk] == cfg.mask_id]


def process_logit(cand_pos, logits, n_u, mask_id=None):
    """process_logit (Alg. 1 line 20; D13, D22).

    token = argmax over the vocabulary without the mask token (lowest id on ties; D22: unmasking
    commits a token, so [M] is never a prediction); confidence = that token's softmax probability
    over the whole vocabulary = 1 / sum(exp(z - z_token)); pick the min(n_u, |cand|) most confident
    positions, ties to the lowest position. Returns (positions, tokens, confidences) in selection order.
    """
    cand_pos = np.asarray(cand_pos, dtype=np.int64)
    if len(cand_pos) == 0:
        return cand_pos, np.zeros(0, dtype=np.int64), np.zeros(0)
    z = np.asarray(logits, dtype=np.float64)
    za = z.copy()
    if mask_id is not None:
        za[:, mask_id] = -np.inf
    tok = za.argmax(axis=1)
    m = za.max(axis=1)
    conf = 1.0 / np.exp(z - m[:, None]).sum(axis=1)
    order = sorted(range(len(cand_pos)), key=lambda i: (-conf[i], cand_pos[i]))[:n_u]
    order = np.asarray(order, dtype=np.int64)
    return cand_pos[order], tok[order], conf[order]


# --------------------------------------------------------------------------- generation (Alg. 1)

def step_mode(t, run):
    """Alg. 1 mode schedule: FullStep if t < T_full; full input if t % period == 0; else R only."""
    if t < run.T_full:
        return MODE_FULL
    return MODE_FI if t % run.full_period == 0 else MODE_RO


@dataclass
class SeqState:
    tokens: np.ndarray
    caches: list = field(default_factory=list)     # LayerCache per layer
    H0: np.ndarray = None
    idx_carried: np.ndarray = None                  # idx_sal across steps (None until first sparse step)
    decoded_prev: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int64))
    sal_counts: list = field(default_factory=list)  # per step: [n_layers] salient counts
    layer_results: list = field(default_factory=list)  # SparseLayerResult per layer of the last sparse step


def init_state(prompt, cfg, run):
    """R <- [mask] x L_R (Alg. 1 line 1)."""
    toks = np.concatenate([np.asarray(prompt, dtype=np.int64),
                           np.full(run.L_R, cfg.mask_id, dtype=np.int64)])
    return SeqState(tokens=toks)


def full_step(st, W, cfg):
    """FullStep (Alg. 2): rebuild every cache from the current tokens; returns H_L."""
    x = W["emb"][st.tokens]
    st.H0 = x.copy()
    st.caches = []
    for lw in W["layers"]:
        lc = full_layer(x, lw, cfg)
        st.caches.append(lc)
        x = lc.H
    return x


def layer1_idx(st, run, input_rows):
    """Layer-1 idx_in of a sparse step (Alg. 1 P:815-819 + D5)."""
    if st.idx_carried is None:                       # idx <- [L_P .. L_P+L_R)
        st.idx_carried = np.arange(run.L_P, run.N, dtype=np.int64)
    base = st.idx_carried
    if run.layer1_policy == 1:
        base = np.union1d(base, st.decoded_prev)
    return np.intersect1d(base, input_rows).astype(np.int64)


def sparse_step(st, W, cfg, run, mode, tau, q_mode="cache"):
    """SparseStep over all layers (Alg. 3); updates caches and idx_carried; returns H_L."""
    N = run.N
    input_rows = np.arange(N) if mode == MODE_FI else np.arange(run.L_P, N)
    idx = layer1_idx(st, run, input_rows)
    q_extra = ()
    if run.layer1_policy == 0 and len(st.decoded_prev):
        q_extra = np.intersect1d(st.decoded_prev, input_rows)     # D6 Q-only write under 'carried'
    st.H0 = W["emb"][st.tokens]                                     # Alg. 3 line 1
    x_all = st.H0
    counts = []
    st.layer_results = []
    taus = np.broadcast_to(np.asarray(tau, dtype=np.float64), (cfg.n_layers,))
    for l, lw in enumerate(W["layers"]):
        thr = taus[l]
        if getattr(run, "select_mode", 0) == 1:              # fraction-controlled (D19)
            thr = (lambda s, f=taus[l]: quantile_threshold(s, f))
        r = sparse_layer(x_all, st.caches[l], lw, cfg, idx, thr, input_rows, run.cmp,
                         q_mode=q_mode, q_extra=q_extra if l == 0 else ())
        idx = r.idx_out
        st.layer_results.append(r)
        counts.append(len(idx))
        x_all = st.caches[l].H
    st.idx_carried = idx                                              # P:819 / P:902
    st.sal_counts.append(counts)
    return x_all


def denoise_step(st, W, cfg, run, t, tau, q_mode="cache", force_full=False):
    """One iteration of Alg. 1's loop body. Returns (positions, tokens)."""
    mode = MODE_FULL if force_full else step_mode(t, run)
    if mode == MODE_FULL:
        HL = full_step(st, W, cfg)
    else:
        HL = sparse_step(st, W, cfg, run, mode, tau, q_mode=q_mode)
    cand = candidate_rows(st.tokens, cfg, run)
    logits = lm_logits(HL[cand], W, cfg) if len(cand) else np.zeros((0, cfg.vocab))
    pos, tok, _ = process_logit(cand, logits, run.n_u, cfg.mask_id)
    st.tokens[pos] = tok
    st.decoded_prev = np.sort(pos)
    return pos, tok


def generate(prompts, W, cfg, run, tau, q_mode="cache"):
    """Alg. 1 for a batch of independent sequences (D16). Returns (tokens [b][N], states)."""
    states = [init_state(p, cfg, run) for p in prompts]
    for st in states:
        for t in range(run.T_total):
            denoise_step(st, W, cfg, run, t, tau, q_mode=q_mode)
    return np.stack([s.tokens for s in states]), states


def generate_full(prompts, W, cfg, run):
    """Full-recompute comparison path: FullStep at every step, same unmasking."""
    states = [init_state(p, cfg, run) for p in prompts]
    for st in states:
        for t in range(run.T_total):
            denoise_step(st, W, cfg, run, t, None, force_full=True)
    return np.stack([s.tokens for s in states]), states


# --------------------------------------------------------------------------- paper arithmetic

def fastdllm_computed_tokens(L_P, L_R, B, n_u, dual):
    """§4.2.4 computed-tokens-per-step example: PrefixCache computes the active block
    plus everything after it; DualCache only the active block; each block costs B/n_u steps, and
    one full refresh over L_P+L_R tokens per block is amortised over those steps."""
    n_blocks = L_R // B
    steps_per_block = B // n_u
    total = 0.0
    for k in range(n_blocks):
        per_step = B if dual else (L_R - k * B)
        total += (steps_per_block - 1) * per_step + (L_P + L_R)
    return total / (n_blocks * steps_per_block)
