/*
 * dyllm.h — C ABI of libdyllm.so, the B200 (sm_100a) implementation of DyLLM's
 * salient-token denoising step (arxiv 2603.08026).
 *
 * Citations: P:n = PAPER.md line n (in /root/reference, not shipped), S:n = SPEC.md
 * line n, Dn = a reading in DESIGN.md §2.
 *
 * Conventions (apply to every call)
 *  - Status: 0 = DYLLM_OK, > 0 informational, < 0 error. Nothing throws across the ABI.
 *    dyllm_last_error() returns a thread-local message for the last failing call.
 *  - Handles (dyllm_ctx / dyllm_weights / dyllm_cache) are library-owned: create/destroy pairs.
 *  - `d_` pointers are caller-owned DEVICE memory on the ctx's device; `h_` pointers are host
 *    memory. Caller buffers must stay valid until the ctx stream has passed the call.
 *  - Every compute call is asynchronous on the ctx stream (no host synchronisation inside,
 *    row counts stay on the device), except the calls documented as synchronous.
 *  - Arguments are validated before anything is enqueued; a CUDA error is sticky and is
 *    reported (DYLLM_E_CUDA) by the next call on the ctx.
 *  - Row ids: a token row is identified by r = seq * N + pos with N = L_P + L_R and pos the
 *    0-based global position in the sequence. An index LIST is a packed array of
 *    row ids, ascending, grouped by sequence, plus offsets off[batch+1] (off[0] = 0,
 *    off[batch] = total count). Lists live on the device.
 *  - Tensors: bf16 row-major. K/V caches [batch][N][n_kv_heads*head_dim]; Q and C caches
 *    [batch][N][n_heads*head_dim]; hidden/FFN_OUT caches H_l [batch][N][d_model].
 */
#ifndef DYLLM_API_H_
#define DYLLM_API_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  DYLLM_OK = 0,
  DYLLM_DONE = 1,       /* no masked token left in any sequence */
  DYLLM_E_ARG = -1,     /* null / out-of-range argument */
  DYLLM_E_SHAPE = -2,   /* shape not supported by the kernels (see dyllm_model_cfg) */
  DYLLM_E_INDEX = -3,   /* layer / step / which out of range */
  DYLLM_E_STATE = -4,   /* cache not initialised, or wrong mode */
  DYLLM_E_CUDA = -5,    /* CUDA runtime / driver error (sticky) */
  DYLLM_E_NCCL = -6,    /* reserved: tensor-parallel collectives */
  DYLLM_E_NOMEM = -7    /* device allocation failed */
};

typedef struct dyllm_ctx dyllm_ctx;
typedef struct dyllm_weights dyllm_weights;
typedef struct dyllm_cache dyllm_cache;
typedef struct dyllm_tp dyllm_tp;

/* Model shape (LLaDA / Dream style transformer, BASELINE.json configs).
 * Constraints: d_model % 64 == 0, head_dim in {16, 32, 64, 128}, n_heads % n_kv_heads == 0,
 * d_ff % 128 == 0, rope on all head_dim dims (rotate-half, D10). dtype 0 (bf16, the product
 * path) or 1 (fp32-parity mode: fp32 caches / scratch / arithmetic, SIMT kernels, D12; a
 * correctness mode at the north_star's 1e-4 bar, not a throughput path; no incremental softmax
 * statistics, so DYLLM_STATS is unavailable). In fp32 mode every tensor the cache accessors hand
 * out (K, V, Q, C, H) is fp32 instead of bf16; weights stay bf16 in both modes. */
typedef struct {
  int32_t n_layers, d_model, n_heads, n_kv_heads, head_dim, d_ff, vocab, mask_id;
  float rope_theta, rms_eps;
  int32_t qkv_bias;      /* 1: Q/K/V projections carry a bias (Dream / Qwen2.5) */
  int32_t residual_mode; /* 0: pre-norm residual block (D2 primary); 1: paper_literal Alg. 2/3 */
  int32_t dtype;         /* 0: bf16 storage, fp32 accumulate; 1: fp32-parity mode (D12) */
} dyllm_model_cfg;

/* Generation shape and schedule (Alg. 1). */
typedef struct {
  int32_t batch, L_P, L_R;
  int32_t block;         /* semi-AR block size B; must divide L_R */
  int32_t n_u;           /* tokens unmasked per step per sequence; must divide block so
                            that T_total = L_R / n_u steps unmask every position */
  int32_t T_full;        /* warm-up FullSteps */
  int32_t full_period;   /* sparse step takes Concat(P,R) when t % full_period == 0 */
  int32_t layer1_policy; /* 0: carried (Alg. 1 literal); 1: carried ∪ decoded (D5, default) */
  int32_t cmp;           /* 0: s < tau (Alg. 3, D1); 1: s <= tau (§3.2) */
  int32_t select_mode;   /* 0: fixed threshold, the `tau` arguments are tau (the paper's rule);
                            1: fraction-controlled (D19), the `tau` arguments are fractions f in [0,1]
                               and every layer of every sequence thresholds at its own f-quantile of s
                               (tau* = similarity of rank round(f*L), strict '<') */
} dyllm_run_cfg;

/* input_mode of dyllm_layer_step / dyllm_select_salient */
enum { DYLLM_INPUT_FULL = 0 /* Concat(P,R): rows [0,N) */, DYLLM_INPUT_RESPONSE = 1 /* R: rows [L_P,N) */ };

/* `which` of dyllm_cache_tensor / dyllm_cache_copy. DYLLM_STATS (head_dim 128 only): the per-(row,
 * head) softmax statistics of the fused attention, float2 (m, l) [batch][N][n_heads] with
 * m = row max of the scores in the exp2 domain (s * log2(e) / sqrt(head_dim)) and l = sum of
 * 2^(score - m) over all N keys, i.e. log2 of Alg. 4's softmax normaliser is m + log2(l). */
enum { DYLLM_K = 0, DYLLM_V = 1, DYLLM_Q = 2, DYLLM_C = 3, DYLLM_H = 4, DYLLM_STATS = 5 };

/* ------------------------------------------------------------------ context */
const char *dyllm_last_error(void);
int dyllm_version(void);                 /* returns an integer version, e.g. 100 */

/* Create a context on `device`; `cuda_stream` is a cudaStream_t every call of the ctx launches on
 * (NULL = a new non-blocking stream owned by the ctx; pass cudaStreamLegacy, 0x1, for the legacy
 * default stream). Synchronous. */
int dyllm_ctx_create(int device, void *cuda_stream, dyllm_ctx **out);
int dyllm_ctx_sync(dyllm_ctx *ctx);      /* synchronous: waits for the ctx stream */
void dyllm_ctx_destroy(dyllm_ctx *ctx);

/* ------------------------------------------------------------------ weights (DS10) */
/* Number of bf16 elements of the host blob expected by dyllm_weights_load for `cfg`. Blob order
 * (all bf16, torch-Linear layout W[out][in]): emb[V][d], g_final[d], lm_head[V][d], then for each
 * layer: g_attn[d], wq[H*hd][d], wk[KVH*hd][d], wv[KVH*hd][d], (bq, bk, bv if qkv_bias),
 * wo[d][H*hd], g_ffn[d], w_gate[F][d], w_up[F][d], w_down[d][F]. */
int64_t dyllm_weights_blob_elems(const dyllm_model_cfg *cfg);
/* Upload a host blob (uint16 bf16 bit patterns, `n_elems` long). Synchronous. */
int dyllm_weights_load(dyllm_ctx *ctx, const dyllm_model_cfg *cfg, const uint16_t *h_blob,
                       int64_t n_elems, dyllm_weights **out);
/* On-device counter-based init (IH4 generator) with the same values
 * synth/gen.py produces for (seed, std): projections/embedding/lm-head ~ IH4(std), gains = 1,
 * biases ~ IH4(std). Synchronous. */
int dyllm_weights_init_random(dyllm_ctx *ctx, const dyllm_model_cfg *cfg, uint64_t seed, double std,
                              dyllm_weights **out);
void dyllm_weights_destroy(dyllm_weights *w);

/* ------------------------------------------------------------------ caches (DS1-DS5) */
/* Allocate the per-layer K/V/Q/C/H caches, H_0 and all scratch for `run`. Synchronous. */
int dyllm_cache_create(dyllm_ctx *ctx, const dyllm_weights *w, const dyllm_run_cfg *run,
                       dyllm_cache **out);
void dyllm_cache_destroy(dyllm_cache *c);

/* dyllm_cache_init = FullStep (Alg. 2) on d_tokens[batch][N] (int32): embeds all
 * rows into H_0 and writes K, V, Q, C, H for every layer and row. Also resets the salient-set
 * state (idx_sal = None, Alg. 1). Asynchronous. */
int dyllm_cache_init(dyllm_ctx *ctx, const dyllm_weights *w, dyllm_cache *c, const int32_t *d_tokens);

/* One layer of SparseStep (Alg. 3 lines 3-16) on layer `layer` (0-based):
 *   input  : hidden H_{layer} (H_0 = embeddings) and caches of `layer` inside `c`;
 *            salient list idx_in (d_idx_in, d_off_in[batch+1]) = previous layer's selection (D4),
 *            every entry must be an input row of `input_mode`;
 *            tau = cosine threshold (tau > 1: all salient, tau < -1: none).
 *   output : H_{layer+1} updated in place for the selected rows (other rows keep FFN_OUT_cache,
 *            P:896); K/V/Q rows of idx_in and C rows of all input rows updated;
 *            selected list written to d_idx_out / d_off_out (capacity batch*N / batch+1);
 *            d_sim_out (nullable) receives s per input row at index r (float[batch*N]).
 * Asynchronous; counts stay on the device. */
int dyllm_layer_step(dyllm_ctx *ctx, const dyllm_weights *w, dyllm_cache *c, int layer, int input_mode,
                     const int32_t *d_idx_in, const int32_t *d_off_in, float tau,
                     int32_t *d_idx_out, int32_t *d_off_out, float *d_sim_out);

/* One iteration of Alg. 1's loop body at step t:
 *   t < T_full -> FullStep; else SparseStep over all layers with input Concat(P,R) when
 *   t % full_period == 0, else R only; idx_sal initialised to the response rows on the first
 *   sparse step; layer-1 idx_in per layer1_policy (D5).
 *   Then logits for the masked rows of the active semi-AR block, confidence = max softmax
 *   probability, argmax token; per sequence the n_u most confident positions (ties: lowest
 *   position; argmax ties: lowest id; D13) are committed into d_tokens.
 *   h_tau[n_layers] : host array of per-layer thresholds (D17; all equal = the paper's setting)
 *   d_tokens        : [batch][N] int32, in/out
 *   d_dec_pos/tok   : [batch][n_u] int32 out: decoded row ids (-1 if none) and token ids
 *   d_sal_counts    : nullable [n_layers][batch] int32 out: |idx_sal| per layer and sequence
 * Asynchronous. Returns DYLLM_DONE without work once t >= T_total. */
int dyllm_denoise_step(dyllm_ctx *ctx, const dyllm_weights *w, dyllm_cache *c, int t,
                       const float *h_tau, int32_t *d_tokens, int32_t *d_dec_pos, int32_t *d_dec_tok,
                       int32_t *d_sal_counts);

/* Full-recompute comparison path: FullStep (all caches rewritten) + the same unmasking rule.
 * Asynchronous. */
int dyllm_full_step(dyllm_ctx *ctx, const dyllm_weights *w, dyllm_cache *c, int32_t *d_tokens,
                    int32_t *d_dec_pos, int32_t *d_dec_tok);

/* process_logit + commit alone (Alg. 1 lines 20-21) on the current last-layer hidden
 * states: the unmasking rule of dyllm_denoise_step without the layer stack. Asynchronous. */
int dyllm_unmask(dyllm_ctx *ctx, const dyllm_weights *w, dyllm_cache *c, int32_t *d_tokens, int32_t *d_dec_pos,
                 int32_t *d_dec_tok);

/* Device pointer to one cache tensor of one layer (layer in [0,n_layers); which = DYLLM_K..STATS;
 * for DYLLM_H, layer in [0, n_layers] where H_0 = embeddings). Synchronous, no copy. Handing out
 * K, Q or STATS (writable views) invalidates the layer's incremental attention statistics (see
 * dyllm_cache_refresh_stats). DYLLM_E_STATE for STATS when the head_dim keeps none. */
int dyllm_cache_tensor(const dyllm_cache *c, int layer, int which, void **d_ptr, int64_t *n_elems);
/* Copy a cache tensor to (export=1) or from (export=0) `ptr`; `ptr_on_device` = 1 if ptr is
 * device memory (bf16 tensors: 2 B per element, STATS: 8 B). Asynchronous on the ctx stream.
 * Test / teacher-forcing hook. An export leaves the statistics valid; importing K or
 * Q invalidates them; importing STATS marks them current (the caller asserts they belong to the
 * layer's K and Q). */
int dyllm_cache_copy(dyllm_ctx *ctx, dyllm_cache *c, int layer, int which, void *ptr,
                     int ptr_on_device, int export_);
/* Recompute, densely, the per-(row, head) softmax statistics (row max, sum of exps) of one layer
 * from its current Q and K caches. The head_dim-128 attention keeps them to update response rows
 * incrementally (only the salient keys changed, so the normaliser is updated by their
 * old and new terms instead of a pass over all N keys); they are written by every FullStep and
 * denoising step and invalidated whenever dyllm_cache_tensor hands out K or Q of the layer (the
 * next step then runs that layer densely). Test hook after writing caches from outside.
 * Asynchronous. Returns DYLLM_OK without work for other head dims. */
int dyllm_cache_refresh_stats(dyllm_ctx *ctx, dyllm_cache *c, int layer);
/* Set the carried salient list (idx_sal between steps) — test hook; NULL resets to None. */
int dyllm_cache_set_carried(dyllm_ctx *ctx, dyllm_cache *c, const int32_t *d_idx, const int32_t *d_off);

/* Set the rows decoded at the previous step (Alg. 1 line 21; their embeddings changed and
 * they enter layer-1 idx_in under layer1_policy 1, D5, or get a Q-only refresh under policy 0) —
 * test hook for resynchronised multi-step parity. d_dec = [batch][n_u] row ids
 * (-1 = none), device memory; NULL = no decoded rows. Asynchronous. */
int dyllm_cache_set_decoded(dyllm_ctx *ctx, dyllm_cache *c, const int32_t *d_dec);
/* Per-layer trace of dyllm_denoise_step's sparse steps (parity and paper-analysis hook, SURVEY
 * §8c.4 / §8f4): when d_lists != NULL, layer l's selected list idx_out (row ids) is copied to
 * d_lists + l*batch*N and its offsets to d_offs + l*(batch+1); when d_sims != NULL, s of every
 * input row r of layer l is written to d_sims[l*batch*N + r]. Caller-owned device buffers that
 * must outlive the traced steps; NULLs disable. d_lists and d_offs are both set or both NULL. */
int dyllm_cache_set_trace(dyllm_ctx *ctx, dyllm_cache *c, int32_t *d_lists, int32_t *d_offs, float *d_sims);

/* ------------------------------------------------------------------ kernel-level calls */
/* K1: temporal cosine similarity of C_new vs C_cache for the input rows of every
 * sequence, threshold (strict '<' unless cmp=1), stream compaction into a packed list,
 * and commit C_cache <- C_new for those rows.
 *   d_c_new, d_c_cache : [batch][N][width] bf16 (width % 8 == 0)
 *   row_lo             : first input position (0 for full input, L_P for response-only)
 * Outputs as in dyllm_layer_step. Asynchronous. */
int dyllm_select_salient(dyllm_ctx *ctx, int batch, int N, int row_lo, int width, const void *d_c_new,
                         void *d_c_cache, float tau, int cmp, int32_t *d_idx_out, int32_t *d_off_out,
                         float *d_sim_out);

/* Plain bf16 tcgen05 GEMM, D[M][N] = A[M][K] · W[N][K]^T (+ resid[M][N]) (+ bias[N]), fp32
 * accumulate, bf16 out. M = *d_M if d_M != NULL (device-resident count, M <= M_cap) else M_cap.
 * K % 64 == 0, N % 8 == 0. Asynchronous. */
int dyllm_gemm_bf16(dyllm_ctx *ctx, const int32_t *d_M, int M_cap, int N, int K, const void *d_A,
                    const void *d_W, void *d_D, const void *d_resid, const void *d_bias);

/* ------------------------------------------------------------------ tensor parallelism */
/* Megatron-style tensor parallelism over attention heads and FFN channels. Shard g of a group of
 * `world` holds heads [g*H/world, (g+1)*H/world) (query and kv heads, so n_heads and n_kv_heads must
 * both divide by world) and FFN channels [g*F/world, ...): its weights are a dyllm_weights built
 * for the LOCAL model cfg (n_heads/world, n_kv_heads/world, d_ff/world; wq/wk/wv/bias rows and wo
 * columns of its heads, gate/up rows and down columns of its channels; embeddings, gains and the
 * LM head whole), its K/V/Q/C caches hold its heads, and hidden states H_l are replicated. Per
 * sparse layer three all-reduces (sums over the shards in shard order): the per-row similarity
 * partials (<C_new, C_old>, |C_new|^2, |C_old|^2 over the shard's heads; every shard thresholds the
 * same sums, so the salient lists agree), the O projection (shard 0 adds the residual)
 * and the FFN down projection (shard 0 adds h), whose rows are then scattered into H_l.
 * Two backends:
 *  - loopback (nccl_unique_id == NULL): the group's `world` shards live in THIS process on the
 *    ctx's device and run one after another; the all-reduce is one kernel over the shards'
 *    buffers (row counts read on the device, no host synchronisation). This is the one-device
 *    test harness of the TP math.
 *  - NCCL (one process per GPU, `rank` of `world`): ncclAllReduce on the ctx stream; the row count
 *    of a device-side list is read back before each hidden-state all-reduce (one synchronisation
 *    per collective). NCCL is loaded at run time (dlopen "libnccl.so.2"); DYLLM_E_NCCL if absent.
 * bf16 (dtype 0) only. */
int dyllm_tp_unique_id(void *h_out, int n_bytes);  /* NCCL unique id (n_bytes >= 128); synchronous */
int dyllm_tp_create(dyllm_ctx *ctx, int world, int rank, const void *nccl_unique_id, dyllm_tp **out);
/* Register cache `c` (created from shard `shard`'s weights) as that shard (loopback: every shard
 * in [0, world); NCCL: shard == rank). Shapes are checked against the group. */
int dyllm_tp_attach(dyllm_tp *tp, int shard, dyllm_cache *c);
/* FullStep (Alg. 2) on every local shard; w[i] = weights of the i-th attached local shard. */
int dyllm_tp_cache_init(dyllm_tp *tp, const dyllm_weights *const *w, const int32_t *d_tokens);
/* dyllm_denoise_step over the group (same arguments; d_sal_counts nullable). Loopback: the
 * caller's d_tokens / d_dec_pos / d_dec_tok belong to shard 0; the other shards decide on private
 * copies of the same tokens (identical decisions: H_L is bit-identical on every shard). */
int dyllm_tp_denoise_step(dyllm_tp *tp, const dyllm_weights *const *w, int t, const float *h_tau,
                          int32_t *d_tokens, int32_t *d_dec_pos, int32_t *d_dec_tok, int32_t *d_sal_counts);
void dyllm_tp_destroy(dyllm_tp *tp);

/* ------------------------------------------------------------------ instrumentation */
/* Kernel classes timed by the profiler (CUDA events on the ctx stream around each launch). */
enum {
  DYLLM_KC_QKV_GEMM = 0, DYLLM_KC_QKV_POST = 1, DYLLM_KC_ATTN = 2, DYLLM_KC_SELECT = 3, DYLLM_KC_O_GEMM = 4,
  DYLLM_KC_GU_GEMM = 5, DYLLM_KC_DOWN_GEMM = 6, DYLLM_KC_GATHER = 7, DYLLM_KC_SCATTER = 8, DYLLM_KC_LM_GEMM = 9,
  DYLLM_KC_OTHER = 10, DYLLM_KC_COUNT = 11,
  DYLLM_KC_FULL = 16 /* added to the class of launches made by a FullStep */
};
/* enable = 1: record one event pair per launch from now on (clears previous records); 0: stop. */
int dyllm_ctx_profile(dyllm_ctx *ctx, int enable);
/* Synchronous: per-launch durations (ms, launch order) of class `kclass`; returns the number of
 * records (writes at most max_n). */
int dyllm_ctx_profile_read(dyllm_ctx *ctx, int kclass, float *h_ms, int max_n);
/* Process-wide number of kernels libdyllm has launched so far. */
uint64_t dyllm_launch_count(void);

/* Process-wide kernel-path options (A/B testing and parity of alternative kernels).
 * DYLLM_OPT_SKINNY_GEMM (default 1): route GEMMs whose device row count is <= 512 to the 2-CTA
 * weight-stationary kernel; 0 = always the 1-CTA kernel. Returns the previous value. */
/* DYLLM_OPT_SKINNY_SPLIT (default 0 = auto): split-K granularity of the skinny kernel, in units
 * per 256-row weight block (clamped to a divisor of K/64); results are identical for every value
 * up to fp32 summation order. */
/* DYLLM_OPT_ATTN_FUSED (default 1): head_dim 128 uses the fused tcgen05 attention kernel
 * (attn_fused.cu); 0 = the two-kernel path (tcgen05 row statistics + mma.sync P.V). */
/* DYLLM_OPT_SKINNY_ONE_CHUNK (default 0 = automatic): largest device row count the skinny kernel
 * keeps in a single activation chunk (above it: chunks of <= 256 rows). */
/* DYLLM_OPT_PDL (default 1): launch every kernel with programmatic dependent launch (a kernel's
 * setup overlaps its predecessor; each kernel waits for its predecessor before touching memory). */
/* DYLLM_OPT_ATTN_INC (default 1): incremental softmax statistics for response tiles (see
 * dyllm_cache_refresh_stats); 0 = every tile computes its normaliser over all N keys. */
/* DYLLM_OPT_ATTN_T4 (default 32, range 0..32): in libraries built with -DDYLLM_FA_T4=1, the fused
 * attention computes exact-row tiles of at most this many rows transposed (S^T = K Q^T with the
 * keys on the 128 MMA rows, O^T = V^T P^T), so the tensor and exp work follows the row count
 * instead of a 128-row tile; 0 disables. The default build compiles those tiles out (measured
 * faster overall) and accepts the option without effect. */
/* DYLLM_OPT_ATTN_PINC (default 1): in full-input steps, prompt tiles update their rows' softmax
 * statistics by the keys changed since the previous full-input step (the list U: idx_in, then the
 * keys written by the response-only steps since), instead of recomputing them over all N keys
 * (SURVEY §8f1, D20). 0 = dense prompt tiles. */
enum { DYLLM_OPT_SKINNY_GEMM = 1, DYLLM_OPT_SKINNY_SPLIT = 2, DYLLM_OPT_ATTN_FUSED = 3, DYLLM_OPT_SKINNY_ONE_CHUNK = 4,
       DYLLM_OPT_PDL = 5, DYLLM_OPT_ATTN_INC = 6, DYLLM_OPT_ATTN_T4 = 7, DYLLM_OPT_ATTN_PINC = 8,
       DYLLM_OPT_ATTN_COS = 9, DYLLM_OPT_SKINNY_CHUNK = 10, DYLLM_OPT_SKINNY_KROT = 11,
       DYLLM_OPT_SKINNY_DEBUG = 12, DYLLM_OPT_SKINNY_KB = 13, DYLLM_OPT_QKV_FUSED = 14 };
/* DYLLM_OPT_QKV_FUSED (default 2): with head_dim 128 and at most 16384 rows, the QKV projection's
 * epilogue applies the bias and RoPE and writes the Q / K / V cache rows, dV and the compact copies
 * itself (SURVEY §8 rows a2 + a3 fused) — 1: in FullSteps, 2: in FullSteps and
 * full-input sparse steps, 0: never (the projection writes a bf16 QKV scratch and a separate kernel
 * does a3). Response-only steps stay unfused: there each SM pair holds one QKV tile and the fused
 * epilogue is exposed (measured slower). */
/* DYLLM_OPT_SKINNY_KB (default 0 = 128): k-block width of the skinny kernel's shared-memory ring
 * stages, 128 or 64 columns (64: half-size stages, twice as many in flight). */
/* DYLLM_OPT_SKINNY_DEBUG (default 0; measurement only, results are garbage when set): bit 0 runs
 * the skinny kernel without its operand TMA loads, bit 1 without its MMAs. */
/* DYLLM_OPT_SKINNY_KROT (default 0): the skinny kernel walks the k-blocks of a weight block's
 * segment starting at (block index x value) mod its k-block count, so that the pairs running
 * at the same time read different parts of the shared activation rows (same sums, another
 * accumulation order). */
/* DYLLM_OPT_SKINNY_CHUNK (default 0 = 256): largest number of activation rows per chunk of the
 * skinny GEMM when the rows are chunked (tuning hook). */
/* DYLLM_OPT_ATTN_COS (default 0, measured slower): head_dim-128 sparse steps form C_new, commit it to the C cache and
 * compute the per-(row, head) cosine partials in the attention epilogue; the
 * selection kernel then reads 16 bytes per (row, head) instead of both context rows. 0 = the
 * attention writes dC / C rows to scratch and the selection kernel forms, compares and commits. */
int dyllm_set_option(int option, int value);

/* Debug hook: when d_buf != NULL, kernels of family `which` (0 = skinny GEMM) write %globaltimer
 * stamps of their phases to d_buf ([grid][16] uint64, caller-owned device memory, must hold one
 * row per CTA of every traced launch); which = 1: the fused attention kernel writes per-role
 * mbarrier wait cycles (slots 0-2 producers, 3-8 MMA issuer, 9-12 softmax, 13 total). NULL disables. Process-wide; not thread-safe. */
int dyllm_debug_trace_buffer(int which, void *d_buf);

#ifdef __cplusplus
}
#endif
#endif /* DYLLM_API_H_ */
