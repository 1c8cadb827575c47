// dyllm.cu — the C ABI (include/dyllm.h) and the step orchestration:
// FullStep (Alg. 2), the per-layer SparseStep (Alg. 3 with Alg. 4 folded into the attention
// kernel), the denoise step (Alg. 1 body) and the unmasking rule. No host synchronisation
// inside a step: every kernel reads its row counts from device memory.
#include <nvtx3/nvToolsExt.h>
#include <dlfcn.h>
#include <math.h>
#include <nccl.h>

#include <atomic>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "fp32.h"
#include "internal.h"
#include "kernels.h"

// ------------------------------------------------------------------ error state
namespace dy {
static thread_local std::string g_err;
void set_error(const std::string &m) { g_err = m; }
}  // namespace dy

using namespace dy;

#define CHECK_ARG(cond, msg)        \
  do {                              \
    if (!(cond)) {                  \
      set_error(msg);               \
      return DYLLM_E_ARG;           \
    }                               \
  } while (0)
#define RET(expr)                   \
  do {                              \
    int _rc = (expr);               \
    if (_rc != DYLLM_OK) return _rc; \
  } while (0)

struct ProfRec {
  int cls;
  cudaEvent_t a, b;
};
struct dyllm_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 148;
  unsigned *masks = nullptr;   // K1 ballot words (capacity kMaskCap)
  unsigned *ticket = nullptr;  // K1 last-CTA ticket
  float *sk_ws = nullptr;      // skinny GEMM split-K partials
  int *sk_ctr = nullptr;       // skinny GEMM split-K counters
  int *attn_ctr = nullptr;     // fused attention scheduler counters [2]
  int *attn_fix = nullptr;     // fused attention fixup list [1 + kFixCap] (count zero between steps)
  // instrumentation
  bool prof = false;
  int cls_offset = 0;          // DYLLM_KC_FULL while a FullStep enqueues
  std::vector<cudaEvent_t> pool;
  size_t pool_next = 0;
  std::vector<ProfRec> recs;
};

static std::atomic<uint64_t> g_launches{0};

static cudaEvent_t prof_event(dyllm_ctx *c) {
  if (c->pool_next == c->pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->pool.push_back(e);
  }
  return c->pool[c->pool_next++];
}
// NVTX ranges (SURVEY §5 tracing): one per denoising / full step, per layer and per kernel
// launch, named by the kernel class; header-only NVTX v3 (no-ops unless a tool such as nsys or
// ncu --nvtx injects itself)
static const char *const kClassName[DYLLM_KC_COUNT] = {"qkv_gemm", "qkv_post", "attn",   "select",
                                                        "o_gemm",   "gu_gemm",  "down_gemm", "gather",
                                                        "scatter",  "lm_gemm",  "other"};
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
struct NvtxLayer {
  explicit NvtxLayer(int l) {
    char b[24];
    snprintf(b, sizeof(b), "layer %d", l);
    nvtxRangePushA(b);
  }
  ~NvtxLayer() { nvtxRangePop(); }
};

// RAII scope around one kernel launch: counts it and, when profiling, brackets it with events.
struct KScope {
  dyllm_ctx *c;
  int cls;
  cudaEvent_t a = nullptr;
  KScope(dyllm_ctx *ctx, int k) : c(ctx), cls(k + ctx->cls_offset) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    nvtxRangePushA(kClassName[k]);
    if (c->prof) {
      a = prof_event(c);
      cudaEventRecord(a, c->stream);
    }
  }
  ~KScope() {
    if (a) {
      cudaEvent_t b = prof_event(c);
      cudaEventRecord(b, c->stream);
      c->recs.push_back({cls, a, b});
    }
    nvtxRangePop();
  }
};
#define KL(cls, stmt)                  \
  do {                                 \
    KScope _ks(ctx, DYLLM_KC_##cls);   \
    stmt;                              \
  } while (0)
static constexpr int64_t kMaskCap = 1 << 20;
static constexpr int kFixCap = 1 << 16;
static bool g_attn_inc_enabled = true;   // test hook: incremental attention statistics (response tiles)
static bool g_attn_pinc_enabled = true;  // test hook: incremental prompt statistics in full-input steps
// fused similarity partials in the attention epilogue: built and parity-tested, off by
// default — same-box A/B (tools/gpu_r2_cos.sh): attention 141 -> 178 us per launch (the C_old read
// lands on each item's serial chain), selection 48 -> 26 us: 716 vs 724 tok/s
static bool g_attn_fuse_cos = false;
static int g_qkv_fused = 2;  // EPI_QKV: a3 in the QKV projection's epilogue: 1 FullSteps, 2 + full-input steps (DYLLM_OPT_QKV_FUSED)

struct LayerW {
  bf16 *g_attn, *wqkv, *bqkv, *wo, *g_ffn, *wgu, *wd;
};
struct dyllm_weights {
  dyllm_model_cfg cfg;
  bf16 *emb = nullptr, *g_final = nullptr, *lm_head = nullptr;
  std::vector<LayerW> L;
  std::vector<void *> allocs;
};
struct LayerC {
  bf16 *K, *V, *Q, *C, *H;
  float2 *st = nullptr;  // [rows][H] softmax statistics (m c, l) of the fused attention (head_dim 128)
  mutable bool st_ok = false;  // statistics of the response rows are current (incremental tiles
                               // allowed); cleared whenever K or Q may be written from outside
  // incremental prompt statistics of full-input steps: the prompt rows' statistics are
  // current as of the start of `epoch` (every full-input attention, FullStep or refresh begins a new
  // one); a key row written since then has dtag == epoch and its key at the epoch start in Kfi
  bf16 *Kfi = nullptr;
  uint32_t *dtag = nullptr;
  uint32_t epoch = 1;
  mutable bool pst_ok = false;
};
struct dyllm_cache {
  dyllm_model_cfg m;
  dyllm_run_cfg r;
  dyllm_ctx *ctx;
  int N, rows;
  std::vector<LayerC> L;
  bf16 *H0;
  bf16 *Xn, *qkv, *dV, *Qx, *Kx, *Kxo, *Cn, *Cg, *h, *hn, *act, *ffo, *Xf;
  uint32_t *rowflag;     // [rows] == row_tag: exact row (idx_in) of the current layer step
  uint8_t *snapm;        // [rows] packed rows written for the first time in their statistics epoch (EPI_QKV)
  uint32_t row_tag = 0;  // advanced by every layer step (no clearing pass over rowflag)
  float4 *partials;
  int *lst[2], *lst_off[2];
  int *carried, *carried_off;
  bool carried_valid = false;
  int *ap_rows, *ap_off, *all_rows, *all_off, *zero_off, *lm_rows, *lm_off;
  int *dec_prev;
  int *qx_rows, *qx_off;  // layer1_policy 0: decoded rows outside idx_in (Q-only refresh, D6)
  int *urows = nullptr, *ucnt = nullptr;  // changed-key lists U of a full-input step ([b][N], [b])
  bf16 *Kun = nullptr, *Kuo = nullptr;    // their keys now / at the statistics epoch (compact per sequence)
  float4 *cos_part = nullptr;             // [rows][H] similarity partials of the fused attention epilogue
  // tensor parallelism: this cache is shard tp_shard of a group (local heads / FFN)
  dyllm_tp *tp = nullptr;
  int tp_shard = 0;
  float4 *tp_part = nullptr;              // [rows] this shard's similarity partial sums, then the group's
  int32_t *tp_tokens = nullptr;           // loopback shards > 0: private copy of the step's tokens
  int32_t *tr_lists = nullptr, *tr_offs = nullptr;  // dyllm_cache_set_trace (caller-owned)
  float *tr_sims = nullptr;
  float *sim;  // per-row similarity scratch (fraction mode)
  float2 *rope_cs;  // [N][head_dim/2] (cos, sin) table
  float2 *stats;    // [b*N][H] attention row statistics scratch
  // fp32-parity mode (dtype 1): every cache / scratch row above is fp32 (element size es)
  int es = 2;
  float *gu32 = nullptr;      // [rows][2F] interleaved gate/up products
  float *logits32 = nullptr;  // [b*block][vocab]
  int *posmap = nullptr;      // [rows] index of a row in idx_in, -1 otherwise
  bool have_dec_prev = false;
  bool initialized = false;
  std::vector<void *> allocs;
};

static int dalloc(std::vector<void *> &v, void **p, size_t bytes) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) {
    set_error(std::string("cudaMalloc(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
    return DYLLM_E_NOMEM;
  }
  v.push_back(*p);
  return DYLLM_OK;
}
template <typename T>
static int dalloc_t(std::vector<void *> &v, T **p, size_t count) {
  return dalloc(v, reinterpret_cast<void **>(p), count * sizeof(T));
}

static int sticky(dyllm_ctx *ctx) {
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) {
    set_error(std::string("sticky CUDA error: ") + cudaGetErrorString(e));
    return DYLLM_E_CUDA;
  }
  (void)ctx;
  return DYLLM_OK;
}

static int validate_model(const dyllm_model_cfg *m) {
  if (!m) {
    set_error("null model cfg");
    return DYLLM_E_ARG;
  }
  const int hd = m->head_dim;
  if (m->n_layers < 1 || m->d_model < 64 || m->n_heads < 1 || m->n_kv_heads < 1 || m->vocab < 2 ||
      m->mask_id < 0 || m->mask_id >= m->vocab || m->dtype < 0 || m->dtype > 1) {
    set_error("model cfg out of range");
    return DYLLM_E_ARG;
  }
  if (m->d_model % 64 || (hd != 16 && hd != 32 && hd != 64 && hd != 128) || m->n_heads % m->n_kv_heads ||
      (m->n_heads * hd) % 64 || m->d_ff % 128 || m->vocab % 8 || m->residual_mode < 0 || m->residual_mode > 1) {
    set_error("model cfg shape unsupported: d_model%64, head_dim in {16,32,64,128}, H%KVH, (H*hd)%64, d_ff%128, vocab%8");
    return DYLLM_E_SHAPE;
  }
  return DYLLM_OK;
}

extern "C" {

const char *dyllm_last_error(void) { return g_err.c_str(); }
int dyllm_version(void) { return 100; }

int dyllm_ctx_create(int device, void *cuda_stream, dyllm_ctx **out) {
  CHECK_ARG(out, "null out");
  DY_CUDA(cudaSetDevice(device));
  dyllm_ctx *c = new dyllm_ctx();
  c->device = device;
  if (cuda_stream) {
    c->stream = static_cast<cudaStream_t>(cuda_stream);
  } else {
    DY_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  DY_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
  int major = 0;
  DY_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  if (major != 10) {
    set_error("libdyllm requires an sm_100 (B200) device");
    delete c;
    return DYLLM_E_ARG;
  }
  DY_CUDA(cudaMalloc(&c->masks, kMaskCap * sizeof(unsigned)));
  // K1 tickets: [0] global last-CTA ticket, [1 + s] per-sequence tickets (fraction mode, batch <= 1024)
  DY_CUDA(cudaMalloc(&c->ticket, 1025 * sizeof(unsigned)));
  DY_CUDA(cudaMemset(c->ticket, 0, 1025 * sizeof(unsigned)));
  DY_CUDA(cudaMalloc(&c->sk_ws, skinny_ws_floats(c->num_sms) * sizeof(float)));
  DY_CUDA(cudaMalloc(&c->sk_ctr, kSkinnyCtrCap * sizeof(int)));
  DY_CUDA(cudaMemset(c->sk_ctr, 0, kSkinnyCtrCap * sizeof(int)));
  DY_CUDA(cudaMalloc(&c->attn_ctr, 2 * sizeof(int)));
  DY_CUDA(cudaMemset(c->attn_ctr, 0, 2 * sizeof(int)));
  DY_CUDA(cudaMalloc(&c->attn_fix, (1 + kFixCap) * sizeof(int)));
  DY_CUDA(cudaMemset(c->attn_fix, 0, (1 + kFixCap) * sizeof(int)));
  *out = c;
  return DYLLM_OK;
}

int dyllm_ctx_sync(dyllm_ctx *ctx) {
  CHECK_ARG(ctx, "null ctx");
  DY_CUDA(cudaStreamSynchronize(ctx->stream));
  return DYLLM_OK;
}

void dyllm_ctx_destroy(dyllm_ctx *ctx) {
  if (!ctx) return;
  cudaStreamSynchronize(ctx->stream);
  cudaFree(ctx->masks);
  cudaFree(ctx->ticket);
  cudaFree(ctx->sk_ws);
  cudaFree(ctx->sk_ctr);
  cudaFree(ctx->attn_ctr);
  cudaFree(ctx->attn_fix);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

// ------------------------------------------------------------------ weights
int64_t dyllm_weights_blob_elems(const dyllm_model_cfg *m) {
  if (validate_model(m) != DYLLM_OK) return -1;
  const int64_t d = m->d_model, qw = static_cast<int64_t>(m->n_heads) * m->head_dim,
                kw = static_cast<int64_t>(m->n_kv_heads) * m->head_dim, F = m->d_ff, V = m->vocab;
  int64_t per = d + qw * d + 2 * kw * d + (m->qkv_bias ? qw + 2 * kw : 0) + d * qw + d + 2 * F * d + d * F;
  return V * d + d + V * d + per * m->n_layers;
}

static int alloc_weights(const dyllm_model_cfg *m, dyllm_weights *w) {
  const int64_t d = m->d_model, qw = static_cast<int64_t>(m->n_heads) * m->head_dim,
                kw = static_cast<int64_t>(m->n_kv_heads) * m->head_dim, F = m->d_ff, V = m->vocab;
  w->cfg = *m;
  RET(dalloc_t(w->allocs, &w->emb, V * d));
  RET(dalloc_t(w->allocs, &w->g_final, d));
  RET(dalloc_t(w->allocs, &w->lm_head, V * d));
  w->L.resize(m->n_layers);
  for (auto &L : w->L) {
    RET(dalloc_t(w->allocs, &L.g_attn, d));
    RET(dalloc_t(w->allocs, &L.wqkv, (qw + 2 * kw) * d));
    L.bqkv = nullptr;
    if (m->qkv_bias) RET(dalloc_t(w->allocs, &L.bqkv, qw + 2 * kw));
    RET(dalloc_t(w->allocs, &L.wo, d * qw));
    RET(dalloc_t(w->allocs, &L.g_ffn, d));
    RET(dalloc_t(w->allocs, &L.wgu, 2 * F * d));
    RET(dalloc_t(w->allocs, &L.wd, d * F));
  }
  return DYLLM_OK;
}

void dyllm_weights_destroy(dyllm_weights *w) {
  if (!w) return;
  for (void *p : w->allocs) cudaFree(p);
  delete w;
}

int dyllm_weights_load(dyllm_ctx *ctx, const dyllm_model_cfg *m, const uint16_t *h_blob, int64_t n_elems,
                       dyllm_weights **out) {
  CHECK_ARG(ctx && h_blob && out, "null argument");
  RET(validate_model(m));
  const int64_t need = dyllm_weights_blob_elems(m);
  if (n_elems != need) {
    set_error("blob has " + std::to_string(n_elems) + " elements, expected " + std::to_string(need));
    return DYLLM_E_SHAPE;
  }
  dyllm_weights *w = new dyllm_weights();
  int rc = alloc_weights(m, w);
  if (rc) {
    dyllm_weights_destroy(w);
    return rc;
  }
  const int64_t d = m->d_model, qw = static_cast<int64_t>(m->n_heads) * m->head_dim,
                kw = static_cast<int64_t>(m->n_kv_heads) * m->head_dim, F = m->d_ff, V = m->vocab;
  const uint16_t *p = h_blob;
  auto put = [&](bf16 *dst, int64_t n) -> int {
    DY_CUDA(cudaMemcpy(dst, p, n * 2, cudaMemcpyHostToDevice));
    p += n;
    return DYLLM_OK;
  };
#define PUT(dst, n)                 \
  do {                              \
    int _r = put(dst, n);           \
    if (_r) {                       \
      dyllm_weights_destroy(w);     \
      return _r;                    \
    }                               \
  } while (0)
  PUT(w->emb, V * d);
  PUT(w->g_final, d);
  PUT(w->lm_head, V * d);
  for (auto &L : w->L) {
    PUT(L.g_attn, d);
    PUT(L.wqkv, (qw + 2 * kw) * d);   // wq, wk, wv are consecutive in the blob
    if (m->qkv_bias) PUT(L.bqkv, qw + 2 * kw);
    PUT(L.wo, d * qw);
    PUT(L.g_ffn, d);
    // gate / up interleaved in blocks of kGuIl rows: [gate blk][up blk] (SwiGLU GEMM epilogues)
    const uint16_t *gate = p, *up = p + F * d;
    for (int64_t b = 0; b < F / kGuIl; ++b) {
      cudaError_t e1 =
          cudaMemcpy(L.wgu + (2 * b) * kGuIl * d, gate + b * kGuIl * d, kGuIl * d * 2, cudaMemcpyHostToDevice);
      cudaError_t e2 =
          cudaMemcpy(L.wgu + (2 * b + 1) * kGuIl * d, up + b * kGuIl * d, kGuIl * d * 2, cudaMemcpyHostToDevice);
      if (e1 != cudaSuccess || e2 != cudaSuccess) {
        set_error("cudaMemcpy gate/up failed");
        dyllm_weights_destroy(w);
        return DYLLM_E_CUDA;
      }
    }
    p += 2 * F * d;
    PUT(L.wd, d * F);
  }
#undef PUT
  *out = w;
  return DYLLM_OK;
}

static uint64_t mix64_host(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static uint64_t stream_key(uint64_t seed, uint64_t stream) { return mix64_host(seed ^ mix64_host(stream)); }
enum { T_WQ = 1, T_WK = 2, T_WV = 3, T_BQ = 4, T_BK = 5, T_BV = 6, T_WO = 7, T_GATE = 8, T_UP = 9, T_DOWN = 10,
       T_EMB = 20, T_LM = 22 };
static constexpr uint64_t kGlobalLayer = 65535;

int dyllm_weights_init_random(dyllm_ctx *ctx, const dyllm_model_cfg *m, uint64_t seed, double std,
                              dyllm_weights **out) {
  CHECK_ARG(ctx && out, "null argument");
  RET(validate_model(m));
  dyllm_weights *w = new dyllm_weights();
  int rc = alloc_weights(m, w);
  if (rc) {
    dyllm_weights_destroy(w);
    return rc;
  }
  const int64_t d = m->d_model, qw = static_cast<int64_t>(m->n_heads) * m->head_dim,
                kw = static_cast<int64_t>(m->n_kv_heads) * m->head_dim, F = m->d_ff, V = m->vocab;
  const float scale = static_cast<float>(std / sqrt((65536.0 * 65536.0 - 1.0) / 3.0));
  cudaStream_t st = ctx->stream;
  auto key = [&](uint64_t layer, int code) { return stream_key(seed, layer * 64 + code); };
  launch_ih4_fill(w->emb, V, d, key(kGlobalLayer, T_EMB), 0, 0, scale, st);
  launch_fill_const(w->g_final, d, 1.f, st);
  launch_ih4_fill(w->lm_head, V, d, key(kGlobalLayer, T_LM), 0, 0, scale, st);
  for (int l = 0; l < m->n_layers; ++l) {
    LayerW &L = w->L[l];
    launch_fill_const(L.g_attn, d, 1.f, st);
    launch_fill_const(L.g_ffn, d, 1.f, st);
    launch_ih4_fill(L.wqkv, qw, d, key(l, T_WQ), 0, 0, scale, st);
    launch_ih4_fill(L.wqkv + qw * d, kw, d, key(l, T_WK), 0, 0, scale, st);
    launch_ih4_fill(L.wqkv + (qw + kw) * d, kw, d, key(l, T_WV), 0, 0, scale, st);
    if (m->qkv_bias) {
      launch_ih4_fill(L.bqkv, 1, qw, key(l, T_BQ), 0, 0, scale, st);
      launch_ih4_fill(L.bqkv + qw, 1, kw, key(l, T_BK), 0, 0, scale, st);
      launch_ih4_fill(L.bqkv + qw + kw, 1, kw, key(l, T_BV), 0, 0, scale, st);
    }
    launch_ih4_fill(L.wo, d, qw, key(l, T_WO), 0, 0, scale, st);
    launch_ih4_fill(L.wgu, 2 * F, d, key(l, T_GATE), key(l, T_UP), kGuIl, scale, st);
    launch_ih4_fill(L.wd, d, F, key(l, T_DOWN), 0, 0, scale, st);
  }
  cudaError_t e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("init_random: ") + cudaGetErrorString(e));
    dyllm_weights_destroy(w);
    return DYLLM_E_CUDA;
  }
  *out = w;
  return DYLLM_OK;
}

// ------------------------------------------------------------------ caches
int dyllm_cache_create(dyllm_ctx *ctx, const dyllm_weights *w, const dyllm_run_cfg *r, dyllm_cache **out) {
  CHECK_ARG(ctx && w && r && out, "null argument");
  const dyllm_model_cfg &m = w->cfg;
  if (r->batch < 1 || r->batch > 1024 || r->L_P < 1 || r->L_R < 1 || r->block < 1 || r->block > 256 ||
      r->L_R % r->block || r->n_u < 1 || r->n_u > 64 || r->n_u > r->block || r->block % r->n_u || r->T_full < 0 || r->full_period < 1 ||
      r->layer1_policy < 0 || r->layer1_policy > 1 || r->cmp < 0 || r->cmp > 1 || r->L_P + r->L_R > 32768 ||
      r->select_mode < 0 || r->select_mode > 1) {
    set_error("run cfg out of range (batch<=1024, block<=256 | L_R, n_u<=64 | block, N<=32768)");
    return DYLLM_E_ARG;
  }
  dyllm_cache *c = new dyllm_cache();
  c->m = m;
  c->r = *r;
  c->ctx = ctx;
  c->N = r->L_P + r->L_R;
  c->rows = r->batch * c->N;
  const int64_t rows = c->rows, d = m.d_model, qw = static_cast<int64_t>(m.n_heads) * m.head_dim,
                kw = static_cast<int64_t>(m.n_kv_heads) * m.head_dim, F = m.d_ff;
  const int64_t lm_cap = static_cast<int64_t>(r->batch) * r->block;
  auto &A = c->allocs;
  int rc = DYLLM_OK;
#define AL(p, n)                        \
  do {                                  \
    rc = dalloc_t(A, &(p), (n));        \
    if (rc) {                           \
      dyllm_cache_destroy(c);           \
      return rc;                        \
    }                                   \
  } while (0)
  // activation rows: bf16, or fp32 in the fp32-parity mode (elements of es bytes)
  const bool f32 = m.dtype == 1;
  c->es = f32 ? 4 : 2;
#define ALE(p, n)                                                                          \
  do {                                                                                     \
    rc = dalloc(A, reinterpret_cast<void **>(&(p)), static_cast<size_t>(n) * c->es);     \
    if (rc) {                                                                              \
      dyllm_cache_destroy(c);                                                              \
      return rc;                                                                           \
    }                                                                                      \
  } while (0)
  c->L.resize(m.n_layers);
  for (auto &L : c->L) {
    ALE(L.K, rows * kw);
    ALE(L.V, rows * kw);
    ALE(L.Q, rows * qw);
    ALE(L.C, rows * qw);
    ALE(L.H, rows * d);
    if (m.head_dim == 128 && !f32) {
      AL(L.st, rows * m.n_heads);
      AL(L.Kfi, rows * kw);
      AL(L.dtag, rows);
    }
  }
  if (m.head_dim == 128 && !f32) {
    AL(c->urows, rows);
    AL(c->ucnt, r->batch);
    AL(c->Kun, rows * kw);
    AL(c->Kuo, rows * kw);
    AL(c->cos_part, rows * m.n_heads);
  }
  ALE(c->H0, rows * d);
  ALE(c->Xn, rows * d);
  ALE(c->qkv, rows * (qw + 2 * kw));
  ALE(c->dV, rows * kw);
  ALE(c->Qx, rows * qw);
  ALE(c->Kx, rows * kw);
  ALE(c->Kxo, rows * kw);
  AL(c->rowflag, rows);
  AL(c->snapm, rows);
  ALE(c->Cn, rows * qw);
  ALE(c->Cg, rows * qw);
  ALE(c->h, rows * d);
  ALE(c->hn, rows * d);
  ALE(c->act, rows * F);
  ALE(c->ffo, rows * d);
  ALE(c->Xf, lm_cap * d);
  AL(c->partials, lm_cap * gemm_lmhead_ntiles(m.vocab));
  if (f32) {
    AL(c->gu32, rows * 2 * F);
    AL(c->logits32, lm_cap * m.vocab);
    AL(c->posmap, rows);
  }
#undef ALE
  for (int i = 0; i < 2; ++i) {
    AL(c->lst[i], rows);
    AL(c->lst_off[i], r->batch + 1);
  }
  AL(c->carried, rows);
  AL(c->carried_off, r->batch + 1);
  AL(c->ap_rows, rows);
  AL(c->ap_off, r->batch + 1);
  AL(c->all_rows, rows);
  AL(c->all_off, r->batch + 1);
  AL(c->zero_off, r->batch + 1);
  AL(c->lm_rows, lm_cap);
  AL(c->lm_off, r->batch + 1);
  AL(c->dec_prev, static_cast<int64_t>(r->batch) * r->n_u);
  AL(c->qx_rows, rows);
  AL(c->qx_off, r->batch + 1);
  AL(c->sim, rows);
  AL(c->rope_cs, static_cast<int64_t>(c->N) * (m.head_dim / 2));
  AL(c->stats, rows * m.n_heads);
#undef AL
  cudaStream_t st = ctx->stream;
  // compact scratch rows past the live count are read (with zero weight) by attention tiles:
  // start them finite
  const bool ok = cudaMemsetAsync(c->dV, 0, rows * kw * c->es, st) == cudaSuccess &&
                  cudaMemsetAsync(c->Kx, 0, rows * kw * c->es, st) == cudaSuccess &&
                  cudaMemsetAsync(c->Kxo, 0, rows * kw * c->es, st) == cudaSuccess &&
                  cudaMemsetAsync(c->rowflag, 0, rows * sizeof(uint32_t), st) == cudaSuccess &&
                  cudaMemsetAsync(c->Qx, 0, rows * qw * c->es, st) == cudaSuccess &&
                  cudaMemsetAsync(c->zero_off, 0, (r->batch + 1) * sizeof(int), st) == cudaSuccess;
  bool ok2 = ok;
  // list buffers start defined (whole-capacity copies of partly used lists, e.g. the carried set,
  // would otherwise read uninitialised tails: compute-sanitizer initcheck)
  for (int i = 0; i < 2; ++i) ok2 = ok2 && cudaMemsetAsync(c->lst[i], 0, rows * sizeof(int), st) == cudaSuccess;
  ok2 = ok2 && cudaMemsetAsync(c->carried, 0, rows * sizeof(int), st) == cudaSuccess;
  for (auto &L : c->L)
    if (L.dtag) ok2 = ok2 && cudaMemsetAsync(L.dtag, 0, rows * sizeof(uint32_t), st) == cudaSuccess;
  if (c->Kun)
    ok2 = ok2 && cudaMemsetAsync(c->Kun, 0, rows * kw * 2, st) == cudaSuccess &&
          cudaMemsetAsync(c->Kuo, 0, rows * kw * 2, st) == cudaSuccess;
  if (!ok2) {
    set_error("memset failed");
    dyllm_cache_destroy(c);
    return DYLLM_E_CUDA;
  }
  launch_build_list(0, nullptr, nullptr, nullptr, 0, 0, r->batch, c->N, 0, 0, c->all_rows, c->all_off, st);
  launch_rope_table(c->rope_cs, c->N, m.head_dim, static_cast<double>(m.rope_theta), st);
  if (cudaStreamSynchronize(st) != cudaSuccess || cudaGetLastError() != cudaSuccess) {
    set_error("cache_create: CUDA error");
    dyllm_cache_destroy(c);
    return DYLLM_E_CUDA;
  }
  *out = c;
  return DYLLM_OK;
}

static void tp_forget(dyllm_tp *tp, const dyllm_cache *c);  // tensor-parallel group bookkeeping (below)

void dyllm_cache_destroy(dyllm_cache *c) {
  if (!c) return;
  if (c->tp) tp_forget(c->tp, c);  // a group must not keep a destroyed shard
  for (void *p : c->allocs) cudaFree(p);
  delete c;
}

// ------------------------------------------------------------------ step internals
static int gemm(dyllm_ctx *ctx, const int *M_ptr, int M_cap, int N, int K, const bf16 *A, const bf16 *W, bf16 *D,
                int ldd, int epi, const bf16 *resid = nullptr, int ldr = 0, const int *resid_rows = nullptr,
                const bf16 *bias = nullptr, float4 *partials = nullptr, const int *out_rows = nullptr,
                int excl_col = -1) {
  GemmCall g;
  g.excl_col = excl_col;
  g.M_ptr = M_ptr;
  g.M_cap = M_cap;
  g.N = N;
  g.K = K;
  g.A = A;
  g.W = W;
  g.D = D;
  g.ldd = ldd;
  g.resid = resid;
  g.ldr = ldr;
  g.resid_rows = resid_rows;
  g.bias = bias;
  g.partials = partials;
  g.out_rows = out_rows;
  g.epi = epi;
  g.ws = ctx->sk_ws;
  g.ctr = ctx->sk_ctr;
  return gemm_launch(g, ctx->num_sms, ctx->stream);
}

// a2 + a3 in one launch (EPI_QKV): the QKV projection of the rows of A whose epilogue applies the bias
// and RoPE and writes the cache rows, dV and the compact copies (q: everything but A / W / bias)
static bool qkv_fusable(const dyllm_cache *c, bool full_step) {
  const dyllm_model_cfg &m = c->m;
  const int qw = m.n_heads * m.head_dim, kw = m.n_kv_heads * m.head_dim;
  return g_qkv_fused >= (full_step ? 1 : 2) && g_skinny_enabled && m.head_dim == 128 && c->rows <= kSkinnyMaxM &&
         (qw + 2 * kw) % 256 == 0 && m.d_model % 128 == 0;
}
static int gemm_qkv(dyllm_ctx *ctx, const dyllm_cache *c, const int *M_ptr, const bf16 *A, const bf16 *W,
                    const bf16 *bias, const QkvEpi &q) {
  const dyllm_model_cfg &m = c->m;
  GemmCall g;
  g.M_ptr = M_ptr;
  g.M_cap = c->rows;
  g.N = (m.n_heads + 2 * m.n_kv_heads) * m.head_dim;
  g.K = m.d_model;
  g.A = A;
  g.W = W;
  g.bias = bias;
  g.epi = EPI_QKV;
  g.ws = ctx->sk_ws;
  g.ctr = ctx->sk_ctr;
  g.qkv = q;
  return gemm_launch(g, ctx->num_sms, ctx->stream);
}

// post-attention block on rows listed by (rows, M_ptr): h = x + C W_o ; out = h + FFN(RMSNorm(h))
// (residual_mode 0) or h = RMSNorm(C W_o) ; out = FFN(h) (paper_literal).
// A_c: contiguous C rows [M][qw]; x rows read through resid_rows from Hprev; result in `out`.
static int post_attention(dyllm_ctx *ctx, const dyllm_weights *w, dyllm_cache *c, int l, const int *M_ptr,
                          const bf16 *A_c, const bf16 *Hprev, const int *resid_rows, bf16 *out) {
  const dyllm_model_cfg &m = c->m;
  const int d = m.d_model, qw = m.n_heads * m.head_dim, F = m.d_ff, rows = c->rows;
  const LayerW &L = w->L[l];
  cudaStream_t st = ctx->stream;
  const bool res = m.residual_mode == 0;
  KL(O_GEMM, RET(gemm(ctx, M_ptr, rows, d, qw, A_c, L.wo, c->h, d, res ? EPI_RESID : EPI_BF16, Hprev, d, resid_rows)));
  KL(OTHER, launch_rmsnorm_rows(c->h, M_ptr, rows, L.g_ffn, m.rms_eps, c->hn, d, st));
  KL(GU_GEMM, RET(gemm(ctx, M_ptr, rows, 2 * F, d, c->hn, L.wgu, c->act, F, EPI_SWIGLU)));
  // the down projection writes its rows straight into H_l at their row ids (scatter-back fused,
  // rows outside the list keep their cached output)
  KL(DOWN_GEMM, RET(gemm(ctx, M_ptr, rows, d, F, c->act, L.wd, out, d, res ? EPI_RESID : EPI_BF16, c->h, d, nullptr,
                         nullptr, nullptr, resid_rows)));
  return DYLLM_OK;
}

// ------------------------------------------------------------------ fp32-parity mode (dtype 1, D12)
// The same step structure as the bf16 path below, on fp32 rows with the SIMT kernels of fp32.cu.
static inline float *fp(void *p) { return static_cast<float *>(p); }

static f32::GemmF32 g32(const int *M_ptr, int M_cap, int N, int K, const float *A, const bf16 *W, float *D, int ldd) {
  f32::GemmF32 g;
  g.M_ptr = M_ptr;
  g.M_cap = M_cap;
  g.N = N;
  g.K = K;
  g.A = A;
  g.lda = K;
  g.W = W;
  g.D = D;
  g.ldd = ldd;
  return g;
}

// O-proj + FFN on the rows listed by (rows, M_ptr) (nullptr: all rows); A_c rows read at a_rows.
static void post_attention_f32(dyllm_ctx *ctx, const dyllm_weights *w, dyllm_cache *c, int l, const int *M_ptr,
                               const float *A_c, const int *a_rows, const float *Hprev, const int *rows, float *out) {
  const dyllm_model_cfg &m = c->m;
  const int d = m.d_model, qw = m.n_heads * m.head_dim, F = m.d_ff, R = c->rows;
  const LayerW &L = w->L[l];
  cudaStream_t st = ctx->stream;
  const bool res = m.residual_mode == 0;
  f32::GemmF32 go = g32(M_ptr, R, d, qw, A_c, L.wo, fp(c->h), d);
  go.a_rows = a_rows;
  if (res) {  // h = x + C W_o
    go.resid = Hprev;
    go.ldr = d;
    go.resid_rows = rows;
  }
  KL(O_GEMM, f32::gemm(go, st));
  KL(OTHER, f32::gather_rmsnorm(fp(c->h), nullptr, M_ptr, R, L.g_ffn, m.rms_eps, fp(c->hn), d, st));
  KL(GU_GEMM, f32::gemm(g32(M_ptr, R, 2 * F, d, fp(c->hn), L.wgu, c->gu32, 2 * F), st));
  KL(OTHER, f32::swiglu(c->gu32, M_ptr, R, F, fp(c->act), st));
  f32::GemmF32 gd = g32(M_ptr, R, d, F, fp(c->act), L.wd, out, d);
  gd.out_rows = rows;  // scatter-back
  if (res) {
    gd.resid = fp(c->h);
    gd.ldr = d;
  }
  KL(DOWN_GEMM, f32::gemm(gd, st));
}

static int full_step_f32(dyllm_ctx *ctx, const dyllm_weights *w, dyllm_cache *c, const int *d_tokens) {
  const dyllm_model_cfg &m = c->m;
  const int d = m.d_model, qw = m.n_heads * m.head_dim, kw = m.n_kv_heads * m.head_dim, rows = c->rows;
  cudaStream_t st = ctx->stream;
  ctx->cls_offset = DYLLM_KC_FULL;
  KL(OTHER, f32::embed(d_tokens, nullptr, nullptr, rows, w->emb, fp(c->H0), d, st));
  for (int l = 0; l < m.n_layers; ++l) {
    const LayerW &L = w->L[l];
    LayerC &C = c->L[l];
    const float *Hprev = fp(l == 0 ? c->H0 : c->L[l - 1].H);
    KL(GATHER, f32::gather_rmsnorm(Hprev, nullptr, nullptr, rows, L.g_attn, m.rms_eps, fp(c->Xn), d, st));
    KL(QKV_GEMM, f32::gemm(g32(nullptr, rows, qw + 2 * kw, d, fp(c->Xn), L.wqkv, fp(c->qkv), qw + 2 * kw), st));
    KL(QKV_POST, f32::qkv_post(fp(c->qkv), nullptr, nullptr, rows, L.bqkv, c->N, m.n_heads, m.n_kv_heads, m.head_dim,
                               c->rope_cs, fp(C.Q), fp(C.K), fp(C.V), nullptr, 0, st));
    f32::F32Attn a{};
    a.batch = c->r.batch;
    a.N = c->N;
    a.H = m.n_heads;
    a.KVH = m.n_kv_heads;
    a.hd = m.head_dim;
    a.row_lo = 0;
    a.scale = 1.f / sqrtf(static_cast<float>(m.head_dim));
    a.Q = fp(C.Q);
    a.K = fp(C.K);
    a.V = fp(C.V);
    a.C_cache = fp(C.C);
    a.C_out = fp(C.C);
    a.all_exact = true;
    KL(ATTN, f32::attention(a, st));
    post_attention_f32(ctx, w, c, l, nullptr, fp(C.C), nullptr, Hprev, nullptr, fp(C.H));
  }
  ctx->cls_offset = 0;
  c->carried_valid = false;
  c->have_dec_prev = false;
  c->initialized = true;
  DY_CUDA(cudaGetLastError());
  return DYLLM_OK;
}

static int layer_step_f32(dyllm_ctx *ctx, const dyllm_weights *w, dyllm_cache *c, int l, int row_lo,
                          const int *idx_in, const int *off_in, float tau, int *idx_out, int *off_out, float *sim,
                          int *counts) {
  const dyllm_model_cfg &m = c->m;
  const int b = c->r.batch, N = c->N, rows = c->rows;
  const int d = m.d_model, qw = m.n_heads * m.head_dim, kw = m.n_kv_heads * m.head_dim;
  const LayerW &L = w->L[l];
  LayerC &C = c->L[l];
  const float *Hprev = fp(l == 0 ? c->H0 : c->L[l - 1].H);
  cudaStream_t st = ctx->stream;
  const int *M_in = off_in + b;
  // a1-a3: RMSNorm(x[idx_in]) -> QKV -> RoPE, dV (before the overwrite), in-place K/V/Q rows
  KL(GATHER, f32::gather_rmsnorm(Hprev, idx_in, M_in, rows, L.g_attn, m.rms_eps, fp(c->Xn), d, st));
  KL(QKV_GEMM, f32::gemm(g32(M_in, rows, qw + 2 * kw, d, fp(c->Xn), L.wqkv, fp(c->qkv), qw + 2 * kw), st));
  KL(QKV_POST, f32::qkv_post(fp(c->qkv), idx_in, M_in, rows, L.bqkv, N, m.n_heads, m.n_kv_heads, m.head_dim,
                             c->rope_cs, fp(C.Q), fp(C.K), fp(C.V), fp(c->dV), 0, st));
  // a4: exact rows (idx_in) and Alg. 4 rows, dense over the merged K
  KL(OTHER, f32::posmap(idx_in, M_in, rows, c->posmap, st));
  f32::F32Attn a{};
  a.batch = b;
  a.N = N;
  a.H = m.n_heads;
  a.KVH = m.n_kv_heads;
  a.hd = m.head_dim;
  a.row_lo = row_lo;
  a.scale = 1.f / sqrtf(static_cast<float>(m.head_dim));
  a.Q = fp(C.Q);
  a.K = fp(C.K);
  a.V = fp(C.V);
  a.dV = fp(c->dV);
  a.C_cache = fp(C.C);
  a.C_out = fp(c->Cn);
  a.sal_rows = idx_in;
  a.sal_off = off_in;
  a.posmap = c->posmap;
  a.all_exact = false;
  KL(ATTN, f32::attention(a, st));
  // a5: cosine + threshold + compaction, C_cache <- C_new
  const bool fmode = c->r.select_mode == 1;
  KL(SELECT, f32::select(fp(c->Cn), fp(C.C), b, N, row_lo, qw, fmode ? 2.f : tau, c->r.cmp, fmode ? tau : -1.f,
                         sim ? sim : c->sim, idx_out, off_out, counts, st));
  // a6-a8 on idx_out, scattered into H_l
  post_attention_f32(ctx, w, c, l, off_out + b, fp(C.C), idx_out, Hprev, idx_out, fp(C.H));
  DY_CUDA(cudaGetLastError());
  return DYLLM_OK;
}

// FullStep (Alg. 2): every row of every sequence, all caches rewritten.
// FullStep layer, phase 1 (Alg. 2 lines 3-5): every row's Q/K/V and exact context
static int full_attn_phase(dyllm_ctx *ctx, const dyllm_weights *w, dyllm_cache *c, int l) {
  const dyllm_model_cfg &m = c->m;
  const int d = m.d_model, qw = m.n_heads * m.head_dim, kw = m.n_kv_heads * m.head_dim, rows = c->rows;
  cudaStream_t st = ctx->stream;
  const LayerW &L = w->L[l];
  LayerC &C = c->L[l];
  const bf16 *Hprev = l == 0 ? c->H0 : c->L[l - 1].H;
    KL(GATHER, launch_gather_rmsnorm(Hprev, nullptr, nullptr, rows, L.g_attn, m.rms_eps, c->Xn, d, st));
    if (qkv_fusable(c, true)) {
      QkvEpi q;
      q.N = c->N;
      q.H = m.n_heads;
      q.KVH = m.n_kv_heads;
      q.rope_cs = c->rope_cs;
      q.Qc = C.Q;
      q.Kc = C.K;
      q.Vc = C.V;
      KL(QKV_GEMM, RET(gemm_qkv(ctx, c, nullptr, c->Xn, L.wqkv, L.bqkv, q)));
    } else {
      KL(QKV_GEMM, RET(gemm(ctx, nullptr, rows, qw + 2 * kw, d, c->Xn, L.wqkv, c->qkv, qw + 2 * kw, EPI_BF16)));
      KL(QKV_POST, launch_qkv_post(c->qkv, nullptr, nullptr, rows, L.bqkv, c->N, m.n_heads, m.n_kv_heads, m.head_dim,
                                   c->rope_cs, C.Q, C.K, C.V, nullptr, nullptr, nullptr, nullptr, nullptr, 0u, st));
    }
    AttnArgs a{};
    a.batch = c->r.batch;
    a.N = c->N;
    a.H = m.n_heads;
    a.KVH = m.n_kv_heads;
    a.hd = m.head_dim;
    a.Q = C.Q;
    a.K = C.K;
    a.V = C.V;
    a.dV = nullptr;
    a.C_cache = C.C;
    a.C_out = C.C;
    a.ex_rows = c->all_rows;
    a.ex_off = c->all_off;
    a.ap_rows = c->ap_rows;
    a.ap_off = c->zero_off;
    a.sal_rows = c->all_rows;
    a.sal_off = c->zero_off;
    a.max_rows_per_seq = c->N;
    a.scale = 1.f / sqrtf(static_cast<float>(m.head_dim));
    a.row_lo = 0;
    a.stats = c->stats;
    a.num_sms = ctx->num_sms;
    a.full_only = true;  // every row exact: Qx = the Q cache, ex_rows = identity
    a.work_ctr = ctx->attn_ctr;
    const bool fused = m.head_dim == 128 && g_attn_fused_enabled;
    a.stats_cache = fused ? C.st : nullptr;  // every row's statistics written
    a.fix = ctx->attn_fix;
    a.fix_cap = kFixCap;
    KL(ATTN, RET(attention_launch(a, st)));
    if (fused) {  // rows whose single-pass softmax could overflow (rare): two-pass recomputation
      AttnArgs f = a;
      f.mode = 1;
      KL(OTHER, RET(attention_launch(f, st)));
    }
    C.st_ok = fused;
    C.pst_ok = fused;  // every row's statistics were just computed: a new epoch
    ++C.epoch;
  return DYLLM_OK;
}

static int full_step_impl(dyllm_ctx *ctx, const dyllm_weights *w, dyllm_cache *c, const int *d_tokens) {
  if (c->m.dtype == 1) return full_step_f32(ctx, w, c, d_tokens);
  const dyllm_model_cfg &m = c->m;
  const int d = m.d_model, qw = m.n_heads * m.head_dim, kw = m.n_kv_heads * m.head_dim, rows = c->rows;
  cudaStream_t st = ctx->stream;
  ctx->cls_offset = DYLLM_KC_FULL;
  KL(OTHER, launch_embed_rows(d_tokens, nullptr, nullptr, rows, w->emb, c->H0, d, st));
  for (int l = 0; l < m.n_layers; ++l) {
    const NvtxLayer layer_range(l);
    const LayerW &L = w->L[l];
    LayerC &C = c->L[l];
    const bf16 *Hprev = l == 0 ? c->H0 : c->L[l - 1].H;
    RET(full_attn_phase(ctx, w, c, l));
    int prc = post_attention(ctx, w, c, l, nullptr, C.C, Hprev, nullptr, C.H);
    if (prc) {
      ctx->cls_offset = 0;
      return prc;
    }
  }
  ctx->cls_offset = 0;
  c->carried_valid = false;
  c->have_dec_prev = false;
  c->initialized = true;
  DY_CUDA(cudaGetLastError());
  return DYLLM_OK;
}

// Phase 1 of a sparse layer step (Alg. 3 lines 3-11): a1-a4 up to the new contexts. Returns the
// layer step's row tag and whether the attention epilogue already formed the similarity partials.
static int attn_phase(dyllm_ctx *ctx, const dyllm_weights *w, dyllm_cache *c, int l, int row_lo, const int *idx_in,
                      const int *off_in, uint32_t *tag_out, bool *fuse_cos_out) {
  const dyllm_model_cfg &m = c->m;
  const int b = c->r.batch, N = c->N, rows = c->rows;
  const int d = m.d_model, qw = m.n_heads * m.head_dim, kw = m.n_kv_heads * m.head_dim;
  const LayerW &L = w->L[l];
  LayerC &C = c->L[l];
  const bf16 *Hprev = l == 0 ? c->H0 : c->L[l - 1].H;
  cudaStream_t st = ctx->stream;
  const int *M_in = off_in + b;
  const bool fused = m.head_dim == 128 && g_attn_fused_enabled;
  const uint32_t tag = ++c->row_tag;
  // exact rows = idx_in; approximate rows = input rows \ idx_in: the fused path marks the exact
  // rows in qkv_post (row tag), the other attention kernels take an explicit approximate list
  if (!fused) KL(OTHER, launch_approx_rows(idx_in, off_in, b, N, row_lo, c->ap_rows, c->ap_off, st));
  // incremental statistics need the overwritten key rows (Kxo) and current
  // statistics; under the literal layer-1 policy, decoded rows outside idx_in get a new Q at
  // layer 0 without a statistics update, so that layer stays dense
  const bool inc = fused && g_attn_inc_enabled && C.st_ok && !(l == 0 && c->r.layer1_policy == 0);
  bf16 *Kfi = fused ? C.Kfi : nullptr;
  // (default: option 2) the fused epilogue pays where the projection runs several tiles per SM
  // pair (full-input steps, the FullStep): there its a3 work overlaps the next tiles' main loops.
  // In response-only steps each pair holds one tile, the epilogue is exposed, and a3 spread over
  // every SM as its own kernel is faster (ncu launch lists: QKV + a3 53.1 + 14.0 us unfused vs
  // 79.6 us fused at response-only size; 110.4 + 32.6 vs 128.9 us full-input)
  if (qkv_fusable(c, false) && row_lo < c->r.L_P) {
    // a1 (+ a3's row bookkeeping: exact-row tag, first write in the statistics epoch), then a2 + a3
    // in the projection's epilogue: RoPE, dV (before the overwrite), in-place K / V / Q cache rows
    RowMark mk;
    mk.rowflag = fused ? c->rowflag : nullptr;
    mk.tag = tag;
    if (Kfi) {
      mk.dtag = C.dtag;
      mk.epoch = C.epoch;
      mk.snap = c->snapm;
    }
    KL(GATHER, launch_gather_rmsnorm(Hprev, idx_in, M_in, rows, L.g_attn, m.rms_eps, c->Xn, d, st, mk));
    QkvEpi q;
    q.idx = idx_in;
    q.N = N;
    q.H = m.n_heads;
    q.KVH = m.n_kv_heads;
    q.rope_cs = c->rope_cs;
    q.Qc = C.Q;
    q.Kc = C.K;
    q.Vc = C.V;
    q.dV = c->dV;
    q.Qx = c->Qx;
    q.Kx = c->Kx;
    q.Kxo = inc ? c->Kxo : nullptr;
    q.Kfi = Kfi;
    q.snap = c->snapm;
    KL(QKV_GEMM, RET(gemm_qkv(ctx, c, M_in, c->Xn, L.wqkv, L.bqkv, q)));
  } else {
    // a1 + a2: RMSNorm(x[idx_in]) -> QKV projection of the changed rows
    KL(GATHER, launch_gather_rmsnorm(Hprev, idx_in, M_in, rows, L.g_attn, m.rms_eps, c->Xn, d, st));
    KL(QKV_GEMM, RET(gemm(ctx, M_in, rows, qw + 2 * kw, d, c->Xn, L.wqkv, c->qkv, qw + 2 * kw, EPI_BF16)));
    // a3: RoPE, dV (before overwrite), in-place K/V/Q cache rows
    KL(QKV_POST, launch_qkv_post(c->qkv, idx_in, M_in, rows, L.bqkv, N, m.n_heads, m.n_kv_heads, m.head_dim,
                                 c->rope_cs, C.Q, C.K, C.V, c->dV, c->Qx, c->Kx, inc ? c->Kxo : nullptr,
                                 fused ? c->rowflag : nullptr, tag, st, 0, Kfi, C.dtag, C.epoch));
  }
  // full-input step with current prompt statistics: the keys changed since they were current
  const bool full_in = row_lo < c->r.L_P;
  const bool pinc = fused && full_in && g_attn_inc_enabled && g_attn_pinc_enabled && C.pst_ok;
  if (pinc)
    KL(OTHER, launch_build_u(idx_in, off_in, c->rowflag, tag, C.dtag, C.epoch, C.K, C.Kfi, b, N, kw, c->urows, c->Kun,
                             c->Kuo, c->ucnt, st));
  // a4: exact rows + approximate rows (Alg. 4) -> Cn
  AttnArgs a{};
  a.batch = b;
  a.N = N;
  a.H = m.n_heads;
  a.KVH = m.n_kv_heads;
  a.hd = m.head_dim;
  a.Q = C.Q;
  a.K = C.K;
  a.V = C.V;
  a.dV = c->dV;
  a.C_cache = C.C;
  // fused kernel: the epilogue commits C_new into the C cache itself and leaves the similarity
  // partials; other head dims write C_new (exact) / dC (approximate) rows to Cn
  const bool fuse_cos = fused && g_attn_fuse_cos && !c->tp;  // tensor parallel: partials over shards
  a.C_out = fuse_cos ? C.C : c->Cn;
  a.cos_part = fuse_cos ? c->cos_part : nullptr;
  a.ex_rows = idx_in;
  a.ex_off = off_in;
  a.ap_rows = c->ap_rows;
  a.ap_off = c->ap_off;
  a.sal_rows = idx_in;
  a.sal_off = off_in;
  a.max_rows_per_seq = N - row_lo;
  a.scale = 1.f / sqrtf(static_cast<float>(m.head_dim));
  a.row_lo = row_lo;
  a.stats = c->stats;
  a.num_sms = ctx->num_sms;
  a.Qx = c->Qx;
  a.Kx = c->Kx;
  a.rowflag = c->rowflag;
  a.row_tag = tag;
  a.work_ctr = ctx->attn_ctr;
  a.stats_cache = fused ? C.st : nullptr;
  a.Kxo = c->Kxo;
  a.inc = inc;
  a.resp_lo = c->r.L_P;
  a.fix = ctx->attn_fix;
  a.fix_cap = kFixCap;
  a.Kun = c->Kun;
  a.Kuo = c->Kuo;
  a.ucnt = c->ucnt;
  a.pinc = pinc;
  KL(ATTN, RET(attention_launch(a, st)));
  if (fused) {  // tiles whose incremental update cancelled or whose single pass could overflow (rare)
    AttnArgs f = a;
    f.mode = 1;
    KL(OTHER, RET(attention_launch(f, st)));  // not an attention pass of its own (roofline accounting)
  }
  // every input row's statistics are now current (dense tiles, incremental tiles, exact rows);
  // after a full-input step that includes the prompt rows: a new epoch
  C.st_ok = fused;
  if (fused && full_in) {
    C.pst_ok = true;
    ++C.epoch;
  }
  *tag_out = tag;
  *fuse_cos_out = fuse_cos;
  return DYLLM_OK;
}

// One layer of SparseStep (Alg. 3 lines 3-16) on internal lists.
static int layer_step_impl(dyllm_ctx *ctx, const dyllm_weights *w, dyllm_cache *c, int l, int row_lo,
                           const int *idx_in, const int *off_in, float tau, int *idx_out, int *off_out, float *sim,
                           int *counts) {
  if (c->m.dtype == 1) return layer_step_f32(ctx, w, c, l, row_lo, idx_in, off_in, tau, idx_out, off_out, sim, counts);
  const dyllm_model_cfg &m = c->m;
  const int b = c->r.batch, N = c->N, rows = c->rows;
  const int qw = m.n_heads * m.head_dim;
  const LayerC &C = c->L[l];
  const bf16 *Hprev = l == 0 ? c->H0 : c->L[l - 1].H;
  cudaStream_t st = ctx->stream;
  uint32_t tag = 0;
  bool fuse_cos = false;
  RET(attn_phase(ctx, w, c, l, row_lo, idx_in, off_in, &tag, &fuse_cos));
  // a5: cosine similarity + threshold + compaction; C_cache <- Cn for the input rows
  const bool fmode = c->r.select_mode == 1;
  const bool delta = attention_writes_delta(m.head_dim);  // fused kernel: Cn = dC for approximate rows
  KL(SELECT, launch_select(c->Cn, C.C, b, N, row_lo, qw, fmode ? 2.f : tau, c->r.cmp, fmode ? tau : -1.f, idx_out,
                           off_out, (fmode && !sim) ? c->sim : sim, ctx->masks, ctx->ticket, counts,
                           delta ? c->rowflag : nullptr, tag, (delta || fuse_cos) ? off_in : nullptr, st,
                           fuse_cos ? c->cos_part : nullptr, m.n_heads));
  const int *M_out = off_out + b;
  // a6 + a7 on idx_out, a8 scatter-back into H_l (other rows keep FFN_OUT_cache)
  KL(GATHER, launch_gather_rows(C.C, idx_out, M_out, rows, c->Cg, qw, st));
  RET(post_attention(ctx, w, c, l, M_out, c->Cg, Hprev, idx_out, C.H));
  DY_CUDA(cudaGetLastError());
  return DYLLM_OK;
}

// logits of the masked rows of the active block -> unmask + commit (a9)
static int unmask_impl(dyllm_ctx *ctx, const dyllm_weights *w, dyllm_cache *c, int *d_tokens, int *d_dec_pos,
                       int *d_dec_tok) {
  const dyllm_model_cfg &m = c->m;
  const dyllm_run_cfg &r = c->r;
  cudaStream_t st = ctx->stream;
  const int lm_cap = r.batch * r.block;
  const bf16 *HL = c->L[m.n_layers - 1].H;
  KL(OTHER, launch_lm_candidates(d_tokens, r.batch, r.L_P, r.L_R, r.block, m.mask_id, c->lm_rows, c->lm_off, st));
  if (m.dtype == 1) {  // fp32-parity mode: full logits rows, then one (max, sum exp, argmax) partial per row
    const int *M_lm = c->lm_off + r.batch;
    KL(GATHER, f32::gather_rmsnorm(fp(c->L[m.n_layers - 1].H), c->lm_rows, M_lm, lm_cap, w->g_final, m.rms_eps,
                                   fp(c->Xf), m.d_model, st));
    KL(LM_GEMM, f32::gemm(g32(M_lm, lm_cap, m.vocab, m.d_model, fp(c->Xf), w->lm_head, c->logits32, m.vocab), st));
    KL(OTHER, f32::lm_reduce(c->logits32, M_lm, lm_cap, m.vocab, m.mask_id, c->partials, st));
    KL(OTHER, launch_lm_select_commit(c->partials, 1, c->lm_rows, c->lm_off, r.batch, r.n_u, d_tokens, c->dec_prev,
                                      d_dec_tok, w->emb, nullptr, m.d_model, st, fp(c->H0)));
  } else {
  KL(GATHER, launch_gather_rmsnorm(HL, c->lm_rows, c->lm_off + r.batch, lm_cap, w->g_final, m.rms_eps, c->Xf,
                                   m.d_model, st));
  KL(LM_GEMM, RET(gemm(ctx, c->lm_off + r.batch, lm_cap, m.vocab, m.d_model, c->Xf, w->lm_head, nullptr, 0, EPI_LMHEAD,
                       nullptr, 0, nullptr, nullptr, c->partials, nullptr, m.mask_id)));
  KL(OTHER, launch_lm_select_commit(c->partials, gemm_lmhead_ntiles(m.vocab), c->lm_rows, c->lm_off, r.batch, r.n_u,
                                    d_tokens, c->dec_prev, d_dec_tok, w->emb, c->H0, m.d_model, st));
  }
  if (d_dec_pos)
    DY_CUDA(cudaMemcpyAsync(d_dec_pos, c->dec_prev, sizeof(int) * r.batch * r.n_u, cudaMemcpyDeviceToDevice, st));
  c->have_dec_prev = true;
  DY_CUDA(cudaGetLastError());
  return DYLLM_OK;
}

// ------------------------------------------------------------------ ABI: steps
int dyllm_cache_init(dyllm_ctx *ctx, const dyllm_weights *w, dyllm_cache *c, const int32_t *d_tokens) {
  CHECK_ARG(ctx && w && c && d_tokens, "null argument");
  RET(sticky(ctx));
  return full_step_impl(ctx, w, c, d_tokens);
}

int dyllm_layer_step(dyllm_ctx *ctx, const dyllm_weights *w, dyllm_cache *c, int layer, int input_mode,
                     const int32_t *d_idx_in, const int32_t *d_off_in, float tau, int32_t *d_idx_out,
                     int32_t *d_off_out, float *d_sim_out) {
  CHECK_ARG(ctx && w && c && d_idx_in && d_off_in && d_idx_out && d_off_out, "null argument");
  if (layer < 0 || layer >= c->m.n_layers) {
    set_error("layer out of range");
    return DYLLM_E_INDEX;
  }
  CHECK_ARG(input_mode == DYLLM_INPUT_FULL || input_mode == DYLLM_INPUT_RESPONSE, "bad input_mode");
  if (!c->initialized) {
    set_error("cache not initialised (call dyllm_cache_init first)");
    return DYLLM_E_STATE;
  }
  RET(sticky(ctx));
  const int row_lo = input_mode == DYLLM_INPUT_FULL ? 0 : c->r.L_P;
  return layer_step_impl(ctx, w, c, layer, row_lo, d_idx_in, d_off_in, tau, d_idx_out, d_off_out, d_sim_out, nullptr);
}

}  // extern "C"

// Layer-1 list of a sparse step (Alg. 1, D5) into lst[0], and under the literal layer-1
// policy the Q-only refresh of rows decoded at t-1 (D6)
static int layer1_prepare(dyllm_ctx *ctx, const dyllm_weights *w, dyllm_cache *c, int row_lo) {
  const dyllm_run_cfg &r = c->r;
  cudaStream_t st = ctx->stream;
  // layer-1 idx_in: carried (or response rows when None) [∪ decoded rows, D5], ∩ input rows
  KL(OTHER, launch_build_list(1, c->carried_valid ? c->carried : nullptr, c->carried_off,
                              c->have_dec_prev ? c->dec_prev : nullptr, r.n_u, r.layer1_policy, r.batch, c->N, row_lo,
                              r.L_P, c->lst[0], c->lst_off[0], st));
  if (r.layer1_policy == 0 && c->have_dec_prev) {
    // literal Alg. 1: rows decoded at t-1 stay out of layer-1 idx_in unless carried, but their
    // embedding changed, so their query does too (Alg. 3 line 4 recomputes Q for every input
    // row; D6 keeps a Q cache): refresh Q alone for decoded rows outside idx_in
    const dyllm_model_cfg &m = c->m;
    const int d = m.d_model, qw = m.n_heads * m.head_dim, kw = m.n_kv_heads * m.head_dim;
    const LayerW &L0 = w->L[0];
    KL(OTHER, launch_build_list(2, c->carried_valid ? c->carried : nullptr, c->carried_off, c->dec_prev, r.n_u, 0,
                                r.batch, c->N, row_lo, r.L_P, c->qx_rows, c->qx_off, st));
    const int *M_q = c->qx_off + r.batch;
    if (m.dtype == 1) {
      KL(GATHER, f32::gather_rmsnorm(fp(c->H0), c->qx_rows, M_q, c->rows, L0.g_attn, m.rms_eps, fp(c->Xn), d, st));
      KL(QKV_GEMM, f32::gemm(g32(M_q, c->rows, qw + 2 * kw, d, fp(c->Xn), L0.wqkv, fp(c->qkv), qw + 2 * kw), st));
      KL(QKV_POST, f32::qkv_post(fp(c->qkv), c->qx_rows, M_q, c->rows, L0.bqkv, c->N, m.n_heads, m.n_kv_heads,
                                 m.head_dim, c->rope_cs, fp(c->L[0].Q), nullptr, nullptr, nullptr, 1, st));
    } else {
    KL(GATHER, launch_gather_rmsnorm(c->H0, c->qx_rows, M_q, c->rows, L0.g_attn, m.rms_eps, c->Xn, d, st));
    KL(QKV_GEMM, RET(gemm(ctx, M_q, c->rows, qw + 2 * kw, d, c->Xn, L0.wqkv, c->qkv, qw + 2 * kw, EPI_BF16)));
    KL(QKV_POST, launch_qkv_post(c->qkv, c->qx_rows, M_q, c->rows, L0.bqkv, c->N, m.n_heads, m.n_kv_heads,
                                 m.head_dim, c->rope_cs, c->L[0].Q, nullptr, nullptr, nullptr, nullptr, nullptr,
                                 nullptr, nullptr, 0u, st, 1));
    }
  }
  return DYLLM_OK;
}

extern "C" {

int dyllm_denoise_step(dyllm_ctx *ctx, const dyllm_weights *w, dyllm_cache *c, int t, const float *h_tau,
                       int32_t *d_tokens, int32_t *d_dec_pos, int32_t *d_dec_tok, int32_t *d_sal_counts) {
  CHECK_ARG(ctx && w && c && d_tokens && d_dec_tok, "null argument");
  const dyllm_run_cfg &r = c->r;
  const int T_total = (r.L_R + r.n_u - 1) / r.n_u;
  if (t < 0) {
    set_error("t < 0");
    return DYLLM_E_INDEX;
  }
  if (t >= T_total) return DYLLM_DONE;
  RET(sticky(ctx));
  cudaStream_t st = ctx->stream;
  const NvtxRange step_range(t < r.T_full ? "dyllm full step" : (t % r.full_period == 0 ? "dyllm full-input step"
                                                                                         : "dyllm response-only step"));
  if (t < r.T_full) {
    RET(full_step_impl(ctx, w, c, d_tokens));
  } else {
    CHECK_ARG(h_tau, "null tau");
    if (!c->initialized) {
      set_error("sparse step before any FullStep (T_full = 0 needs dyllm_cache_init)");
      return DYLLM_E_STATE;
    }
    const int row_lo = (t % r.full_period == 0) ? 0 : r.L_P;
    RET(layer1_prepare(ctx, w, c, row_lo));
    int cur = 0;
    for (int l = 0; l < c->m.n_layers; ++l) {
      const NvtxLayer layer_range(l);
      float *sim_tr = c->tr_sims ? c->tr_sims + static_cast<int64_t>(l) * c->rows : nullptr;
      RET(layer_step_impl(ctx, w, c, l, row_lo, c->lst[cur], c->lst_off[cur], h_tau[l], c->lst[cur ^ 1],
                          c->lst_off[cur ^ 1], sim_tr, d_sal_counts ? d_sal_counts + l * r.batch : nullptr));
      cur ^= 1;
      if (c->tr_lists) {
        DY_CUDA(cudaMemcpyAsync(c->tr_lists + static_cast<int64_t>(l) * c->rows, c->lst[cur], sizeof(int) * c->rows,
                                cudaMemcpyDeviceToDevice, st));
        DY_CUDA(cudaMemcpyAsync(c->tr_offs + static_cast<int64_t>(l) * (r.batch + 1), c->lst_off[cur],
                                sizeof(int) * (r.batch + 1), cudaMemcpyDeviceToDevice, st));
      }
    }
    DY_CUDA(cudaMemcpyAsync(c->carried, c->lst[cur], sizeof(int) * c->rows, cudaMemcpyDeviceToDevice, st));
    DY_CUDA(cudaMemcpyAsync(c->carried_off, c->lst_off[cur], sizeof(int) * (r.batch + 1), cudaMemcpyDeviceToDevice, st));
    c->carried_valid = true;
  }
  return unmask_impl(ctx, w, c, d_tokens, d_dec_pos, d_dec_tok);
}

int dyllm_full_step(dyllm_ctx *ctx, const dyllm_weights *w, dyllm_cache *c, int32_t *d_tokens, int32_t *d_dec_pos,
                    int32_t *d_dec_tok) {
  CHECK_ARG(ctx && w && c && d_tokens && d_dec_tok, "null argument");
  RET(sticky(ctx));
  const NvtxRange step_range("dyllm full step");
  RET(full_step_impl(ctx, w, c, d_tokens));
  return unmask_impl(ctx, w, c, d_tokens, d_dec_pos, d_dec_tok);
}

int dyllm_unmask(dyllm_ctx *ctx, const dyllm_weights *w, dyllm_cache *c, int32_t *d_tokens, int32_t *d_dec_pos,
                 int32_t *d_dec_tok) {
  CHECK_ARG(ctx && w && c && d_tokens && d_dec_tok, "null argument");
  if (!c->initialized) {
    set_error("cache not initialised");
    return DYLLM_E_STATE;
  }
  RET(sticky(ctx));
  return unmask_impl(ctx, w, c, d_tokens, d_dec_pos, d_dec_tok);
}

}  // extern "C"

// ------------------------------------------------------------------ tensor parallelism
// NCCL is resolved at run time (the loopback backend needs none; the torch process usually has it)
struct NcclApi {
  bool ok = false;
  decltype(&ncclGetUniqueId) get_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
};
static NcclApi &nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.get_id = reinterpret_cast<decltype(api.get_id)>(dlsym(h, "ncclGetUniqueId"));
      api.init_rank = reinterpret_cast<decltype(api.init_rank)>(dlsym(h, "ncclCommInitRank"));
      api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
      api.destroy = reinterpret_cast<decltype(api.destroy)>(dlsym(h, "ncclCommDestroy"));
      api.ok = api.get_id && api.init_rank && api.all_reduce && api.destroy;
    }
  }
  return api;
}

struct dyllm_tp {
  dyllm_ctx *ctx = nullptr;
  int world = 1, rank = 0;
  bool loopback = true;
  ncclComm_t comm = nullptr;
  std::vector<dyllm_cache *> shard;  // loopback: world shards; NCCL: this rank's
  int *h_cnt = nullptr;              // pinned: device row counts read back for NCCL
};

static void tp_forget(dyllm_tp *tp, const dyllm_cache *c) {
  for (dyllm_cache *&sh : tp->shard)
    if (sh == c) sh = nullptr;
}

// Sum of a per-shard buffer over the group, in shard order, left in every shard's buffer.
// buf_of(c): the shard's buffer; M_ptr (nullable): shard 0's device row count; width: elements per row.
template <typename F>
static int tp_reduce(dyllm_tp *tp, F buf_of, const int *M_ptr, int M_cap, int width, bool f32) {
  dyllm_ctx *ctx = tp->ctx;
  cudaStream_t st = ctx->stream;
  if (tp->loopback) {
    TpPtrs p{};
    for (int g = 0; g < tp->world; ++g) p.p[g] = buf_of(tp->shard[g]);
    KL(OTHER, launch_tp_reduce(p, tp->world, M_ptr, M_cap, width, f32 ? 1 : 0, st));
    DY_CUDA(cudaGetLastError());
    return DYLLM_OK;
  }
  int M = M_cap;
  if (M_ptr) {  // the list length lives on the device: read it back (one synchronisation)
    DY_CUDA(cudaMemcpyAsync(tp->h_cnt, M_ptr, sizeof(int), cudaMemcpyDeviceToHost, st));
    DY_CUDA(cudaStreamSynchronize(st));
    M = std::min(*tp->h_cnt, M_cap);
  }
  if (M <= 0) return DYLLM_OK;
  void *b = buf_of(tp->shard[0]);
  if (nccl_api().all_reduce(b, b, static_cast<size_t>(M) * width, f32 ? ncclFloat32 : ncclBfloat16, ncclSum, tp->comm,
                            st) != ncclSuccess) {
    set_error("ncclAllReduce failed");
    return DYLLM_E_NCCL;
  }
  return DYLLM_OK;
}

// O projection + FFN of a shard on the rows (rows, M_ptr) (nullptr: all rows), with the group's
// all-reduces: h = x + sum_g C_g W_o,g (shard 0 adds x), out = h + sum_g FFN_g(RMSNorm(h)) (shard 0
// adds h); residual_mode 1 (paper_literal): h = RMSNorm(sum_g C_g W_o,g), out = sum_g FFN_g(h).
// A_c(c): the shard's context rows (contiguous, aligned with rows); out rows land in H_l at `rows`.
// rows_of(c) -> RowList{row ids, device count}: the shard's list (ignored when all_rows)
struct RowList {
  const int *rows;
  const int *count;
};
template <typename FA, typename FR>
static int tp_post_attention(dyllm_tp *tp, const dyllm_weights *const *W, int l, FA A_c, FR rows_of, bool all_rows) {
  const int G = static_cast<int>(tp->shard.size());
  dyllm_ctx *ctx = tp->ctx;
  cudaStream_t st = ctx->stream;
  dyllm_cache *c0 = tp->shard[0];
  const dyllm_model_cfg &m0 = c0->m;
  const int d = m0.d_model, R = c0->rows, b = c0->r.batch;
  const bool res = m0.residual_mode == 0;
  for (int i = 0; i < G; ++i) {
    dyllm_cache *c = tp->shard[i];
    const dyllm_model_cfg &m = c->m;
    const int qw = m.n_heads * m.head_dim;
    const bool first = (tp->loopback ? i : tp->rank) == 0;
    const RowList rl = rows_of(c);
    const int *rows = all_rows ? nullptr : rl.rows;
    const int *M_ptr = all_rows ? nullptr : rl.count;
    const bf16 *Hprev = l == 0 ? c->H0 : c->L[l - 1].H;
    KL(O_GEMM, RET(gemm(ctx, M_ptr, R, d, qw, A_c(c), W[i]->L[l].wo, c->h, d, (res && first) ? EPI_RESID : EPI_BF16,
                        Hprev, d, rows)));
  }
  RET(tp_reduce(tp, [](dyllm_cache *c) { return static_cast<void *>(c->h); },
                all_rows ? nullptr : rows_of(c0).count, R, d, false));
  for (int i = 0; i < G; ++i) {
    dyllm_cache *c = tp->shard[i];
    const dyllm_model_cfg &m = c->m;
    const int F = m.d_ff;
    const bool first = (tp->loopback ? i : tp->rank) == 0;
    const int *M_ptr = all_rows ? nullptr : rows_of(c).count;
    const LayerW &L = W[i]->L[l];
    KL(OTHER, launch_rmsnorm_rows(c->h, M_ptr, R, L.g_ffn, m.rms_eps, c->hn, d, st));
    KL(GU_GEMM, RET(gemm(ctx, M_ptr, R, 2 * F, d, c->hn, L.wgu, c->act, F, EPI_SWIGLU)));
    bf16 *out = all_rows ? c->L[l].H : c->ffo;
    KL(DOWN_GEMM, RET(gemm(ctx, M_ptr, R, d, F, c->act, L.wd, out, d, (res && first) ? EPI_RESID : EPI_BF16, c->h, d)));
  }
  RET(tp_reduce(tp, [l, all_rows](dyllm_cache *c) { return static_cast<void *>(all_rows ? c->L[l].H : c->ffo); },
                all_rows ? nullptr : rows_of(c0).count, R, d, false));
  if (!all_rows)  // scatter-back of the summed rows: rows outside the list keep their output
    for (int i = 0; i < G; ++i) {
      dyllm_cache *c = tp->shard[i];
      const RowList rl = rows_of(c);
      KL(OTHER, launch_scatter_rows(c->ffo, rl.rows, rl.count, R, c->L[l].H, d, st));
    }
  (void)b;
  return DYLLM_OK;
}

static int tp_full_step(dyllm_tp *tp, const dyllm_weights *const *W, const int *d_tokens) {
  const int G = static_cast<int>(tp->shard.size());
  dyllm_ctx *ctx = tp->ctx;
  const int nl = tp->shard[0]->m.n_layers;
  ctx->cls_offset = DYLLM_KC_FULL;
  for (int i = 0; i < G; ++i) {
    dyllm_cache *c = tp->shard[i];
    KL(OTHER, launch_embed_rows(d_tokens, nullptr, nullptr, c->rows, W[i]->emb, c->H0, c->m.d_model, ctx->stream));
  }
  int rc = DYLLM_OK;
  for (int l = 0; l < nl && rc == DYLLM_OK; ++l) {
    for (int i = 0; i < G && rc == DYLLM_OK; ++i) rc = full_attn_phase(ctx, W[i], tp->shard[i], l);
    if (rc == DYLLM_OK)
      rc = tp_post_attention(tp, W, l, [l](dyllm_cache *c) { return static_cast<const bf16 *>(c->L[l].C); },
                             [](dyllm_cache *) { return RowList{nullptr, nullptr}; }, true);
  }
  ctx->cls_offset = 0;
  RET(rc);
  for (dyllm_cache *c : tp->shard) {
    c->carried_valid = false;
    c->have_dec_prev = false;
    c->initialized = true;
  }
  DY_CUDA(cudaGetLastError());
  return DYLLM_OK;
}

// One sparse layer of the group: a1-a4 per shard, similarity partials summed over the shards,
// the same threshold / compaction on every shard, then O projection and FFN with their all-reduces.
static int tp_layer_step(dyllm_tp *tp, const dyllm_weights *const *W, int l, int row_lo, int cur, float tau,
                         int *counts) {
  const int G = static_cast<int>(tp->shard.size());
  dyllm_ctx *ctx = tp->ctx;
  cudaStream_t st = ctx->stream;
  dyllm_cache *c0 = tp->shard[0];
  const int b = c0->r.batch, N = c0->N, R = c0->rows;
  const bool fmode = c0->r.select_mode == 1;
  std::vector<uint32_t> tags(G);
  for (int i = 0; i < G; ++i) {
    dyllm_cache *c = tp->shard[i];
    const dyllm_model_cfg &m = c->m;
    bool fc = false;
    RET(attn_phase(ctx, W[i], c, l, row_lo, c->lst[cur], c->lst_off[cur], &tags[i], &fc));
    const bool delta = attention_writes_delta(m.head_dim);
    // this shard's partial sums (dot, |C_new|^2, |C_old|^2) per input row; C_cache <- C_new
    KL(SELECT, launch_select(c->Cn, c->L[l].C, b, N, row_lo, m.n_heads * m.head_dim, 2.f, c->r.cmp, -1.f, nullptr,
                             nullptr, nullptr, ctx->masks, ctx->ticket, nullptr, delta ? c->rowflag : nullptr, tags[i],
                             delta ? c->lst_off[cur] : nullptr, st, nullptr, 0, c->tp_part));
  }
  RET(tp_reduce(tp, [](dyllm_cache *c) { return static_cast<void *>(c->tp_part); }, nullptr, R, 4, true));
  for (int i = 0; i < G; ++i) {
    dyllm_cache *c = tp->shard[i];
    float *sim_tr = c->tr_sims ? c->tr_sims + static_cast<int64_t>(l) * c->rows : nullptr;
    // identical sums on every shard: identical similarities, thresholds and lists
    KL(SELECT, launch_select(nullptr, nullptr, b, N, row_lo, 8, fmode ? 2.f : tau, c->r.cmp, fmode ? tau : -1.f,
                             c->lst[cur ^ 1], c->lst_off[cur ^ 1], (fmode && !sim_tr) ? c->sim : sim_tr, ctx->masks,
                             ctx->ticket, i == 0 ? counts : nullptr, nullptr, 0u, c->lst_off[cur], st, c->tp_part, 1));
    const dyllm_model_cfg &m = c->m;
    KL(GATHER, launch_gather_rows(c->L[l].C, c->lst[cur ^ 1], c->lst_off[cur ^ 1] + b, R, c->Cg,
                                  m.n_heads * m.head_dim, st));
    if (c->tr_lists) {  // dyllm_cache_set_trace on a shard: its per-layer lists
      DY_CUDA(cudaMemcpyAsync(c->tr_lists + static_cast<int64_t>(l) * c->rows, c->lst[cur ^ 1], sizeof(int) * c->rows,
                              cudaMemcpyDeviceToDevice, st));
      DY_CUDA(cudaMemcpyAsync(c->tr_offs + static_cast<int64_t>(l) * (b + 1), c->lst_off[cur ^ 1], sizeof(int) * (b + 1),
                              cudaMemcpyDeviceToDevice, st));
    }
  }
  return tp_post_attention(tp, W, l, [](dyllm_cache *c) { return static_cast<const bf16 *>(c->Cg); },
                           [cur](dyllm_cache *c) { return RowList{c->lst[cur ^ 1], c->lst_off[cur ^ 1] + c->r.batch}; }, false);
}

extern "C" {

int dyllm_tp_unique_id(void *h_out, int n_bytes) {
  CHECK_ARG(h_out && n_bytes >= static_cast<int>(sizeof(ncclUniqueId)), "need a 128-byte buffer");
  NcclApi &api = nccl_api();
  if (!api.ok) {
    set_error("libnccl.so.2 not found");
    return DYLLM_E_NCCL;
  }
  ncclUniqueId id;
  if (api.get_id(&id) != ncclSuccess) {
    set_error("ncclGetUniqueId failed");
    return DYLLM_E_NCCL;
  }
  std::memcpy(h_out, &id, sizeof(id));
  return DYLLM_OK;
}

int dyllm_tp_create(dyllm_ctx *ctx, int world, int rank, const void *nccl_unique_id, dyllm_tp **out) {
  CHECK_ARG(ctx && out, "null argument");
  CHECK_ARG(world >= 1 && world <= kTpMax, "world out of range (1..8)");
  dyllm_tp *tp = new dyllm_tp();
  tp->ctx = ctx;
  tp->world = world;
  tp->loopback = nccl_unique_id == nullptr;
  tp->rank = tp->loopback ? 0 : rank;
  if (!tp->loopback) {
    if (rank < 0 || rank >= world) {
      delete tp;
      set_error("rank out of range");
      return DYLLM_E_ARG;
    }
    NcclApi &api = nccl_api();
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof(id));
    if (!api.ok || api.init_rank(&tp->comm, world, id, rank) != ncclSuccess) {
      delete tp;
      set_error(api.ok ? "ncclCommInitRank failed" : "libnccl.so.2 not found");
      return DYLLM_E_NCCL;
    }
    if (cudaMallocHost(&tp->h_cnt, sizeof(int)) != cudaSuccess) {
      api.destroy(tp->comm);
      delete tp;
      set_error("cudaMallocHost failed");
      return DYLLM_E_NOMEM;
    }
  }
  tp->shard.assign(tp->loopback ? world : 1, nullptr);
  *out = tp;
  return DYLLM_OK;
}

int dyllm_tp_attach(dyllm_tp *tp, int shard, dyllm_cache *c) {
  CHECK_ARG(tp && c, "null argument");
  const int slot = tp->loopback ? shard : 0;
  if (shard < 0 || shard >= tp->world || (!tp->loopback && shard != tp->rank)) {
    set_error("shard out of range (NCCL: shard must be the rank)");
    return DYLLM_E_INDEX;
  }
  if (c->m.dtype != 0) {
    set_error("tensor parallelism: bf16 caches only");
    return DYLLM_E_ARG;
  }
  for (dyllm_cache *o : tp->shard)
    if (o && (o->m.d_model != c->m.d_model || o->m.n_layers != c->m.n_layers || o->m.n_heads != c->m.n_heads ||
              o->m.n_kv_heads != c->m.n_kv_heads || o->m.d_ff != c->m.d_ff || o->N != c->N ||
              o->r.batch != c->r.batch || o->m.residual_mode != c->m.residual_mode)) {
      set_error("tensor parallelism: shard shapes differ");
      return DYLLM_E_SHAPE;
    }
  if (!c->tp_part) {
    RET(dalloc_t(c->allocs, &c->tp_part, c->rows));
    RET(dalloc_t(c->allocs, &c->tp_tokens, c->rows + static_cast<int64_t>(c->r.batch) * c->r.n_u));
  }
  c->tp = tp;
  c->tp_shard = shard;
  tp->shard[slot] = c;
  return DYLLM_OK;
}

static int tp_check(dyllm_tp *tp, const dyllm_weights *const *w) {
  CHECK_ARG(tp && w, "null argument");
  for (size_t i = 0; i < tp->shard.size(); ++i) {
    if (!tp->shard[i] || !w[i]) {
      set_error("tensor parallelism: every local shard needs a cache and weights");
      return DYLLM_E_STATE;
    }
  }
  return sticky(tp->ctx);
}

int dyllm_tp_cache_init(dyllm_tp *tp, const dyllm_weights *const *w, const int32_t *d_tokens) {
  CHECK_ARG(d_tokens, "null tokens");
  RET(tp_check(tp, w));
  return tp_full_step(tp, w, d_tokens);
}

int dyllm_tp_denoise_step(dyllm_tp *tp, const dyllm_weights *const *w, int t, const float *h_tau, int32_t *d_tokens,
                          int32_t *d_dec_pos, int32_t *d_dec_tok, int32_t *d_sal_counts) {
  CHECK_ARG(d_tokens && d_dec_tok, "null argument");
  RET(tp_check(tp, w));
  dyllm_ctx *ctx = tp->ctx;
  cudaStream_t st = ctx->stream;
  const int G = static_cast<int>(tp->shard.size());
  dyllm_cache *c0 = tp->shard[0];
  const dyllm_run_cfg &r = c0->r;
  const int T_total = (r.L_R + r.n_u - 1) / r.n_u;
  if (t < 0) {
    set_error("t < 0");
    return DYLLM_E_INDEX;
  }
  if (t >= T_total) return DYLLM_DONE;
  if (t < r.T_full) {
    RET(tp_full_step(tp, w, d_tokens));
  } else {
    CHECK_ARG(h_tau, "null tau");
    for (dyllm_cache *c : tp->shard)
      if (!c->initialized) {
        set_error("sparse step before any FullStep");
        return DYLLM_E_STATE;
      }
    const int row_lo = (t % r.full_period == 0) ? 0 : r.L_P;
    for (int i = 0; i < G; ++i) RET(layer1_prepare(ctx, w[i], tp->shard[i], row_lo));
    int cur = 0;
    for (int l = 0; l < c0->m.n_layers; ++l) {
      RET(tp_layer_step(tp, w, l, row_lo, cur, h_tau[l], d_sal_counts ? d_sal_counts + l * r.batch : nullptr));
      cur ^= 1;
    }
    for (dyllm_cache *c : tp->shard) {
      DY_CUDA(cudaMemcpyAsync(c->carried, c->lst[cur], sizeof(int) * c->rows, cudaMemcpyDeviceToDevice, st));
      DY_CUDA(cudaMemcpyAsync(c->carried_off, c->lst_off[cur], sizeof(int) * (r.batch + 1), cudaMemcpyDeviceToDevice,
                              st));
      c->carried_valid = true;
    }
  }
  // unmasking: every shard decides on the same (bit-identical) H_L and the same tokens
  for (int i = 1; i < G; ++i)
    DY_CUDA(cudaMemcpyAsync(tp->shard[i]->tp_tokens, d_tokens, sizeof(int32_t) * c0->rows, cudaMemcpyDeviceToDevice,
                            st));
  RET(unmask_impl(ctx, w[0], c0, d_tokens, d_dec_pos, d_dec_tok));
  for (int i = 1; i < G; ++i) {
    dyllm_cache *c = tp->shard[i];
    RET(unmask_impl(ctx, w[i], c, c->tp_tokens, nullptr, c->tp_tokens + c->rows));
  }
  return DYLLM_OK;
}

void dyllm_tp_destroy(dyllm_tp *tp) {
  if (!tp) return;
  for (dyllm_cache *c : tp->shard)
    if (c) c->tp = nullptr;
  if (tp->comm) nccl_api().destroy(tp->comm);
  if (tp->h_cnt) cudaFreeHost(tp->h_cnt);
  delete tp;
}

// ------------------------------------------------------------------ ABI: instrumentation
int dyllm_ctx_profile(dyllm_ctx *ctx, int enable) {
  CHECK_ARG(ctx, "null ctx");
  if (enable) {
    DY_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->recs.clear();
    ctx->pool_next = 0;
  }
  ctx->prof = enable != 0;
  return DYLLM_OK;
}

int dyllm_ctx_profile_read(dyllm_ctx *ctx, int kclass, float *h_ms, int max_n) {
  CHECK_ARG(ctx, "null ctx");
  DY_CUDA(cudaStreamSynchronize(ctx->stream));
  int n = 0;
  for (const ProfRec &r : ctx->recs) {
    if (r.cls != kclass) continue;
    if (h_ms && n < max_n) {
      float ms = 0.f;
      DY_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
      h_ms[n] = ms;
    }
    ++n;
  }
  return n;
}

uint64_t dyllm_launch_count(void) { return g_launches.load(); }

int dyllm_set_option(int option, int value) {
  if (option == DYLLM_OPT_SKINNY_GEMM) {
    const int prev = g_skinny_enabled ? 1 : 0;
    g_skinny_enabled = value != 0;
    return prev;
  }
  if (option == DYLLM_OPT_ATTN_FUSED) {
    const int prev = g_attn_fused_enabled ? 1 : 0;
    g_attn_fused_enabled = value != 0;
    return prev;
  }
  if (option == DYLLM_OPT_SKINNY_ONE_CHUNK) {
    const int prev = g_skinny_one_chunk;
    g_skinny_one_chunk = value < 0 ? 0 : value;
    return prev;
  }
  if (option == DYLLM_OPT_PDL) {
    const int prev = g_pdl_enabled ? 1 : 0;
    g_pdl_enabled = value != 0;
    return prev;
  }
  if (option == DYLLM_OPT_ATTN_INC) {
    const int prev = g_attn_inc_enabled ? 1 : 0;
    g_attn_inc_enabled = value != 0;
    return prev;
  }
  if (option == DYLLM_OPT_ATTN_PINC) {
    const int prev = g_attn_pinc_enabled ? 1 : 0;
    g_attn_pinc_enabled = value != 0;
    return prev;
  }
  if (option == DYLLM_OPT_SKINNY_CHUNK) {
    const int prev = g_skinny_chunk_rows;
    g_skinny_chunk_rows = value < 0 ? 0 : value;
    return prev;
  }
  if (option == DYLLM_OPT_SKINNY_KB) {
    const int prev = g_skinny_kb;
    g_skinny_kb = value == 64 ? 64 : 0;
    return prev;
  }
  if (option == DYLLM_OPT_SKINNY_DEBUG) {
    const int prev = g_skinny_dbg;
    g_skinny_dbg = value & 15;
    return prev;
  }
  if (option == DYLLM_OPT_SKINNY_KROT) {
    const int prev = g_skinny_krot;
    g_skinny_krot = value < 0 ? 0 : value;
    return prev;
  }
  if (option == DYLLM_OPT_QKV_FUSED) {
    const int prev = g_qkv_fused;
    g_qkv_fused = value < 0 ? 0 : value > 2 ? 2 : value;
    return prev;
  }
  if (option == DYLLM_OPT_ATTN_COS) {
    const int prev = g_attn_fuse_cos ? 1 : 0;
    g_attn_fuse_cos = value != 0;
    return prev;
  }
  if (option == DYLLM_OPT_ATTN_T4) {
    const int prev = g_attn_t4_rows;
    g_attn_t4_rows = value < 0 ? 0 : (value > 32 ? 32 : value);
    return prev;
  }
  if (option == DYLLM_OPT_SKINNY_SPLIT) {
    const int prev = g_skinny_split;
    g_skinny_split = value < 0 ? 0 : value;
    return prev;
  }
  set_error("unknown option");
  return DYLLM_E_ARG;
}

int dyllm_debug_trace_buffer(int which, void *d_buf) {
  if (which == 0) {
    g_skinny_trace = static_cast<unsigned long long *>(d_buf);
    return DYLLM_OK;
  }
  if (which == 1) {
    g_attn_trace = static_cast<unsigned long long *>(d_buf);
    return DYLLM_OK;
  }
  if (which == 2) {
    g_attn_events = static_cast<unsigned long long *>(d_buf);
    return DYLLM_OK;
  }
  if (which == 3) {
    g_sel_trace = static_cast<unsigned long long *>(d_buf);
    return DYLLM_OK;
  }
  set_error("unknown trace buffer");
  return DYLLM_E_ARG;
}

// ------------------------------------------------------------------ ABI: cache access
// device pointer, element count and element size of one cache tensor (no side effects)
static int tensor_ptr(const dyllm_cache *c, int layer, int which, void **d_ptr, int64_t *n_elems, int *elem_bytes) {
  CHECK_ARG(c && d_ptr, "null argument");
  const int64_t rows = c->rows, d = c->m.d_model, qw = static_cast<int64_t>(c->m.n_heads) * c->m.head_dim,
                kw = static_cast<int64_t>(c->m.n_kv_heads) * c->m.head_dim;
  int eb = c->es;
  int64_t n = 0;
  if (which == DYLLM_H) {
    if (layer < 0 || layer > c->m.n_layers) {
      set_error("layer out of range");
      return DYLLM_E_INDEX;
    }
    *d_ptr = layer == 0 ? c->H0 : c->L[layer - 1].H;
    n = rows * d;
  } else {
    if (layer < 0 || layer >= c->m.n_layers || which < 0 || which > DYLLM_STATS) {
      set_error("layer/which out of range");
      return DYLLM_E_INDEX;
    }
    const LayerC &L = c->L[layer];
    switch (which) {
      case DYLLM_K: *d_ptr = L.K; n = rows * kw; break;
      case DYLLM_V: *d_ptr = L.V; n = rows * kw; break;
      case DYLLM_Q: *d_ptr = L.Q; n = rows * qw; break;
      case DYLLM_C: *d_ptr = L.C; n = rows * qw; break;
      default:
        if (!L.st) {
          set_error("no softmax statistics for this head_dim");
          return DYLLM_E_STATE;
        }
        *d_ptr = L.st;
        n = rows * c->m.n_heads;
        eb = 8;
        break;
    }
  }
  if (n_elems) *n_elems = n;
  if (elem_bytes) *elem_bytes = eb;
  return DYLLM_OK;
}

int dyllm_cache_tensor(const dyllm_cache *c, int layer, int which, void **d_ptr, int64_t *n_elems) {
  RET(tensor_ptr(c, layer, which, d_ptr, n_elems, nullptr));
  // K / Q / statistics handed out writable: the incremental softmax statistics of that layer can
  // no longer be trusted until the next dense pass (a denoising step, or dyllm_cache_refresh_stats)
  if (which == DYLLM_K || which == DYLLM_Q || which == DYLLM_STATS) c->L[layer].st_ok = c->L[layer].pst_ok = false;
  return DYLLM_OK;
}

int dyllm_cache_copy(dyllm_ctx *ctx, dyllm_cache *c, int layer, int which, void *ptr, int ptr_on_device, int export_) {
  CHECK_ARG(ctx && c && ptr, "null argument");
  void *dp = nullptr;
  int64_t n = 0;
  int eb = 2;
  RET(tensor_ptr(c, layer, which, &dp, &n, &eb));
  const cudaMemcpyKind k = export_ ? (ptr_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost)
                                   : (ptr_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice);
  if (export_) {  // read-only: the incremental statistics stay valid
    DY_CUDA(cudaMemcpyAsync(ptr, dp, n * eb, k, ctx->stream));
    return DYLLM_OK;
  }
  DY_CUDA(cudaMemcpyAsync(dp, ptr, n * eb, k, ctx->stream));
  c->initialized = true;
  // imported K / Q invalidate the statistics; imported statistics are the caller's claim that
  // they belong to the current K and Q
  if (which == DYLLM_K || which == DYLLM_Q) c->L[layer].st_ok = c->L[layer].pst_ok = false;
  if (which == DYLLM_STATS) {  // every row's statistics, current for the present K: a new epoch
    c->L[layer].st_ok = c->L[layer].pst_ok = true;
    ++c->L[layer].epoch;
  }
  return DYLLM_OK;
}

int dyllm_cache_set_decoded(dyllm_ctx *ctx, dyllm_cache *c, const int32_t *d_dec) {
  CHECK_ARG(ctx && c, "null argument");
  if (!d_dec) {
    c->have_dec_prev = false;
    return DYLLM_OK;
  }
  DY_CUDA(cudaMemcpyAsync(c->dec_prev, d_dec, sizeof(int) * c->r.batch * c->r.n_u, cudaMemcpyDeviceToDevice,
                          ctx->stream));
  c->have_dec_prev = true;
  return DYLLM_OK;
}

int dyllm_cache_set_trace(dyllm_ctx *ctx, dyllm_cache *c, int32_t *d_lists, int32_t *d_offs, float *d_sims) {
  CHECK_ARG(ctx && c, "null argument");
  CHECK_ARG((d_lists == nullptr) == (d_offs == nullptr), "d_lists and d_offs go together");
  c->tr_lists = d_lists;
  c->tr_offs = d_offs;
  c->tr_sims = d_sims;
  return DYLLM_OK;
}

int dyllm_cache_set_carried(dyllm_ctx *ctx, dyllm_cache *c, const int32_t *d_idx, const int32_t *d_off) {
  CHECK_ARG(ctx && c, "null argument");
  if (!d_idx || !d_off) {
    c->carried_valid = false;
    return DYLLM_OK;
  }
  DY_CUDA(cudaMemcpyAsync(c->carried_off, d_off, sizeof(int) * (c->r.batch + 1), cudaMemcpyDeviceToDevice, ctx->stream));
  DY_CUDA(cudaMemcpyAsync(c->carried, d_idx, sizeof(int) * c->rows, cudaMemcpyDeviceToDevice, ctx->stream));
  c->carried_valid = true;
  return DYLLM_OK;
}

int dyllm_cache_refresh_stats(dyllm_ctx *ctx, dyllm_cache *c, int layer) {
  CHECK_ARG(ctx && c, "null argument");
  if (layer < 0 || layer >= c->m.n_layers) {
    set_error("layer out of range");
    return DYLLM_E_INDEX;
  }
  RET(sticky(ctx));
  const dyllm_model_cfg &m = c->m;
  LayerC &C = c->L[layer];
  if (m.head_dim != 128 || !g_attn_fused_enabled || !C.st) return DYLLM_OK;  // no incremental path
  AttnArgs a{};
  a.batch = c->r.batch;
  a.N = c->N;
  a.H = m.n_heads;
  a.KVH = m.n_kv_heads;
  a.hd = m.head_dim;
  a.Q = C.Q;
  a.K = C.K;
  a.V = C.V;
  a.C_cache = C.C;
  a.C_out = c->Cn;
  a.ex_rows = c->all_rows;
  a.ex_off = c->zero_off;   // no salient key: no P pass, no output, statistics only
  a.ap_rows = c->ap_rows;
  a.ap_off = c->zero_off;
  a.sal_rows = c->all_rows;
  a.sal_off = c->zero_off;
  a.max_rows_per_seq = 0;
  a.scale = 1.f / sqrtf(static_cast<float>(m.head_dim));
  a.row_lo = 0;
  a.num_sms = ctx->num_sms;
  a.rowflag = c->rowflag;
  a.work_ctr = ctx->attn_ctr;
  a.stats_cache = C.st;
  a.fix = ctx->attn_fix;
  a.fix_cap = kFixCap;
  a.mode = 2;
  KL(ATTN, RET(attention_launch(a, ctx->stream)));
  C.st_ok = C.pst_ok = true;
  ++C.epoch;
  DY_CUDA(cudaGetLastError());
  return DYLLM_OK;
}

// ------------------------------------------------------------------ ABI: kernel-level calls
int dyllm_select_salient(dyllm_ctx *ctx, int batch, int N, int row_lo, int width, const void *d_c_new,
                         void *d_c_cache, float tau, int cmp, int32_t *d_idx_out, int32_t *d_off_out,
                         float *d_sim_out) {
  CHECK_ARG(ctx && d_c_new && d_c_cache && d_idx_out && d_off_out, "null argument");
  CHECK_ARG(batch >= 1 && batch <= 1024 && N >= 1 && row_lo >= 0 && row_lo < N && width >= 8 && width % 8 == 0 &&
                (cmp == 0 || cmp == 1),
            "select_salient: bad shape");
  const int64_t words = static_cast<int64_t>(batch) * ((N - row_lo + 31) / 32);
  CHECK_ARG(words <= kMaskCap, "select_salient: too many rows");
  RET(sticky(ctx));
  KL(SELECT, launch_select(static_cast<const bf16 *>(d_c_new), static_cast<bf16 *>(d_c_cache), batch, N, row_lo, width,
                           tau, cmp, -1.f, d_idx_out, d_off_out, d_sim_out, ctx->masks, ctx->ticket, nullptr, nullptr,
                           0u, nullptr, ctx->stream));
  DY_CUDA(cudaGetLastError());
  return DYLLM_OK;
}

int dyllm_gemm_bf16(dyllm_ctx *ctx, const int32_t *d_M, int M_cap, int N, int K, const void *d_A, const void *d_W,
                    void *d_D, const void *d_resid, const void *d_bias) {
  CHECK_ARG(ctx && d_A && d_W && d_D && M_cap > 0 && N > 0 && K > 0, "null argument");
  RET(sticky(ctx));
  KScope ks(ctx, DYLLM_KC_OTHER);
  return gemm(ctx, d_M, M_cap, N, K, static_cast<const bf16 *>(d_A), static_cast<const bf16 *>(d_W),
              static_cast<bf16 *>(d_D), N, d_resid ? EPI_RESID : EPI_BF16, static_cast<const bf16 *>(d_resid), N,
              nullptr, static_cast<const bf16 *>(d_bias));
}

}  // extern "C"
