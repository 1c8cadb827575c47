// internal.h — host-side internals shared by the libdyllm translation units.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

#include "../../include/dyllm.h"

typedef __nv_bfloat16 bf16;

namespace dy {

void set_error(const std::string &msg);

#define DY_CUDA(expr)                                                                              \
  do {                                                                                             \
    cudaError_t _e = (expr);                                                                       \
    if (_e != cudaSuccess) {                                                                       \
      ::dy::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e) + " @" + __FILE__ + ":" + \
                      std::to_string(__LINE__));                                                   \
      return DYLLM_E_CUDA;                                                                         \
    }                                                                                              \
  } while (0)

// ------------------------------------------------------------------ launches
extern bool g_pdl_enabled;  // programmatic dependent launch for every kernel (dyllm_set_option)
// kern<<<grid, block, smem, st>>>(args...) with programmatic stream serialisation (+ an optional
// cluster shape): the kernel may begin while its predecessor drains; it calls pdl_wait() first.
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int cluster_x,
                     Args &&...args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int n = 0;
  if (g_pdl_enabled) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster_x > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = cluster_x;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// launch from a void helper: a failing runtime call also sets the runtime's last error, which every
// ABI entry point checks (sticky) and every step checks at its end (cudaGetLastError)
#define DY_CUDA_LAUNCH(expr) static_cast<void>(expr)

// ------------------------------------------------------------------ GEMM (gemm.cu)
enum Epi { EPI_BF16 = 0, EPI_RESID = 1, EPI_SWIGLU = 2, EPI_LMHEAD = 3, EPI_QKV = 4 };
// EPI_QKV (skinny kernel, head_dim 128): the QKV projection's epilogue does a3 itself (SURVEY §8
// rows a2 + a3: RoPE at global positions, bias, dV before the overwrite, in-place Q / K / V cache
// rows, the compact copies the attention reads); each CTA's 128 weight rows are one head
struct QkvEpi {
  const int *idx = nullptr;     // row id of each output row (nullable: identity, the FullStep)
  int N = 0, H = 0, KVH = 0;    // sequence length (position = row id % N), query / kv heads
  const float2 *rope_cs = nullptr;  // [N][64] (cos, sin)
  bf16 *Qc = nullptr, *Kc = nullptr, *Vc = nullptr;  // caches [rows][H * 128] / [rows][KVH * 128]
  bf16 *dV = nullptr;           // nullable [M][KVH * 128]: V_new - V_cache (compact)
  bf16 *Qx = nullptr, *Kx = nullptr;  // nullable compact copies of the new Q / K rows
  bf16 *Kxo = nullptr;          // nullable compact copy of the overwritten K rows
  bf16 *Kfi = nullptr;          // nullable: overwritten K rows kept at their row id where snap[m]
  const uint8_t *snap = nullptr;  // [M] first write of the row in its statistics epoch (a1, RowMark)
};
// gate/up rows of W_gu are interleaved in blocks of kGuIl rows ([gate x64][up x64] ...), so a
// 128-row weight tile holds the gate and up rows of the same 64 FFN channels.
constexpr int kGuIl = 64;

struct GemmCall {
  const int *M_ptr = nullptr;  // device row count (nullable -> M_cap)
  int M_cap = 0;               // capacity rows of A (and of D)
  int N = 0;                   // rows of W (for SWIGLU: 2*F interleaved rows)
  int K = 0;
  const bf16 *A = nullptr;     // [M_cap][K]
  const bf16 *W = nullptr;     // [N][K]
  bf16 *D = nullptr;           // output (EPI_BF16/RESID: [M][ldd]; SWIGLU: [M][ldd] with N/2 cols)
  int ldd = 0;
  const bf16 *resid = nullptr; // EPI_RESID: residual rows
  int ldr = 0;
  const int *resid_rows = nullptr;  // nullable: residual row index per output row
  const int *out_rows = nullptr;    // nullable: destination row of each output row in D (scatter)
  const bf16 *bias = nullptr;       // nullable [N]
  float4 *partials = nullptr;       // EPI_LMHEAD: [M_cap][n_tiles] (max, sumexp, argmax, 0)
  int epi = EPI_BF16;
  int m_skip_le = 0;  // standard kernel: do nothing when the device row count is <= this
  int excl_col = -1;  // EPI_LMHEAD: column excluded from the max / argmax (the mask token, D22)
  float *ws = nullptr;  // skinny split-K workspace (skinny_ws_floats(num_sms) floats per ctx)
  int *ctr = nullptr;   // skinny split-K counters (kSkinnyCtrCap, zero between launches)
  QkvEpi qkv;           // EPI_QKV
};
int gemm_launch(const GemmCall &g, int num_sms, cudaStream_t st);
// 2D bf16 tensor map [rows][K] (K contiguous), box {64, box_rows}, SWIZZLE_128B
int make_tmap(CUtensorMap *m, const void *ptr, int rows, int K, int box_rows);
// 3D box {64, box_rows, box_chunks} over [rows][K]: box_chunks 64-column chunks in one TMA op
int make_tmap3(CUtensorMap *m, const void *ptr, int rows, int K, int box_rows, int box_chunks);
int gemm_lmhead_ntiles(int N);
bool skinny_eligible(const GemmCall &g);
constexpr int kSkinnyMaxM = 16384;  // skinny kernel: device row counts 1..16384 (standard kernel above)
constexpr int kSkinnyCtrCap = 4096;  // 2 counters per skinny tile (weight block x activation chunk)
inline int64_t skinny_ws_floats(int num_sms) { return static_cast<int64_t>(num_sms) * 512 * 256; }
extern bool g_skinny_enabled;  // test hook (dyllm_set_option)
extern unsigned long long *g_skinny_trace;
extern int g_skinny_split;
extern int g_skinny_kb;          // skinny k-block width: 0 / 128 or 64 (dyllm_set_option)
extern int g_skinny_dbg;         // measurement hook: 1 no operand loads, 2 no MMAs
extern int g_skinny_krot;        // k-block start offset per weight block (dyllm_set_option)
extern int g_skinny_chunk_rows;  // test hook: largest rows per activation chunk (dyllm_set_option)
extern int g_skinny_one_chunk;  // test hook: largest M in one activation chunk (dyllm_set_option)  // test hook: units per weight block (0 = auto)  // debug hook (dyllm_debug_trace_buffer)
int gemm_skinny_launch(const GemmCall &g, int num_sms, cudaStream_t st);  // gemm_skinny.cu

// ------------------------------------------------------------------ kernels (kernels.cu)
struct AttnArgs {
  int batch, N, H, KVH, hd;
  const bf16 *Q;          // [b][N][H*hd]
  const bf16 *K, *V;      // [b][N][KVH*hd]
  const bf16 *dV;         // [M_in][KVH*hd] compact, aligned with idx_in
  const bf16 *C_cache;    // [b][N][H*hd] (approximate rows: base context)
  bf16 *C_out;            // [b][N][H*hd]
  const int *ex_rows, *ex_off;  // exact-row list (row ids) + offsets [b+1]
  const int *ap_rows, *ap_off;  // approximate-row list + offsets
  const int *sal_rows, *sal_off;  // idx_in (salient keys) + offsets
  int max_rows_per_seq;         // upper bound of rows per list per sequence
  float scale;
  int row_lo;                   // first input position (0 full input, L_P response-only)
  float2 *stats;                // [b*N][H] (row max, sum-exp) scratch in the exp2 domain
  int num_sms;
  // fused head_dim-128 kernel (attn_fused.cu)
  const bf16 *Qx = nullptr;     // [M_in][H*hd] compact new queries of the exact rows (aligned with ex_rows)
  const bf16 *Kx = nullptr;     // [M_in][KVH*hd] compact new keys of the salient rows (aligned with dV)
  const uint32_t *rowflag = nullptr;  // [b*N] == row_tag: exact row (in idx_in) of this layer step
  uint32_t row_tag = 0;
  bool full_only = false;       // FullStep: every row exact (ex_rows = identity), no approximate tiles
  int *work_ctr = nullptr;      // [2] fused kernel scheduler counters (ctx-owned, zero between launches)
  // incremental softmax statistics (fused kernel)
  float2 *stats_cache = nullptr;  // [b*N][H] per-layer (m c, l), written by every launch for its rows
  const bf16 *Kxo = nullptr;      // [M_in][KVH*hd] compact keys of idx_in BEFORE this step's overwrite
  bool inc = false;               // response-row statistics are current: type-3 tiles
  int resp_lo = 0;                // first response position
  int mode = 0;                   // 0 step, 1 fixup list, 2 statistics refresh
  int *fix = nullptr;             // [1 + fix_cap] fixup list (ctx-owned, count zero between steps)
  int fix_cap = 0;
  // incremental statistics of the prompt rows in full-input steps: the keys changed since those
  // statistics were current (U: idx_in first, then the keys written since), compact per sequence
  // at rows [s*N, s*N + ucnt[s]): new values Kun, values at the statistics' time Kuo
  const bf16 *Kun = nullptr, *Kuo = nullptr;
  const int *ucnt = nullptr;
  bool pinc = false;
  // fused similarity partials (fused kernel, sparse steps): C_out must be C_cache
  float4 *cos_part = nullptr;     // [b*N][H] (dot, |C_new|^2, |C_old|^2, -)
};
int attention_launch(const AttnArgs &a, cudaStream_t st);
int attention_fused_launch(const AttnArgs &a, cudaStream_t st);  // attn_fused.cu
// true when attention_launch writes the delta dC (not C) for the approximate rows of a sparse step
bool attention_writes_delta(int hd);
extern bool g_attn_fused_enabled;  // test hook (dyllm_set_option)
extern int g_attn_t4_rows;        // fused attention: exact-row items of <= this many rows run transposed (0: off)
extern unsigned long long *g_attn_trace;  // debug hook (dyllm_debug_trace_buffer, which = 1)
extern unsigned long long *g_attn_events;  // debug hook (dyllm_debug_trace_buffer, which = 2)
extern unsigned long long *g_sel_trace;    // debug hook (dyllm_debug_trace_buffer, which = 3)

}  // namespace dy
