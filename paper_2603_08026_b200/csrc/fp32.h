// fp32.h — launch wrappers of the fp32-parity mode (fp32.cu; dyllm_model_cfg.dtype = 1, D12).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

typedef __nv_bfloat16 bf16;

namespace dy {
namespace f32 {

// D[out_rows[m] or m][n] = sum_k A[a_rows[m] or m][k] W[n][k] + bias[n] + resid[resid_rows[m] or m][n]
struct GemmF32 {
  const int *M_ptr = nullptr;  // device row count (nullable -> M_cap)
  int M_cap = 0, N = 0, K = 0;
  const float *A = nullptr;
  int lda = 0;
  const int *a_rows = nullptr;
  const bf16 *W = nullptr;     // [N][K]
  float *D = nullptr;
  int ldd = 0;
  const int *out_rows = nullptr;
  const bf16 *bias = nullptr;
  const float *resid = nullptr;
  int ldr = 0;
  const int *resid_rows = nullptr;
};

struct F32Attn {
  int batch, N, H, KVH, hd, row_lo;
  float scale;
  const float *Q, *K, *V;      // caches [b][N][..] (K, V merged: this step's rows already written)
  const float *dV;             // [M_in][KVH*hd] compact, aligned with sal_rows
  const float *C_cache;        // [b][N][H*hd]
  float *C_out;                // [b][N][H*hd]
  const int *sal_rows, *sal_off;  // idx_in + offsets [b+1]
  const int *posmap;           // [b*N] index in idx_in or -1
  bool all_exact;              // FullStep: every row exact
};

void embed(const int *tokens, const int *rows, const int *M_ptr, int M_cap, const bf16 *emb, float *H0, int d,
           cudaStream_t st);
void gather_rmsnorm(const float *src, const int *idx, const int *M_ptr, int M_cap, const bf16 *g, float eps,
                    float *dst, int d, cudaStream_t st);
void gemm(const GemmF32 &g, cudaStream_t st);
void swiglu(const float *gu, const int *M_ptr, int M_cap, int F, float *act, cudaStream_t st);
void qkv_post(const float *qkv, const int *idx, const int *M_ptr, int M_cap, const bf16 *bias, int N, int H, int KVH,
              int hd, const float2 *rope_cs, float *Qc, float *Kc, float *Vc, float *dV, int q_only,
              cudaStream_t st);
void posmap(const int *idx, const int *M_ptr, int rows, int *pm, cudaStream_t st);
void attention(const F32Attn &a, cudaStream_t st);
void select(const float *cn, float *cc, int batch, int N, int row_lo, int width, float tau, int cmp, float frac,
            float *sim, int *idx_out, int *off_out, int *counts, cudaStream_t st);
void lm_reduce(const float *logits, const int *M_ptr, int M_cap, int V, int excl, float4 *partials, cudaStream_t st);

}  // namespace f32
}  // namespace dy
