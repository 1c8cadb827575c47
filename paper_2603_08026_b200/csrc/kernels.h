// kernels.h — launch wrappers of kernels.cu (all asynchronous on `st`).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

typedef __nv_bfloat16 bf16;

namespace dy {
void launch_embed_rows(const int *tokens, const int *rows, const int *M_ptr, int M_cap, const bf16 *emb, bf16 *H0,
                       int d, cudaStream_t st);
// optional row bookkeeping of a1 for the fused a2+a3 epilogue (EPI_QKV): rowflag[r] = tag, and, with
// snap set, snap[i] = (dtag[r] != epoch) then dtag[r] = epoch (statistics epochs, D21)
struct RowMark {
  uint32_t *rowflag = nullptr;
  uint32_t tag = 0;
  uint32_t *dtag = nullptr;
  uint32_t epoch = 0;
  uint8_t *snap = nullptr;
};
void launch_gather_rmsnorm(const bf16 *src, const int *idx, const int *M_ptr, int M_cap, const bf16 *g, float eps,
                           bf16 *dst, int d, cudaStream_t st, RowMark mk = RowMark{});
void launch_gather_rows(const bf16 *src, const int *idx, const int *M_ptr, int M_cap, bf16 *dst, int width,
                        cudaStream_t st);
void launch_scatter_rows(const bf16 *src, const int *idx, const int *M_ptr, int M_cap, bf16 *dst, int width,
                         cudaStream_t st);
void launch_rmsnorm_rows(const bf16 *src, const int *M_ptr, int M_cap, const bf16 *g, float eps, bf16 *dst, int d,
                         cudaStream_t st);
void launch_qkv_post(const bf16 *qkv, const int *idx, const int *M_ptr, int M_cap, const bf16 *bias, int N, int H,
                     int KVH, int hd, const float2 *rope_cs, bf16 *Qc, bf16 *Kc, bf16 *Vc, bf16 *dV, bf16 *Qx,
                     bf16 *Kx, bf16 *Kxo, uint32_t *rowflag, uint32_t tag,
                     cudaStream_t st, int q_only = 0, bf16 *Kfi = nullptr, uint32_t *dtag = nullptr,
                     uint32_t epoch = 0);
void launch_build_u(const int *idx_in, const int *off_in, const uint32_t *rowflag, uint32_t tag, const uint32_t *dtag,
                    uint32_t epoch, const bf16 *K, const bf16 *Kfi, int batch, int N, int kw, int *urows, bf16 *Kun,
                    bf16 *Kuo, int *ucnt, cudaStream_t st);
void launch_rope_table(float2 *cs, int N, int hd, double theta, cudaStream_t st);
void launch_approx_rows(const int *idx_in, const int *off_in, int batch, int N, int row_lo, int *ap_rows,
                        int *ap_off, cudaStream_t st);
void launch_build_list(int mode, const int *carried, const int *carried_off, const int *dec_pos, int n_u, int policy,
                       int batch, int N, int row_lo, int resp_lo, int *out, int *out_off, cudaStream_t st);
void launch_select(const bf16 *c_new, bf16 *c_cache, int batch, int N, int row_lo, int width, float tau, int cmp,
                   float frac, int *idx_out, int *off_out, float *sim_out, unsigned *masks, unsigned *ticket,
                   int *counts, const uint32_t *rowflag, uint32_t tag, const int *dl_off, cudaStream_t st,
                   const float4 *cos_part = nullptr, int H = 0, float4 *part_out = nullptr);
constexpr int kTpMax = 8;
struct TpPtrs {
  void *p[kTpMax];
};
void launch_tp_reduce(const TpPtrs &ptrs, int G, const int *M_ptr, int M_cap, int width, int f32, cudaStream_t st);
void launch_lm_candidates(const int *tokens, int batch, int L_P, int L_R, int block, int mask_id, int *rows, int *off,
                          cudaStream_t st);
void launch_lm_select_commit(const float4 *partials, int n_tiles, const int *rows, const int *off, int batch, int n_u,
                             int *tokens, int *dec_pos, int *dec_tok, const bf16 *emb, bf16 *H0, int d,
                             cudaStream_t st, float *H0f = nullptr);
void launch_ih4_fill(bf16 *dst, int64_t rows, int cols, uint64_t keyA, uint64_t keyB, int il, float scale,
                     cudaStream_t st);
void launch_fill_const(bf16 *dst, int64_t n, float v, cudaStream_t st);
}  // namespace dy
