// fp32.cu — the fp32-parity mode of the salient step (dyllm_model_cfg.dtype = 1, DESIGN D12,
// north_star "1e-4 in fp32 mode"). Same orchestration as the bf16 path (dyllm.cu: lists, device
// row counts, no host sync inside a step), but fp32 storage for every cache and scratch row and
// SIMT fp32 arithmetic: tcgen05 has no fp32 operand kind, and tf32 (10-bit mantissa) cannot reach
// 1e-4. Weights stay bf16 (the blob is bf16, the oracle's weights are bf16-rounded, D12), so the
// products below see exactly the oracle's weights. This mode exists to pin the method at a tight
// tolerance; it is not a throughput path (plain smem-tiled GEMM, one warp per (row, head)
// attention with two passes over the keys, Alg. 4 dense as written — no incremental statistics).
#include <math.h>

#include "common.cuh"
#include "fp32.h"
#include "internal.h"

namespace dy {
namespace f32 {

static inline int grid_cap(int64_t work, int per_block, int cap = 148 * 4) {
  int64_t g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  return static_cast<int>(g < cap ? g : cap);
}

// ---------------------------------------------------------------- a0: H0[r] = E[tok_r]
__global__ void embed_kernel(const int *__restrict__ tokens, const int *__restrict__ rows,
                             const int *__restrict__ M_ptr, int M_cap, const bf16 *__restrict__ emb,
                             float *__restrict__ H0, int d) {
  pdl_wait();
  const int M = M_ptr ? *M_ptr : M_cap;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  for (int i = warp; i < M; i += gridDim.x * blockDim.x / 32) {
    const int r = rows ? rows[i] : i;
    const bf16 *src = emb + static_cast<int64_t>(tokens[r]) * d;
    float *dst = H0 + static_cast<int64_t>(r) * d;
    for (int c = lane; c < d; c += 32) dst[c] = bf2f(src[c]);
  }
}

// ---------------------------------------------------------------- a1: dst[i] = RMSNorm(src[idx[i]]) * g
__global__ void gather_rmsnorm_kernel(const float *__restrict__ src, const int *__restrict__ idx,
                                      const int *__restrict__ M_ptr, int M_cap, const bf16 *__restrict__ g,
                                      float eps, float *__restrict__ dst, int d) {
  pdl_wait();
  const int M = M_ptr ? *M_ptr : M_cap;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  for (int i = warp; i < M; i += gridDim.x * blockDim.x / 32) {
    const float *s = src + static_cast<int64_t>(idx ? idx[i] : i) * d;
    float ss = 0.f;
    for (int c = lane; c < d; c += 32) ss = fmaf(s[c], s[c], ss);
    ss = warp_sum(ss);
    const float inv = 1.f / sqrtf(ss / d + eps);
    float *o = dst + static_cast<int64_t>(i) * d;
    for (int c = lane; c < d; c += 32) o[c] = s[c] * inv * bf2f(g[c]);
  }
}

// ---------------------------------------------------------------- GEMM  D = A W^T (+ epilogue)
// A fp32 [M][K] (row m read at a_rows[m] when given), W bf16 [N][K]. 64x64 output tile per CTA,
// 256 threads x 4x4 outputs, K in steps of 16 through shared memory; fp32 FMA accumulation.
constexpr int kBM = 64, kBN = 64, kBK = 16;
__global__ void __launch_bounds__(256) gemm_kernel(GemmF32 g) {
  pdl_wait();
  const int M = g.M_ptr ? *g.M_ptr : g.M_cap;
  const int m0 = blockIdx.y * kBM, n0 = blockIdx.x * kBN;
  if (m0 >= M) return;
  __shared__ float As[kBK][kBM + 1], Ws[kBK][kBN + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < g.K; k0 += kBK) {
    for (int e = threadIdx.x; e < kBM * kBK; e += 256) {
      const int mm = e / kBK, kk = e % kBK, m = m0 + mm, k = k0 + kk;
      float va = 0.f, vw = 0.f;
      if (m < M && k < g.K) va = g.A[static_cast<int64_t>(g.a_rows ? g.a_rows[m] : m) * g.lda + k];
      if (n0 + mm < g.N && k < g.K) vw = bf2f(g.W[static_cast<int64_t>(n0 + mm) * g.K + k]);
      As[kk][mm] = va;
      Ws[kk][mm] = vw;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kBK; ++kk) {
      float a[4], w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = As[kk][ty * 4 + i];
        w[i] = Ws[kk][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], w[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
    const int64_t orow = g.out_rows ? g.out_rows[m] : m;
    const int64_t rrow = g.resid_rows ? g.resid_rows[m] : m;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= g.N) continue;
      float v = acc[i][j];
      if (g.bias) v += bf2f(g.bias[n]);
      if (g.resid) v += g.resid[rrow * g.ldr + n];
      g.D[orow * g.ldd + n] = v;
    }
  }
}

// SwiGLU over the interleaved gate/up product (blocks of kGuIl rows: [gate][up], dyllm.cu):
// act[m][j] = SiLU(gu[m][gate(j)]) * gu[m][up(j)]
__global__ void swiglu_kernel(const float *__restrict__ gu, const int *__restrict__ M_ptr, int M_cap, int F,
                              float *__restrict__ act) {
  pdl_wait();
  const int M = M_ptr ? *M_ptr : M_cap;
  const int64_t n = static_cast<int64_t>(M) * F;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t m = e / F;
    const int j = static_cast<int>(e - m * F);
    const int col = (j / kGuIl) * 2 * kGuIl + j % kGuIl;
    const float a = gu[m * 2 * F + col], b = gu[m * 2 * F + col + kGuIl];
    act[e] = a / (1.f + expf(-a)) * b;
  }
}

// ---------------------------------------------------------------- a3: RoPE, dV, in-place K/V/Q
// One CTA per listed row i (row id r = idx[i], position r % N). dV[i] = v_new - V[r] is read
// before the overwrite. q_only: Q cache alone (D6 refresh of decoded rows).
__global__ void qkv_post_kernel(const float *__restrict__ qkv, const int *__restrict__ idx,
                                const int *__restrict__ M_ptr, int M_cap, const bf16 *__restrict__ bias, int N,
                                int H, int KVH, int hd, const float2 *__restrict__ rope_cs,
                                float *__restrict__ Qc, float *__restrict__ Kc, float *__restrict__ Vc,
                                float *__restrict__ dV, int q_only) {
  pdl_wait();
  const int M = M_ptr ? *M_ptr : M_cap;
  const int qw = H * hd, kw = KVH * hd, W = qw + 2 * kw, half = hd / 2;
  for (int i = blockIdx.x; i < M; i += gridDim.x) {
    const int r = idx ? idx[i] : i;
    const int pos = r % N;
    const float *src = qkv + static_cast<int64_t>(i) * W;
    const float2 *cs = rope_cs + static_cast<int64_t>(pos) * half;
    const int npairs = (q_only ? H : H + KVH) * half;
    for (int e = threadIdx.x; e < npairs; e += blockDim.x) {
      const int head = e / half, k = e % half;
      const int col = head * hd + k;  // q heads then k heads, contiguous
      float x1 = src[col], x2 = src[col + half];
      if (bias) {
        x1 += bf2f(bias[col]);
        x2 += bf2f(bias[col + half]);
      }
      const float c = cs[k].x, s = cs[k].y;
      const float y1 = x1 * c - x2 * s, y2 = x2 * c + x1 * s;
      float *dst = col < qw ? Qc + static_cast<int64_t>(r) * qw + col : Kc + static_cast<int64_t>(r) * kw + (col - qw);
      dst[0] = y1;
      dst[half] = y2;
    }
    if (q_only) continue;
    for (int e = threadIdx.x; e < kw; e += blockDim.x) {
      float v = src[qw + kw + e];
      if (bias) v += bf2f(bias[qw + kw + e]);
      float *vc = Vc + static_cast<int64_t>(r) * kw + e;
      if (dV) dV[static_cast<int64_t>(i) * kw + e] = v - *vc;
      *vc = v;
    }
  }
}

// posmap[r] = index of row r in idx_in (its compact dV row), -1 for other rows
__global__ void posmap_kernel(const int *__restrict__ idx, const int *__restrict__ M_ptr, int rows,
                              int *__restrict__ posmap) {
  pdl_wait();
  const int M = *M_ptr;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows; e += gridDim.x * blockDim.x) posmap[e] = -1;
  __syncthreads();
  // single CTA: the clear above is ordered before the marks by the barrier
  for (int m = threadIdx.x; m < M; m += blockDim.x) posmap[idx[m]] = m;
}

// ---------------------------------------------------------------- a4: attention (Alg. 2 line 5, Alg. 3 lines 8-11, Alg. 4)
// One warp per (input row r, head h). Pass 1: row max m and l = sum exp(s - m) over all N keys
// (the merged K). Pass 2: exact rows (posmap[r] >= 0, or all rows when all_exact):
// C = sum_j p_j V_j; approximate rows: C = C_cache + sum_{e in idx_in(seq)} p_{idx[e]} dV[e]
// (Alg. 4 A[:, idx] dV). Output: Cout[r] (full context, not a delta).
__global__ void attention_kernel(F32Attn a) {
  pdl_wait();
  extern __shared__ float qs[];  // [warps][hd]
  const int warp_in_cta = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int L = a.N - a.row_lo;
  const int64_t items = static_cast<int64_t>(a.batch) * L * a.H;
  const int qw = a.H * a.hd, kw = a.KVH * a.hd, grp = a.H / a.KVH;
  float *q = qs + warp_in_cta * a.hd;
  const int nd = (a.hd + 31) / 32;  // output dims per lane (lane + 32 i)
  for (int64_t it = blockIdx.x * (blockDim.x / 32) + warp_in_cta; it < items;
       it += static_cast<int64_t>(gridDim.x) * (blockDim.x / 32)) {
    const int h = static_cast<int>(it % a.H);
    const int64_t rl = it / a.H;
    const int s = static_cast<int>(rl / L), p = a.row_lo + static_cast<int>(rl % L);
    const int64_t r = static_cast<int64_t>(s) * a.N + p;
    const int kvh = h / grp;
    __syncwarp();
    for (int c = lane; c < a.hd; c += 32) q[c] = a.Q[r * qw + h * a.hd + c] * a.scale;
    __syncwarp();
    const float *Kb = a.K + static_cast<int64_t>(s) * a.N * kw + kvh * a.hd;
    auto score = [&](int j) {
      const float *k = Kb + static_cast<int64_t>(j) * kw;
      float acc = 0.f;
      for (int c = 0; c < a.hd; ++c) acc = fmaf(q[c], k[c], acc);
      return acc;
    };
    float m = -INFINITY, l = 0.f;
    for (int j = lane; j < a.N; j += 32) {
      const float sc = score(j);
      if (sc > m) {
        l = l * expf(m - sc) + 1.f;
        m = sc;
      } else {
        l += expf(sc - m);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o), l2 = __shfl_xor_sync(0xffffffffu, l, o);
      const float mn = fmaxf(m, m2);
      l = (m == -INFINITY ? 0.f : l * expf(m - mn)) + (m2 == -INFINITY ? 0.f : l2 * expf(m2 - mn));
      m = mn;
    }
    const float inv_l = 1.f / l;
    const bool exact = a.all_exact || a.posmap[r] >= 0;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    if (exact) {
      const float *Vb = a.V + static_cast<int64_t>(s) * a.N * kw + kvh * a.hd;
      for (int j0 = 0; j0 < a.N; j0 += 32) {
        const int j = j0 + lane;
        const float pj = j < a.N ? expf(score(j) - m) * inv_l : 0.f;
        const int nk = min(32, a.N - j0);
        for (int jj = 0; jj < nk; ++jj) {
          const float pb = __shfl_sync(0xffffffffu, pj, jj);
          const float *v = Vb + static_cast<int64_t>(j0 + jj) * kw;
          for (int i = 0; i < nd; ++i)
            if (lane + 32 * i < a.hd) acc[i] = fmaf(pb, v[lane + 32 * i], acc[i]);
        }
      }
    } else {
      const int e0 = a.sal_off[s], e1 = a.sal_off[s + 1];
      for (int b0 = e0; b0 < e1; b0 += 32) {
        const int e = b0 + lane;
        const float pj = e < e1 ? expf(score(a.sal_rows[e] - s * a.N) - m) * inv_l : 0.f;
        const int nk = min(32, e1 - b0);
        for (int jj = 0; jj < nk; ++jj) {
          const float pb = __shfl_sync(0xffffffffu, pj, jj);
          const float *dv = a.dV + static_cast<int64_t>(b0 + jj) * kw + kvh * a.hd;
          for (int i = 0; i < nd; ++i)
            if (lane + 32 * i < a.hd) acc[i] = fmaf(pb, dv[lane + 32 * i], acc[i]);
        }
      }
      for (int i = 0; i < nd; ++i)
        if (lane + 32 * i < a.hd) acc[i] += a.C_cache[r * qw + h * a.hd + lane + 32 * i];
    }
    for (int i = 0; i < nd; ++i)
      if (lane + 32 * i < a.hd) a.C_out[r * qw + h * a.hd + lane + 32 * i] = acc[i];
  }
}

// ---------------------------------------------------------------- a5: similarity, threshold, compaction
// Kernel 1 (one warp per input row): s = <C_new, C_cache> / sqrt(|C_new|^2 |C_cache|^2) (P:259-261,
// D9 zero-norm policy), then C_cache <- C_new (Alg. 3 line 16).
__global__ void cosine_commit_kernel(const float *__restrict__ cn, float *__restrict__ cc, int batch, int N,
                                     int row_lo, int width, float *__restrict__ sim) {
  pdl_wait();
  const int L = N - row_lo;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  for (int i = warp; i < batch * L; i += gridDim.x * blockDim.x / 32) {
    const int64_t r = static_cast<int64_t>(i / L) * N + row_lo + i % L;
    const float *x = cn + r * width;
    float *y = cc + r * width;
    float dot = 0.f, na = 0.f, nb = 0.f;
    for (int c = lane; c < width; c += 32) {
      dot = fmaf(x[c], y[c], dot);
      na = fmaf(x[c], x[c], na);
      nb = fmaf(y[c], y[c], nb);
    }
    dot = warp_sum(dot);
    na = warp_sum(na);
    nb = warp_sum(nb);
    __syncwarp();
    for (int c = lane; c < width; c += 32) y[c] = x[c];
    if (lane == 0) {
      const bool za = na < 1e-24f, zb = nb < 1e-24f;
      sim[r] = (za && zb) ? 1.f : ((za || zb) ? 0.f : dot / sqrtf(na * nb));
    }
  }
}

// Kernel 2 (single CTA): per sequence, threshold (fixed tau, or D19's tau* = similarity of rank
// k = round(f L) found by counting ranks), strict '<' (cmp 1: '<='), stable ballot compaction into
// the packed list + offsets (+ per-sequence counts).
__global__ void threshold_compact_kernel(const float *__restrict__ sim, int batch, int N, int row_lo, float tau,
                                         int cmp, float frac, int *__restrict__ idx_out, int *__restrict__ off_out,
                                         int *__restrict__ counts) {
  pdl_wait();
  __shared__ int warp_cnt[32];
  __shared__ float thr_s;
  const int L = N - row_lo;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  int base = 0;
  if (threadIdx.x == 0) off_out[0] = 0;
  for (int s = 0; s < batch; ++s) {
    const float *sv = sim + static_cast<int64_t>(s) * N + row_lo;
    if (threadIdx.x == 0) thr_s = tau;
    __syncthreads();
    if (frac >= 0.f) {
      const int k = static_cast<int>(floorf(frac * L + 0.5f));
      if (threadIdx.x == 0) thr_s = INFINITY;
      __syncthreads();
      if (k < L)
        for (int i = threadIdx.x; i < L; i += blockDim.x) {
          int below = 0, equal = 0;
          for (int j = 0; j < L; ++j) {
            below += sv[j] < sv[i];
            equal += sv[j] == sv[i];
          }
          if (below <= k && k < below + equal) thr_s = sv[i];  // every writer writes the same value
        }
      __syncthreads();
    }
    const float thr = thr_s;
    for (int p0 = 0; p0 < L; p0 += blockDim.x) {
      const int p = p0 + threadIdx.x;
      const bool keep = p < L && (cmp ? sv[p] <= thr : sv[p] < thr);
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (lane == 0) warp_cnt[warp] = __popc(bal);
      __syncthreads();
      int before = 0, tot = 0;
      for (int w = 0; w < nw; ++w) {
        before += w < warp ? warp_cnt[w] : 0;
        tot += warp_cnt[w];
      }
      if (keep) idx_out[base + before + __popc(bal & ((1u << lane) - 1))] = s * N + row_lo + p;
      base += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      off_out[s + 1] = base;
      if (counts) counts[s] = base - off_out[s];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- a9: LM-head row reduction
// One warp per candidate row: (max, sum exp(z - max), argmax with ties to the lowest id) in the
// float4 partial layout of lm_select_commit_kernel (one tile per row).
__global__ void lm_reduce_kernel(const float *__restrict__ logits, const int *__restrict__ M_ptr, int V, int excl,
                                 float4 *__restrict__ partials) {
  pdl_wait();
  const int M = *M_ptr;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  for (int i = warp; i < M; i += gridDim.x * blockDim.x / 32) {
    const float *z = logits + static_cast<int64_t>(i) * V;
    float m = -INFINITY;
    int am = 0x7fffffff;
    for (int c = lane; c < V; c += 32)  // the mask token is never a prediction (D22)
      if (c != excl && z[c] > m) {
        m = z[c];
        am = c;
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
      const int a2 = __shfl_xor_sync(0xffffffffu, am, o);
      if (m2 > m || (m2 == m && a2 < am)) {
        m = m2;
        am = a2;
      }
    }
    float sm = 0.f;
    for (int c = lane; c < V; c += 32) sm += expf(z[c] - m);
    sm = warp_sum(sm);
    if (lane == 0) partials[i] = make_float4(m, sm, __int_as_float(am), 0.f);
  }
}

// ---------------------------------------------------------------- launch wrappers
void embed(const int *tokens, const int *rows, const int *M_ptr, int M_cap, const bf16 *emb, float *H0, int d,
           cudaStream_t st) {
  DY_CUDA_LAUNCH(launch_k(embed_kernel, dim3(grid_cap(M_cap, 8)), dim3(256), 0, st, 1, tokens, rows, M_ptr, M_cap, emb,
                          H0, d));
}
void gather_rmsnorm(const float *src, const int *idx, const int *M_ptr, int M_cap, const bf16 *g, float eps,
                    float *dst, int d, cudaStream_t st) {
  DY_CUDA_LAUNCH(launch_k(gather_rmsnorm_kernel, dim3(grid_cap(M_cap, 8)), dim3(256), 0, st, 1, src, idx, M_ptr,
                          M_cap, g, eps, dst, d));
}
void gemm(const GemmF32 &g, cudaStream_t st) {
  dim3 grid((g.N + kBN - 1) / kBN, (g.M_cap + kBM - 1) / kBM);
  DY_CUDA_LAUNCH(launch_k(gemm_kernel, grid, dim3(256), 0, st, 1, g));
}
void swiglu(const float *gu, const int *M_ptr, int M_cap, int F, float *act, cudaStream_t st) {
  DY_CUDA_LAUNCH(launch_k(swiglu_kernel, dim3(grid_cap(static_cast<int64_t>(M_cap) * F, 256)), dim3(256), 0, st, 1,
                          gu, M_ptr, M_cap, F, act));
}
void qkv_post(const float *qkv, const int *idx, const int *M_ptr, int M_cap, const bf16 *bias, int N, int H, int KVH,
              int hd, const float2 *rope_cs, float *Qc, float *Kc, float *Vc, float *dV, int q_only,
              cudaStream_t st) {
  DY_CUDA_LAUNCH(launch_k(qkv_post_kernel, dim3(M_cap < 148 * 4 ? (M_cap > 0 ? M_cap : 1) : 148 * 4), dim3(256), 0,
                          st, 1, qkv, idx, M_ptr, M_cap, bias, N, H, KVH, hd, rope_cs, Qc, Kc, Vc, dV, q_only));
}
void posmap(const int *idx, const int *M_ptr, int rows, int *pm, cudaStream_t st) {
  DY_CUDA_LAUNCH(launch_k(posmap_kernel, dim3(1), dim3(1024), 0, st, 1, idx, M_ptr, rows, pm));
}
void attention(const F32Attn &a, cudaStream_t st) {
  const int64_t items = static_cast<int64_t>(a.batch) * (a.N - a.row_lo) * a.H;
  const int warps = 8;
  DY_CUDA_LAUNCH(launch_k(attention_kernel, dim3(grid_cap(items, warps, 148 * 8)), dim3(32 * warps),
                          warps * a.hd * sizeof(float), st, 1, a));
}
void select(const float *cn, float *cc, int batch, int N, int row_lo, int width, float tau, int cmp, float frac,
            float *sim, int *idx_out, int *off_out, int *counts, cudaStream_t st) {
  DY_CUDA_LAUNCH(launch_k(cosine_commit_kernel, dim3(grid_cap(static_cast<int64_t>(batch) * (N - row_lo), 8)),
                          dim3(256), 0, st, 1, cn, cc, batch, N, row_lo, width, sim));
  DY_CUDA_LAUNCH(launch_k(threshold_compact_kernel, dim3(1), dim3(1024), 0, st, 1, static_cast<const float *>(sim),
                          batch, N, row_lo, tau, cmp, frac, idx_out, off_out, counts));
}
void lm_reduce(const float *logits, const int *M_ptr, int M_cap, int V, int excl, float4 *partials, cudaStream_t st) {
  DY_CUDA_LAUNCH(launch_k(lm_reduce_kernel, dim3(grid_cap(M_cap, 8)), dim3(256), 0, st, 1, logits, M_ptr, V, excl,
                          partials));
}

}  // namespace f32
}  // namespace dy
