// kernels.cu — the HBM-bound kernels of the salient step
// and the list / unmasking plumbing. All row counts are read from device memory.
#include <algorithm>

#include "common.cuh"
#include "internal.h"
#include "kernels.h"

namespace dy {

unsigned long long *g_sel_trace = nullptr;  // debug hook (dyllm_debug_trace_buffer, which = 3)

// ============================================================================ a0: embeddings
// H0[r] = E[tokens[r]] for every row r of the list (or all rows when rows == nullptr).
__global__ void embed_rows_kernel(const int *__restrict__ tokens, const int *__restrict__ rows,
                                  const int *__restrict__ M_ptr, int M_cap, const bf16 *__restrict__ emb,
                                  bf16 *__restrict__ H0, int d) {
  pdl_wait();
  const int M = M_ptr ? *M_ptr : M_cap;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  for (int i = warp; i < M; i += gridDim.x * blockDim.x / 32) {
    const int r = rows ? rows[i] : i;
    const int tok = tokens[r];
    const uint4 *src = reinterpret_cast<const uint4 *>(emb + static_cast<int64_t>(tok) * d);
    uint4 *dst = reinterpret_cast<uint4 *>(H0 + static_cast<int64_t>(r) * d);
    for (int c = lane; c < d / 8; c += 32) dst[c] = src[c];
  }
}

// ============================================================================ a1: gather + RMSNorm
// dst[i] = RMSNorm(src[idx[i]]) * g  (D3), one warp per row, fp32 statistics.
__global__ void gather_rmsnorm_kernel(const bf16 *__restrict__ src, const int *__restrict__ idx,
                                      const int *__restrict__ M_ptr, int M_cap, const bf16 *__restrict__ g,
                                      float eps, bf16 *__restrict__ dst, int d, RowMark mk) {
  pdl_wait();
  const int M = M_ptr ? *M_ptr : M_cap;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  const int nv = d / 8;
  constexpr int VMAX = 16;  // rows up to 4096 wide stay in registers (16 x 16 B per lane)
  for (int i = warp; i < M; i += gridDim.x * blockDim.x / 32) {
    const int r = idx ? idx[i] : i;
    // a3's row bookkeeping when the QKV GEMM epilogue does a3 (EPI_QKV): the row is an exact row of
    // this layer step, and whether its key is written for the first time in the statistics epoch
    // (the epilogue then keeps the overwritten key in Kfi) is decided here, once per row
    if (lane == 0) {
      if (mk.rowflag) mk.rowflag[r] = mk.tag;
      if (mk.snap) {
        mk.snap[i] = mk.dtag[r] != mk.epoch;
        mk.dtag[r] = mk.epoch;
      }
    }
    const uint4 *s = reinterpret_cast<const uint4 *>(src + static_cast<int64_t>(r) * d);
    uint4 *o = reinterpret_cast<uint4 *>(dst + static_cast<int64_t>(i) * d);
    const uint4 *gv = reinterpret_cast<const uint4 *>(g);
    if (nv <= 32 * VMAX) {
      // row and gain loads issued together (one memory round trip per row)
      uint4 v[VMAX], gw[VMAX];
#pragma unroll
      for (int u = 0; u < VMAX; ++u)
        if (lane + u * 32 < nv) v[u] = ld_nc_v4(s + lane + u * 32);
#pragma unroll
      for (int u = 0; u < VMAX; ++u)
        if (lane + u * 32 < nv) gw[u] = gv[lane + u * 32];
      float ss = 0.f;
#pragma unroll
      for (int u = 0; u < VMAX; ++u)
        if (lane + u * 32 < nv) {
          float f[8];
          unpack8(v[u], f);
#pragma unroll
          for (int j = 0; j < 8; ++j) ss += f[j] * f[j];
        }
      ss = warp_sum(ss);
      const float inv = rsqrtf(ss / d + eps);
#pragma unroll
      for (int u = 0; u < VMAX; ++u)
        if (lane + u * 32 < nv) {
          float f[8], w[8];
          unpack8(v[u], f);
          unpack8(gw[u], w);
#pragma unroll
          for (int j = 0; j < 8; ++j) f[j] = f[j] * inv * w[j];
          o[lane + u * 32] = pack8(f);
        }
      continue;
    }
    float ss = 0.f;
    for (int c = lane; c < nv; c += 32) {
      float f[8];
      unpack8(s[c], f);
#pragma unroll
      for (int j = 0; j < 8; ++j) ss += f[j] * f[j];
    }
    ss = warp_sum(ss);
    const float inv = rsqrtf(ss / d + eps);
    for (int c = lane; c < nv; c += 32) {
      float f[8], w[8];
      unpack8(s[c], f);
      unpack8(gv[c], w);
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] = f[j] * inv * w[j];
      o[c] = pack8(f);
    }
  }
}

// warp-cooperative row copy with 8 independent 16-byte loads in flight per lane
__device__ __forceinline__ void copy_row(uint4 *__restrict__ o, const uint4 *__restrict__ s, int nv, int lane) {
  constexpr int U = 8;
  for (int c0 = lane; c0 < nv; c0 += 32 * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c0 + u * 32 < nv) v[u] = ld_nc_v4(s + c0 + u * 32);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c0 + u * 32 < nv) o[c0 + u * 32] = v[u];
  }
}

// plain row gather dst[i] = src[idx[i]] (a6 A-operand: C[idx_out])
__global__ void gather_rows_kernel(const bf16 *__restrict__ src, const int *__restrict__ idx,
                                   const int *__restrict__ M_ptr, int M_cap, bf16 *__restrict__ dst, int width) {
  pdl_wait();
  const int M = M_ptr ? *M_ptr : M_cap;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  const int nv = width / 8;
  for (int i = warp; i < M; i += gridDim.x * blockDim.x / 32) {
    const uint4 *s = reinterpret_cast<const uint4 *>(src + static_cast<int64_t>(idx[i]) * width);
    uint4 *o = reinterpret_cast<uint4 *>(dst + static_cast<int64_t>(i) * width);
    copy_row(o, s, nv, lane);
  }
}

// ============================================================================ a8: scatter-back
// dst[idx[i]] = src[i]  (H_l[idx_out] <- FFN rows); other rows untouched (zero-copy reuse)
__global__ void scatter_rows_kernel(const bf16 *__restrict__ src, const int *__restrict__ idx,
                                    const int *__restrict__ M_ptr, int M_cap, bf16 *__restrict__ dst, int width) {
  pdl_wait();
  const int M = M_ptr ? *M_ptr : M_cap;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  const int nv = width / 8;
  for (int i = warp; i < M; i += gridDim.x * blockDim.x / 32) {
    const uint4 *s = reinterpret_cast<const uint4 *>(src + static_cast<int64_t>(i) * width);
    uint4 *o = reinterpret_cast<uint4 *>(dst + static_cast<int64_t>(idx[i]) * width);
    copy_row(o, s, nv, lane);
  }
}

// ============================================================================ a3: RoPE, dV, cache rows
// For packed row i (row id r = idx[i], pos = r % N): q,k,v = qkv[i] (+bias); RoPE(q,k) at pos
// (rotate-half, D10); dV = v - V_cache[r] captured BEFORE the overwrite;
// Q_cache[r], K_cache[r], V_cache[r] <- q, k, v (D6).
// two CTAs of 512 threads per SM (92 registers left one resident: 4 waves of CTAs for 592 rows)
#ifndef DYLLM_QKVPOST_LB
#define DYLLM_QKVPOST_LB 2
#endif
__global__ void __launch_bounds__(512, DYLLM_QKVPOST_LB) qkv_post_kernel(const bf16 *__restrict__ qkv, const int *__restrict__ idx,
                                const int *__restrict__ M_ptr, int M_cap, const bf16 *__restrict__ bias, int N,
                                int H, int KVH, int hd, const float2 *__restrict__ rope_cs, bf16 *__restrict__ Qc,
                                bf16 *__restrict__ Kc, bf16 *__restrict__ Vc, bf16 *__restrict__ dV,
                                bf16 *__restrict__ Qx, bf16 *__restrict__ Kx, bf16 *__restrict__ Kxo,
                                uint32_t *__restrict__ rowflag, uint32_t tag, int q_only,
                                bf16 *__restrict__ Kfi, uint32_t *__restrict__ dtag, uint32_t epoch) {
  pdl_wait();
  const int M = M_ptr ? *M_ptr : M_cap;
  const int qw = H * hd, kw = KVH * hd, W = qw + 2 * kw;
  const int half = hd / 2, hv = half / 8;  // 8 rotation pairs per thread (16-byte vectors)
  // q_only: refresh the Q cache rows alone (K / V / dV / row flag untouched)
  const int nqk = (q_only ? H : H + KVH) * hv, nvv = q_only ? 0 : kw / 8;
  const int rounds = (max(nqk, nvv) + blockDim.x - 1) / blockDim.x;  // work items per thread (2 at 256 threads, LLaDA)
  for (int i = blockIdx.x; i < M; i += gridDim.x) {
    const int r = idx ? idx[i] : i;
    const int pos = r % N;
    const bf16 *src = qkv + static_cast<int64_t>(i) * W;
    if (rowflag && !q_only && threadIdx.x == 0) rowflag[r] = tag;  // exact row of this layer step (fused attention)
    const float2 *cs = rope_cs + static_cast<int64_t>(pos) * half;
    // statistics epochs (incremental prompt statistics): the first write of a key row
    // since its layer's epoch began keeps the overwritten key in Kfi (the key the prompt rows'
    // statistics were computed with) and marks the row changed. The tag is read here and rewritten
    // after the row's barrier below, so no load of the row waits on a barrier: one round trip for
    // the row id, one for everything else (the overwritten key is read whenever Kxo or Kfi is set)
    const bool snap = Kfi && !q_only && dtag[r] != epoch;
    for (int rd = 0; rd < rounds; ++rd) {
      const int v = rd * blockDim.x + threadIdx.x;
      const bool has_qk = v < nqk, has_v = v < nvv;
      // all loads of this thread first (one memory round trip): its q/k rotation pairs + table,
      // its V slice and the V cache slice it replaces
      int head = 0, k0 = 0, col = 0;
      uint4 u1 = make_uint4(0, 0, 0, 0), u2 = u1, ub1 = u1, ub2 = u1, uv = u1, uvb = u1, uvo = u1, uk1 = u1, uk2 = u1;
      float4 c4[4];
      if (has_qk) {
        head = v / hv;
        k0 = (v - head * hv) * 8;
        col = head * hd + k0;  // q cols [0,qw), k cols [qw, qw+kw): heads contiguous
        u1 = *reinterpret_cast<const uint4 *>(src + col);
        u2 = *reinterpret_cast<const uint4 *>(src + col + half);
        if (bias) {
          ub1 = *reinterpret_cast<const uint4 *>(bias + col);
          ub2 = *reinterpret_cast<const uint4 *>(bias + col + half);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) c4[j] = reinterpret_cast<const float4 *>(cs + k0)[j];
        if ((Kxo || (Kfi && !q_only)) && col >= qw) {  // the key row this step overwrites (incremental statistics)
          const bf16 *ko = Kc + static_cast<int64_t>(r) * kw + (col - qw);
          uk1 = *reinterpret_cast<const uint4 *>(ko);
          uk2 = *reinterpret_cast<const uint4 *>(ko + half);
        }
      }
      const int vc0 = v * 8;
      uint4 *vc = reinterpret_cast<uint4 *>(Vc + static_cast<int64_t>(r) * kw + vc0);
      if (has_v) {
        uv = *reinterpret_cast<const uint4 *>(src + qw + kw + vc0);
        if (bias) uvb = *reinterpret_cast<const uint4 *>(bias + qw + kw + vc0);
        if (dV) uvo = *vc;
      }
      // q and k heads: pairs (x[k], x[k + hd/2]) rotated by pos * theta^(-2k/hd) (table, fp64-derived)
      if (has_qk) {
        float x1[8], x2[8];
        unpack8(u1, x1);
        unpack8(u2, x2);
        if (bias) {
          float b1[8], b2[8];
          unpack8(ub1, b1);
          unpack8(ub2, b2);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            x1[j] += b1[j];
            x2[j] += b2[j];
          }
        }
        const float *cf = reinterpret_cast<const float *>(c4);
        float y1[8], y2[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float cc = cf[2 * j], sn = cf[2 * j + 1];
          y1[j] = x1[j] * cc - x2[j] * sn;
          y2[j] = x2[j] * cc + x1[j] * sn;
        }
        bf16 *dst = (col < qw) ? Qc + static_cast<int64_t>(r) * qw + col : Kc + static_cast<int64_t>(r) * kw + (col - qw);
        const uint4 p1 = pack8(y1), p2 = pack8(y2);
        *reinterpret_cast<uint4 *>(dst) = p1;
        *reinterpret_cast<uint4 *>(dst + half) = p2;
        // compact copies aligned with the packed list (the attention kernel's exact-row queries
        // and salient keys are then contiguous rows: TMA tiles)
        bf16 *cx = (col < qw) ? (Qx ? Qx + static_cast<int64_t>(i) * qw + col : nullptr)
                              : (Kx ? Kx + static_cast<int64_t>(i) * kw + (col - qw) : nullptr);
        if (cx) {
          *reinterpret_cast<uint4 *>(cx) = p1;
          *reinterpret_cast<uint4 *>(cx + half) = p2;
        }
        if (Kxo && col >= qw) {
          bf16 *xo = Kxo + static_cast<int64_t>(i) * kw + (col - qw);
          *reinterpret_cast<uint4 *>(xo) = uk1;
          *reinterpret_cast<uint4 *>(xo + half) = uk2;
        }
        if (snap && col >= qw) {
          bf16 *xf = Kfi + static_cast<int64_t>(r) * kw + (col - qw);
          *reinterpret_cast<uint4 *>(xf) = uk1;
          *reinterpret_cast<uint4 *>(xf + half) = uk2;
        }
      }
      // v: dV = v_new - V_cache (read before the overwrite), then V_cache <- v_new
      if (has_v) {
        float vv[8];
        unpack8(uv, vv);
        if (bias) {
          float bb[8];
          unpack8(uvb, bb);
#pragma unroll
          for (int j = 0; j < 8; ++j) vv[j] += bb[j];
        }
        const uint4 vb = pack8(vv);
        if (dV) {
          float vn[8], vo[8], dd[8];
          unpack8(vb, vn);
          unpack8(uvo, vo);
#pragma unroll
          for (int j = 0; j < 8; ++j) dd[j] = vn[j] - vo[j];
          *reinterpret_cast<uint4 *>(dV + static_cast<int64_t>(i) * kw + vc0) = pack8(dd);
        }
        *vc = vb;
      }
    }
    if (Kfi && !q_only) {
      __syncthreads();  // every thread has read the row's tag before it changes
      if (snap && threadIdx.x == 0) dtag[r] = epoch;
    }
  }
}

// RoPE table cs[pos][k] = (cos, sin)(pos * theta^(-2k/hd)), computed in fp64 once per cache.
__global__ void rope_table_kernel(float2 *__restrict__ cs, int N, int hd, double theta) {
  pdl_wait();
  const int half = hd / 2;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < N * half; e += gridDim.x * blockDim.x) {
    const int pos = e / half, k = e - pos * half;
    const double ang = static_cast<double>(pos) * pow(theta, -2.0 * k / hd);
    double sn, c;
    sincos(ang, &sn, &c);
    cs[e] = make_float2(static_cast<float>(c), static_cast<float>(sn));
  }
}

// ============================================================================ lists
// Approximate-row list of each sequence: input rows [row_lo, N) that are NOT in idx_in
// (exact rows = idx_in itself). One CTA per sequence. ap_off[s] = s*L - off_in[s].
__global__ void approx_rows_kernel(const int *__restrict__ idx_in, const int *__restrict__ off_in, int N,
                                   int row_lo, int *__restrict__ ap_rows, int *__restrict__ ap_off, int batch,
                                   int) {
  pdl_wait();
  extern __shared__ uint8_t flag[];
  __shared__ int warp_cnt[32];
  const int s = blockIdx.x;
  const int L = N - row_lo;
  for (int p = threadIdx.x; p < N; p += blockDim.x) flag[p] = 0;
  __syncthreads();
  const int b0 = off_in[s], b1 = off_in[s + 1];
  for (int j = b0 + threadIdx.x; j < b1; j += blockDim.x) flag[idx_in[j] - s * N] = 1;
  __syncthreads();
  int base = s * L - b0;
  if (threadIdx.x == 0) {
    ap_off[s] = base;
    if (s == batch - 1) ap_off[batch] = batch * L - off_in[batch];
  }
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  for (int p0 = row_lo; p0 < N; p0 += blockDim.x) {
    const int p = p0 + threadIdx.x;
    const bool keep = p < N && !flag[p];
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) warp_cnt[warp] = __popc(m);
    __syncthreads();
    int before = 0, tot = 0;
    for (int w = 0; w < nw; ++w) {
      before += (w < warp) ? warp_cnt[w] : 0;
      tot += warp_cnt[w];
    }
    if (keep) ap_rows[base + before + __popc(m & ((1u << lane) - 1))] = s * N + p;
    base += tot;
    __syncthreads();
  }
}

// Single-CTA list builder used once per step: for each sequence, rows in [row_lo, N) that are
//   mode 0: all rows (identity list)
//   mode 1: in `carried` (its list), or (policy 1) in the decoded set dec_pos[b][n_u]  (D5)
//   mode 2: in the decoded set but NOT in `carried` (the rows whose embedding changed but which the
//           literal layer-1 policy leaves out of idx_in: they get a Q-only refresh, D6)
// Writes a packed row-id list + offsets [b+1].
__global__ void build_list_kernel(int mode, const int *__restrict__ carried, const int *__restrict__ carried_off,
                                  const int *__restrict__ dec_pos, int n_u, int policy, int batch, int N,
                                  int row_lo, int resp_lo, int *__restrict__ out, int *__restrict__ out_off) {
  pdl_wait();
  extern __shared__ uint8_t flag[];
  __shared__ int warp_cnt[32];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  int base = 0;
  if (threadIdx.x == 0) out_off[0] = 0;
  for (int s = 0; s < batch; ++s) {
    for (int p = threadIdx.x; p < N; p += blockDim.x) flag[p] = (mode == 0) ? 1 : 0;
    __syncthreads();
    if (mode == 1) {
      if (carried) {
        for (int j = carried_off[s] + threadIdx.x; j < carried_off[s + 1]; j += blockDim.x)
          flag[carried[j] - s * N] = 1;
      } else {  // idx_sal = None -> the response rows [L_P, N)
        for (int p = resp_lo + threadIdx.x; p < N; p += blockDim.x) flag[p] = 1;
      }
      if (policy == 1 && dec_pos) {
        for (int j = threadIdx.x; j < n_u; j += blockDim.x) {
          const int r = dec_pos[s * n_u + j];
          if (r >= 0) flag[r - s * N] = 1;
        }
      }
    } else if (mode == 2) {
      if (dec_pos)
        for (int j = threadIdx.x; j < n_u; j += blockDim.x) {
          const int r = dec_pos[s * n_u + j];
          if (r >= 0) flag[r - s * N] = 1;
        }
      __syncthreads();
      if (carried) {
        for (int j = carried_off[s] + threadIdx.x; j < carried_off[s + 1]; j += blockDim.x)
          flag[carried[j] - s * N] = 0;
      } else {
        for (int p = resp_lo + threadIdx.x; p < N; p += blockDim.x) flag[p] = 0;
      }
    }
    __syncthreads();
    for (int p0 = row_lo; p0 < N; p0 += blockDim.x) {
      const int p = p0 + threadIdx.x;
      const bool keep = p < N && flag[p];
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (lane == 0) warp_cnt[warp] = __popc(m);
      __syncthreads();
      int before = 0, tot = 0;
      for (int w = 0; w < nw; ++w) {
        before += (w < warp) ? warp_cnt[w] : 0;
        tot += warp_cnt[w];
      }
      if (keep) out[base + before + __popc(m & ((1u << lane) - 1))] = s * N + p;
      base += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) out_off[s + 1] = base;
  }
}

// Changed-key list U of each sequence for the incremental prompt statistics of a full-input step
// (SURVEY §8f1): its idx_in rows in list order (their new keys are the salient keys of the P pass),
// then the other rows whose key was written since the layer's statistics epoch began (ascending).
// Grid (batch, kUgrp): every CTA of a sequence derives the same list (a pass over its N row tags),
// keeps the first kUcap entries in shared memory, and gathers every kUgrp-th of their keys
// compact: Kun = current K, Kuo = the key at the epoch start (Kfi); CTA 0 records the count.
constexpr int kUcap = 256;  // two key tiles: larger lists take the dense path
constexpr int kUgrp = 16;
__global__ void build_u_kernel(const int *__restrict__ idx_in, const int *__restrict__ off_in,
                               const uint32_t *__restrict__ rowflag, uint32_t tag, const uint32_t *__restrict__ dtag,
                               uint32_t epoch, const bf16 *__restrict__ K, const bf16 *__restrict__ Kfi, int N, int kw,
                               int *__restrict__ urows, bf16 *__restrict__ Kun, bf16 *__restrict__ Kuo,
                               int *__restrict__ ucnt) {
  pdl_wait();
  __shared__ int warp_cnt[32];
  __shared__ int u[kUcap];
  const int s = blockIdx.x;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  const int b0 = off_in[s], e = off_in[s + 1] - b0;
  for (int j = threadIdx.x; j < e && j < kUcap; j += blockDim.x) u[j] = idx_in[b0 + j];
  int base = e;
  for (int p0 = 0; p0 < N; p0 += blockDim.x) {
    const int p = p0 + threadIdx.x;
    const int64_t r = static_cast<int64_t>(s) * N + p;
    const bool keep = p < N && dtag[r] == epoch && rowflag[r] != tag;
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) warp_cnt[warp] = __popc(m);
    __syncthreads();
    int before = 0, tot = 0;
    for (int w = 0; w < nw; ++w) {
      before += (w < warp) ? warp_cnt[w] : 0;
      tot += warp_cnt[w];
    }
    const int pos = base + before + __popc(m & ((1u << lane) - 1));
    if (keep && pos < kUcap) u[pos] = static_cast<int>(r);
    base += tot;
    __syncthreads();
  }
  if (blockIdx.y == 0 && threadIdx.x == 0) ucnt[s] = base;
  const int n = min(base, kUcap), nv = kw / 8;
  for (int i = blockIdx.y * nw + warp; i < n; i += gridDim.y * nw) {
    const int64_t r = u[i];
    if (blockIdx.y == 0 && lane == 0) urows[static_cast<int64_t>(s) * N + i] = static_cast<int>(r);
    const uint4 *kn = reinterpret_cast<const uint4 *>(K + r * kw);
    const uint4 *ko = reinterpret_cast<const uint4 *>(Kfi + r * kw);
    uint4 *dn = reinterpret_cast<uint4 *>(Kun + (static_cast<int64_t>(s) * N + i) * kw);
    uint4 *dd = reinterpret_cast<uint4 *>(Kuo + (static_cast<int64_t>(s) * N + i) * kw);
    for (int c = lane; c < nv; c += 32) {
      const uint4 a = ld_nc_v4(kn + c), b = ld_nc_v4(ko + c);
      dn[c] = a;
      dd[c] = b;
    }
  }
}

// ============================================================================ a5: K1
// Temporal cosine similarity + threshold + stream compaction (+ commit C_cache <- C_new).
// grid = (ceil(L/32), batch); 8 warps per CTA, 4 rows per warp; row reads are 16-byte,
// coalesced, all loads of a row issued before the reductions. Each CTA produces one 32-bit
// ballot mask of its 32 rows; the last CTA to finish (atomic ticket) scans the masks of all
// sequences and writes the packed list + offsets (no second launch, no host sync).
constexpr int kSelRowsPerCta = 32;

// Two shapes of the same kernel, chosen by the input length: response-only launches (few CTAs:
// one per SM) run 512 threads = 16 warps x 2 of the CTA's 32 rows with 16 16-byte loads in flight
// per lane; full-input launches (30 CTAs per sequence) run 256 threads = 8 warps x 4 rows with 8
// loads in flight and 64 registers, four CTAs per SM, so that all of them are resident at once
// (with one 512-thread CTA per SM, 480 CTAs took 3.24 waves).
template <int kSelThreads>
__global__ void __launch_bounds__(kSelThreads, kSelThreads >= 512 ? 1 : 4) select_salient_kernel(
    const bf16 *__restrict__ c_new, bf16 *__restrict__ c_cache, int N, int row_lo, int width, float tau,
    int cmp, float frac, int *__restrict__ idx_out, int *__restrict__ off_out, float *__restrict__ sim_out,
    unsigned *__restrict__ masks, unsigned *__restrict__ ticket, int *__restrict__ counts_out,
    const uint32_t *__restrict__ rowflag, uint32_t tag, const int *__restrict__ dl_off,
    const float4 *__restrict__ cos_part, int H, float4 *__restrict__ part_out, unsigned long long *trace) {
  constexpr int kSelWarps = kSelThreads / 32;
  constexpr int kSelU = kSelThreads >= 512 ? 8 : 4;
  pdl_wait();
  // debug hook (dyllm_debug_trace_buffer which = 3): %globaltimer per CTA at start / end of its rows,
  // and of the last CTA's tail: [cta][4]
  auto stamp = [&](int slot) {
    if (trace && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      trace[(blockIdx.y * gridDim.x + blockIdx.x) * 4 + slot] = t;
    }
  };
  stamp(0);
  __shared__ unsigned row_flag[kSelRowsPerCta];
  __shared__ bool is_last;
  const int s = blockIdx.y;
  const int L = N - row_lo;
  const int chunk = blockIdx.x;
  const int nchunks = gridDim.x;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nv = width / 8;
  for (int rr = warp; rr < kSelRowsPerCta; rr += kSelWarps) {  // the CTA's 32 rows over its warps
    const int p = row_lo + chunk * kSelRowsPerCta + rr;
    unsigned f = 0;
    if (p < N && cos_part) {
      // partials mode: the attention epilogue formed C_new, committed it and left per
      // (row, head) partial sums; a sequence without salient keys kept every context (s = 1, D9)
      const int64_t r = static_cast<int64_t>(s) * N + p;
      float sim = 1.f;
      if (dl_off[s + 1] > dl_off[s]) {
        float dot = 0.f, na = 0.f, nb = 0.f;
        for (int h = lane; h < H; h += 32) {
          const float4 v = __ldcg(cos_part + r * H + h);
          dot += v.x;
          na += v.y;
          nb += v.z;
        }
        dot = warp_sum(dot);
        na = warp_sum(na);
        nb = warp_sum(nb);
        const bool za = na < 1e-24f, zb = nb < 1e-24f;  // D9 zero-norm policy
        sim = (za && zb) ? 1.f : (za || zb) ? 0.f : dot / sqrtf(na * nb);
      }
      f = cmp ? (sim <= tau) : (sim < tau);
      if (sim_out && lane == 0) sim_out[r] = sim;
    } else if (p < N) {
      const int64_t r = static_cast<int64_t>(s) * N + p;
      const uint4 *a = reinterpret_cast<const uint4 *>(c_new + r * width);
      uint4 *b = reinterpret_cast<uint4 *>(c_cache + r * width);
      // delta mode (fused attention): c_new holds C itself for exact rows and the delta dC for
      // approximate rows, whose C_new = bf16(C_cache + dC) (C_cache when the sequence has no
      // salient key, dC = 0) is formed here from the C_cache row this kernel reads anyway
      bool take_new = true, add = false;
      if (rowflag) {
        take_new = rowflag[r] == tag;
        add = !take_new && dl_off[s + 1] > dl_off[s];
      }
      float dot = 0.f, na = 0.f, nb = 0.f;
      constexpr int U = kSelU;  // 2*U independent 16-byte loads in flight per lane
      for (int c0 = lane; c0 < nv; c0 += 32 * U) {
        uint4 ua[U], ub[U];
        // both rows are loaded unconditionally (no dependence on the row-kind loads above); an
        // approximate row of a sequence without salient keys then takes C_cache
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int c = c0 + u * 32;
          if (c < nv) {
            ub[u] = b[c];
            ua[u] = ld_nc_v4(a + c);
          }
        }
        if (!take_new && !add) {
#pragma unroll
          for (int u = 0; u < U; ++u) ua[u] = ub[u];
        }
        if (add) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            float fa[8], fb[8];
            unpack8(ua[u], fa);
            unpack8(ub[u], fb);
#pragma unroll
            for (int j = 0; j < 8; ++j) fa[j] += fb[j];
            ua[u] = pack8(fa);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int c = c0 + u * 32;
          if (c < nv) {
            float fa[8], fb[8];
            unpack8(ua[u], fa);
            unpack8(ub[u], fb);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              dot = fmaf(fa[j], fb[j], dot);
              na = fmaf(fa[j], fa[j], na);
              nb = fmaf(fb[j], fb[j], nb);
            }
            b[c] = ua[u];  // commit C_cache <- C (Alg. 3 line 16)
          }
        }
      }
      dot = warp_sum(dot);
      na = warp_sum(na);
      nb = warp_sum(nb);
      if (part_out && lane == 0) part_out[r] = make_float4(dot, na, nb, 0.f);
      float sim;
      const bool za = na < 1e-24f, zb = nb < 1e-24f;   // D9 zero-norm policy
      if (za && zb) sim = 1.f;
      else if (za || zb) sim = 0.f;
      else sim = dot / sqrtf(na * nb);   // identical rows: sqrt(fl(x*x)) == x -> exactly 1
      f = cmp ? (sim <= tau) : (sim < tau);
      if (sim_out && lane == 0) sim_out[r] = sim;
    }
    if (lane == 0) row_flag[rr] = f;
  }
  // tensor-parallel shard: only the partial sums over this shard's heads; the threshold
  // and compaction run after the all-reduce (cos_part mode, H = 1), identically on every shard
  if (part_out) return;
  __syncthreads();
  stamp(1);
  __shared__ bool seq_last;
  if (threadIdx.x < 32) {
    const unsigned m = __ballot_sync(0xffffffffu, row_flag[threadIdx.x] != 0);
    if (threadIdx.x == 0) {
      masks[s * nchunks + chunk] = m;
      __threadfence();
      // fraction mode: the last CTA of each sequence finds that sequence's threshold (the
      // sequences in parallel, one SM each) before it arrives at the global ticket
      seq_last = frac >= 0.f && atomicAdd(ticket + 1 + s, 1u) == static_cast<unsigned>(nchunks - 1);
      is_last = false;
      if (!seq_last) is_last = atomicAdd(ticket, 1u) == gridDim.x * gridDim.y - 1;
    }
  }
  __syncthreads();
  const int batch = gridDim.y;
  if (seq_last) {
    __threadfence();
    // fraction-controlled mode (D19): tau* = the similarity of rank k = round(f*L) (0-based) of
    // this sequence, found by an 8-bit radix select over the order-preserving uint32 keys of s
    // with the whole CTA (each pass: a shared histogram of the candidates' next digit, one warp
    // scans it); then the masks are rebuilt as s < tau* (k rows when there are no ties), s <= tau*
    // under cmp = 1. (One warp per sequence measured 14 / 27 us per response-only / full-input
    // launch between the last rows and the compaction, tools/select_trace.py.)
    __shared__ unsigned hist[256];
    __shared__ uint32_t sh_prefix;
    __shared__ int sh_rank;
    const float *sv = sim_out + static_cast<int64_t>(s) * N + row_lo;
    const int k = static_cast<int>(floorf(frac * L + 0.5f));
    auto key_of = [](float f) {
      const uint32_t u = __float_as_uint(f);
      return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    };
    constexpr int kPer = 4;  // similarities per thread kept in registers (L <= 4 * kSelThreads)
    const bool in_regs = L <= kPer * kSelThreads;
    uint32_t keyr[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int i = threadIdx.x + j * kSelThreads;
      keyr[j] = (in_regs && i < L) ? key_of(__ldcg(sv + i)) : 0u;
    }
    float thr = INFINITY;
    if (k < L) {
      uint32_t prefix = 0, pmask = 0;
      int rank = k;
      for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += kSelThreads) hist[i] = 0;
        __syncthreads();
        auto count = [&](uint32_t key, bool valid) {
          const bool in = valid && (key & pmask) == prefix;
          const unsigned act = __ballot_sync(0xffffffffu, in);
          if (in) {  // lanes with the same digit merged: one shared atomic per digit and warp
            const uint32_t dig = (key >> shift) & 255u;
            const unsigned same = __match_any_sync(act, dig);
            if (lane == __ffs(same) - 1) atomicAdd(&hist[dig], static_cast<unsigned>(__popc(same)));
          }
        };
        if (in_regs) {
#pragma unroll
          for (int j = 0; j < kPer; ++j) count(keyr[j], threadIdx.x + j * kSelThreads < L);
        } else {
          for (int i0 = 0; i0 < L; i0 += kSelThreads) {
            const int i = i0 + threadIdx.x;
            count(i < L ? key_of(__ldcg(sv + i)) : 0u, i < L);
          }
        }
        __syncthreads();
        if (warp == 0) {
          unsigned loc[8], sum = 0;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            loc[j] = hist[lane * 8 + j];
            sum += loc[j];
          }
          unsigned incl = sum;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
          }
          const unsigned excl = incl - sum;
          if (static_cast<unsigned>(rank) >= excl && static_cast<unsigned>(rank) < incl) {
            unsigned cnt = excl;
            for (int j = 0; j < 8; ++j) {
              if (static_cast<unsigned>(rank) < cnt + loc[j]) {
                sh_prefix = prefix | (static_cast<uint32_t>(lane * 8 + j) << shift);
                sh_rank = rank - static_cast<int>(cnt);
                break;
              }
              cnt += loc[j];
            }
          }
        }
        __syncthreads();
        prefix = sh_prefix;
        rank = sh_rank;
        pmask |= 255u << shift;
      }
      const uint32_t u = (prefix & 0x80000000u) ? (prefix & 0x7FFFFFFFu) : ~prefix;
      thr = __uint_as_float(u);
    }
    for (int w = warp; w < nchunks; w += kSelWarps) {
      const int i = w * kSelRowsPerCta + lane;
      const float x = i < L ? __ldcg(sv + i) : INFINITY;
      const bool fl = i < L && (cmp ? x <= thr : x < thr);
      const unsigned m = __ballot_sync(0xffffffffu, fl);
      if (lane == 0) masks[s * nchunks + w] = m;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      ticket[1 + s] = 0u;  // re-arm (stream-ordered)
      __threadfence();
      is_last = atomicAdd(ticket, 1u) == gridDim.x * gridDim.y - 1;
    }
    __syncthreads();
  }
  if (!is_last) return;
  stamp(2);
  // ---- last CTA: scan all masks (b * nchunks words) and emit the packed list
  __threadfence();
  const int nwords = batch * nchunks;
  __shared__ int seq_base[1025];
  // per-sequence counts (one warp per sequence, strided)
  for (int sq = warp; sq < batch; sq += kSelWarps) {
    int c = 0;
    for (int w = lane; w < nchunks; w += 32) c += __popc(__ldcg(masks + sq * nchunks + w));
    c = warp_sum_i(c);
    if (lane == 0) seq_base[sq + 1] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    seq_base[0] = 0;
    for (int sq = 0; sq < batch; ++sq) seq_base[sq + 1] += seq_base[sq];
  }
  __syncthreads();
  for (int sq = threadIdx.x; sq <= batch; sq += blockDim.x) {
    off_out[sq] = seq_base[sq];
    if (counts_out && sq < batch) counts_out[sq] = seq_base[sq + 1] - seq_base[sq];
  }
  // each warp handles one sequence at a time: prefix over its words via ballots of popcounts
  for (int sq = warp; sq < batch; sq += kSelWarps) {
    int base = seq_base[sq];
    for (int w0 = 0; w0 < nchunks; w0 += 32) {
      const int w = w0 + lane;
      const unsigned m = (w < nchunks) ? __ldcg(masks + sq * nchunks + w) : 0u;
      int cnt = __popc(m);
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      int pos = base + incl - cnt;
      unsigned mm = m;
      while (mm) {
        const int bit = __ffs(mm) - 1;
        mm &= mm - 1;
        idx_out[pos++] = sq * N + row_lo + w * kSelRowsPerCta + bit;
      }
      base += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
  (void)nwords;
  if (threadIdx.x == 0) *ticket = 0u;  // re-arm for the next launch (stream-ordered)
  stamp(3);
}

// ============================================================================ TP: loopback all-reduce
// Sum over the G shards of a group driven by one process on one device: element e
// of every shard's buffer becomes sum_g buf_g[e], added in shard order 0..G-1 (fp32, one rounding
// for bf16 buffers), so every shard holds bit-identical results. Rows from a device count.
__global__ void tp_reduce_kernel(TpPtrs ptrs, int G, const int *__restrict__ M_ptr, int M_cap, int width, int f32) {
  pdl_wait();
  const int M = M_ptr ? min(*M_ptr, M_cap) : M_cap;
  const int64_t n = static_cast<int64_t>(M) * width;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float acc = 0.f;
    if (f32) {
      for (int g = 0; g < G; ++g) acc += static_cast<const float *>(ptrs.p[g])[e];
      for (int g = 0; g < G; ++g) static_cast<float *>(ptrs.p[g])[e] = acc;
    } else {
      for (int g = 0; g < G; ++g) acc += bf2f(static_cast<const bf16 *>(ptrs.p[g])[e]);
      const bf16 v = f2bf(acc);
      for (int g = 0; g < G; ++g) static_cast<bf16 *>(ptrs.p[g])[e] = v;
    }
  }
}

// ============================================================================ a9: unmasking
// Candidate rows = masked positions of the active semi-AR block of each sequence (D13).
__global__ void lm_candidates_kernel(const int *__restrict__ tokens, int batch, int L_P, int L_R, int block,
                                     int mask_id, int *__restrict__ rows, int *__restrict__ off) {
  pdl_wait();
  // single CTA, one warp per sequence for the search; counts then prefix
  __shared__ int cnt[1024];
  __shared__ int blk_of[1024];
  const int N = L_P + L_R;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  for (int s = warp; s < batch; s += nw) {
    int found = -1;
    for (int k = 0; k < L_R / block && found < 0; ++k) {
      bool any = false;
      for (int j = lane; j < block; j += 32) any |= tokens[s * N + L_P + k * block + j] == mask_id;
      if (__any_sync(0xffffffffu, any)) found = k;
    }
    int c = 0;
    if (found >= 0)
      for (int j = lane; j < block; j += 32) c += tokens[s * N + L_P + found * block + j] == mask_id;
    c = warp_sum_i(c);
    if (lane == 0) {
      cnt[s] = c;
      blk_of[s] = found;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int s = 0; s < batch; ++s) {
      off[s] = acc;
      acc += cnt[s];
    }
    off[batch] = acc;
  }
  __syncthreads();
  for (int s = warp; s < batch; s += nw) {
    const int k = blk_of[s];
    if (k < 0) continue;
    int base = off[s];
    for (int j0 = 0; j0 < block; j0 += 32) {
      const int j = j0 + lane;
      const int p = L_P + k * block + j;
      const bool m = j < block && tokens[s * N + p] == mask_id;
      const unsigned bal = __ballot_sync(0xffffffffu, m);
      if (m) rows[base + __popc(bal & ((1u << lane) - 1))] = s * N + p;
      base += __popc(bal);
    }
  }
}

// Reduce the LM-head partials of each candidate row to (max, sumexp, argmax), confidence =
// max softmax probability = 1 / sum exp(z - max); choose the n_u most confident rows per
// sequence (ties: lowest position), commit the argmax token (ties: lowest id), record the
// decoded rows and refresh H_0 for them (Alg. 1).
__global__ void lm_select_commit_kernel(const float4 *__restrict__ partials, int n_tiles,
                                        const int *__restrict__ rows, const int *__restrict__ off, int n_u,
                                        int *__restrict__ tokens, int *__restrict__ dec_pos,
                                        int *__restrict__ dec_tok, const bf16 *__restrict__ emb,
                                        bf16 *__restrict__ H0, int d, float *__restrict__ H0f) {
  pdl_wait();
  __shared__ float conf[256];
  __shared__ int tok[256];
  __shared__ int chosen[64];
  const int s = blockIdx.x;
  const int b0 = off[s], n = off[s + 1] - b0;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  for (int i = warp; i < n && i < 256; i += nw) {
    const float4 *pr = partials + static_cast<int64_t>(b0 + i) * n_tiles;
    float m = -INFINITY, sm = 0.f;
    int a = 0x7fffffff;
    for (int t = lane; t < n_tiles; t += 32) {
      const float4 v = pr[t];
      const int av = __float_as_int(v.z);
      if (v.x > m) {
        sm = sm * __expf(m - v.x) + v.y;
        m = v.x;
        a = av;
      } else {
        sm += v.y * __expf(v.x - m);
        if (v.x == m && av < a) a = av;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
      const float s2 = __shfl_xor_sync(0xffffffffu, sm, o);
      const int a2 = __shfl_xor_sync(0xffffffffu, a, o);
      const float mn = fmaxf(m, m2);
      const float snew = (m == -INFINITY ? 0.f : sm * __expf(m - mn)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mn));
      int an;
      if (m2 > m) an = a2;
      else if (m > m2) an = a;
      else an = min(a, a2);
      m = mn;
      sm = snew;
      a = an;
    }
    if (lane == 0) {
      conf[i] = 1.f / sm;
      tok[i] = a;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int take = min(n_u, n);
    for (int j = 0; j < n_u; ++j) {
      dec_pos[s * n_u + j] = -1;
      dec_tok[s * n_u + j] = -1;
    }
    for (int j = 0; j < take; ++j) {
      int best = -1;
      for (int i = 0; i < n; ++i) {
        bool used = false;
        for (int q = 0; q < j; ++q) used |= chosen[q] == i;
        if (used) continue;
        if (best < 0 || conf[i] > conf[best] || (conf[i] == conf[best] && rows[b0 + i] < rows[b0 + best])) best = i;
      }
      chosen[j] = best;
      const int r = rows[b0 + best];
      dec_pos[s * n_u + j] = r;
      dec_tok[s * n_u + j] = tok[best];
      tokens[r] = tok[best];
    }
  }
  __syncthreads();
  const int take = min(n_u, n);
  for (int j = warp; j < take; j += nw) {
    const int r = dec_pos[s * n_u + j];
    const int t = dec_tok[s * n_u + j];
    if (H0f) {  // fp32-parity mode (dtype 1)
      for (int c = lane; c < d; c += 32) H0f[static_cast<int64_t>(r) * d + c] = bf2f(emb[static_cast<int64_t>(t) * d + c]);
      continue;
    }
    const uint4 *src = reinterpret_cast<const uint4 *>(emb + static_cast<int64_t>(t) * d);
    uint4 *dst = reinterpret_cast<uint4 *>(H0 + static_cast<int64_t>(r) * d);
    for (int c = lane; c < d / 8; c += 32) dst[c] = src[c];
  }
}

// ============================================================================ K8: IH4 init
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ bf16 ih4_value(uint64_t key, uint64_t i, float scale) {
  const uint64_t h = mix64(key + i);
  const int S = static_cast<int>((h & 0xFFFF) + ((h >> 16) & 0xFFFF) + ((h >> 32) & 0xFFFF) + (h >> 48));
  return __float2bfloat16_rn(__fmul_rn(static_cast<float>(S - 131070), scale));
}
// dst[(row_off + r) * cols + c] = IH4(key, (src_row(r)) * cols + c); rows listed by an optional
// interleave: il > 0 -> dst row r belongs to stream A if (r % (2*il)) < il else stream B, with
// source row (r / (2*il)) * il + r % il  (gate/up interleave of the SwiGLU GEMM, blocks of il).
__global__ void ih4_fill_kernel(bf16 *__restrict__ dst, int64_t rows, int cols, uint64_t keyA, uint64_t keyB,
                                int il, float scale) {
  pdl_wait();
  const int64_t n = rows * cols;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = e / cols, c = e - r * cols;
    uint64_t key = keyA;
    int64_t sr = r;
    if (il > 0) {
      const int64_t blk = r / (2 * il), w = r % (2 * il);
      key = (w < il) ? keyA : keyB;
      sr = blk * il + (w % il);
    }
    dst[e] = ih4_value(key, static_cast<uint64_t>(sr * cols + c), scale);
  }
}
__global__ void fill_const_kernel(bf16 *__restrict__ dst, int64_t n, float v) {
  pdl_wait();
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[e] = __float2bfloat16_rn(v);
}

// ============================================================================ launch wrappers
// Row kernels read their row count from device memory, so the grid is sized for the capacity;
// it is capped at two CTAs per SM (grid-stride loops) so that a small device count does not pay
// for launching and retiring thousands of empty CTAs.
static inline int grid_for(int64_t work, int per_block, int cap = 148 * 2) {
  int64_t g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  return static_cast<int>(g < cap ? g : cap);
}

void launch_embed_rows(const int *tokens, const int *rows, const int *M_ptr, int M_cap, const bf16 *emb, bf16 *H0,
                       int d, cudaStream_t st) {
  DY_CUDA_LAUNCH(launch_k(embed_rows_kernel, dim3(grid_for(M_cap, 8)), dim3(256), 0, st, 1, tokens, rows, M_ptr, M_cap, emb, H0, d));
}
void launch_gather_rmsnorm(const bf16 *src, const int *idx, const int *M_ptr, int M_cap, const bf16 *g, float eps,
                           bf16 *dst, int d, cudaStream_t st, RowMark mk) {
  DY_CUDA_LAUNCH(launch_k(gather_rmsnorm_kernel, dim3(grid_for(M_cap, 4, 148 * 4)), dim3(128), 0, st, 1, src, idx, M_ptr, M_cap, g, eps, dst, d, mk));
}
void launch_gather_rows(const bf16 *src, const int *idx, const int *M_ptr, int M_cap, bf16 *dst, int width,
                        cudaStream_t st) {
  DY_CUDA_LAUNCH(launch_k(gather_rows_kernel, dim3(grid_for(M_cap, 8)), dim3(256), 0, st, 1, src, idx, M_ptr, M_cap, dst, width));
}
void launch_scatter_rows(const bf16 *src, const int *idx, const int *M_ptr, int M_cap, bf16 *dst, int width,
                         cudaStream_t st) {
  DY_CUDA_LAUNCH(launch_k(scatter_rows_kernel, dim3(grid_for(M_cap, 8)), dim3(256), 0, st, 1, src, idx, M_ptr, M_cap, dst, width));
}
void launch_rmsnorm_rows(const bf16 *src, const int *M_ptr, int M_cap, const bf16 *g, float eps, bf16 *dst, int d,
                         cudaStream_t st) {
  DY_CUDA_LAUNCH(launch_k(gather_rmsnorm_kernel, dim3(grid_for(M_cap, 4, 148 * 4)), dim3(128), 0, st, 1, src, nullptr, M_ptr, M_cap, g, eps, dst, d, RowMark{}));
}
void launch_qkv_post(const bf16 *qkv, const int *idx, const int *M_ptr, int M_cap, const bf16 *bias, int N, int H,
                     int KVH, int hd, const float2 *rope_cs, bf16 *Qc, bf16 *Kc, bf16 *Vc, bf16 *dV, bf16 *Qx,
                     bf16 *Kx, bf16 *Kxo, uint32_t *rowflag, uint32_t tag, cudaStream_t st, int q_only, bf16 *Kfi,
                     uint32_t *dtag, uint32_t epoch) {
  const int g = M_cap < 148 * 4 ? M_cap : 148 * 4;  // one row per CTA per pass; capped like grid_for
  const int work = std::max((H + KVH) * (hd / 16), KVH * hd / 8);  // vectors per row of each part
#ifndef DYLLM_QKVPOST_THREADS
#define DYLLM_QKVPOST_THREADS 256  // two work items per thread, every row of a response-only step resident at once
#endif
  const int threads = std::min(DYLLM_QKVPOST_THREADS, std::max(32, (work + 31) / 32 * 32));
  DY_CUDA_LAUNCH(launch_k(qkv_post_kernel, dim3(g > 0 ? g : 1), dim3(threads), 0, st, 1, qkv, idx, M_ptr, M_cap, bias, N, H, KVH, hd, rope_cs, Qc, Kc, Vc,
                                                 dV, Qx, Kx, Kxo, rowflag, tag, q_only, Kfi, dtag, epoch));
}
void launch_build_u(const int *idx_in, const int *off_in, const uint32_t *rowflag, uint32_t tag, const uint32_t *dtag,
                    uint32_t epoch, const bf16 *K, const bf16 *Kfi, int batch, int N, int kw, int *urows, bf16 *Kun,
                    bf16 *Kuo, int *ucnt, cudaStream_t st) {
  DY_CUDA_LAUNCH(launch_k(build_u_kernel, dim3(batch, kUgrp), dim3(256), 0, st, 1, idx_in, off_in, rowflag, tag, dtag, epoch, K,
                          Kfi, N, kw, urows, Kun, Kuo, ucnt));
}
void launch_rope_table(float2 *cs, int N, int hd, double theta, cudaStream_t st) {
  DY_CUDA_LAUNCH(launch_k(rope_table_kernel, dim3(148), dim3(256), 0, st, 1, cs, N, hd, theta));
}
void launch_approx_rows(const int *idx_in, const int *off_in, int batch, int N, int row_lo, int *ap_rows,
                        int *ap_off, cudaStream_t st) {
  DY_CUDA_LAUNCH(launch_k(approx_rows_kernel, dim3(batch), dim3(256), N, st, 1, idx_in, off_in, N, row_lo, ap_rows, ap_off, batch, 0));
}
void launch_build_list(int mode, const int *carried, const int *carried_off, const int *dec_pos, int n_u, int policy,
                       int batch, int N, int row_lo, int resp_lo, int *out, int *out_off, cudaStream_t st) {
  DY_CUDA_LAUNCH(launch_k(build_list_kernel, dim3(1), dim3(1024), N, st, 1, mode, carried, carried_off, dec_pos, n_u, policy, batch, N, row_lo, resp_lo,
                                        out, out_off));
}
void launch_select(const bf16 *c_new, bf16 *c_cache, int batch, int N, int row_lo, int width, float tau, int cmp,
                   float frac, int *idx_out, int *off_out, float *sim_out, unsigned *masks, unsigned *ticket,
                   int *counts, const uint32_t *rowflag, uint32_t tag, const int *dl_off, cudaStream_t st,
                   const float4 *cos_part, int H, float4 *part_out) {
  const int L = N - row_lo;
  dim3 grid((L + kSelRowsPerCta - 1) / kSelRowsPerCta, batch);
  const bool wide = L > 512;
  DY_CUDA_LAUNCH(launch_k(wide ? select_salient_kernel<256> : select_salient_kernel<512>, dim3(grid),
                          dim3(wide ? 256 : 512), 0, st, 1, c_new, c_cache, N, row_lo, width, tau, cmp, frac, idx_out,
                          off_out, sim_out, masks, ticket, counts, rowflag, tag, dl_off, cos_part, H, part_out,
                          g_sel_trace));
}
void launch_lm_candidates(const int *tokens, int batch, int L_P, int L_R, int block, int mask_id, int *rows, int *off,
                          cudaStream_t st) {
  DY_CUDA_LAUNCH(launch_k(lm_candidates_kernel, dim3(1), dim3(1024), 0, st, 1, tokens, batch, L_P, L_R, block, mask_id, rows, off));
}
void launch_lm_select_commit(const float4 *partials, int n_tiles, const int *rows, const int *off, int batch, int n_u,
                             int *tokens, int *dec_pos, int *dec_tok, const bf16 *emb, bf16 *H0, int d,
                             cudaStream_t st, float *H0f) {
  DY_CUDA_LAUNCH(launch_k(lm_select_commit_kernel, dim3(batch), dim3(256), 0, st, 1, partials, n_tiles, rows, off, n_u, tokens, dec_pos, dec_tok, emb, H0,
                                                 d, H0f));
}
void launch_tp_reduce(const TpPtrs &ptrs, int G, const int *M_ptr, int M_cap, int width, int f32, cudaStream_t st) {
  DY_CUDA_LAUNCH(launch_k(tp_reduce_kernel, dim3(148 * 4), dim3(256), 0, st, 1, ptrs, G, M_ptr, M_cap, width, f32));
}
void launch_ih4_fill(bf16 *dst, int64_t rows, int cols, uint64_t keyA, uint64_t keyB, int il, float scale,
                     cudaStream_t st) {
  DY_CUDA_LAUNCH(launch_k(ih4_fill_kernel, dim3(148 * 8), dim3(256), 0, st, 1, dst, rows, cols, keyA, keyB, il, scale));
}
void launch_fill_const(bf16 *dst, int64_t n, float v, cudaStream_t st) {
  DY_CUDA_LAUNCH(launch_k(fill_const_kernel, dim3(148 * 4), dim3(256), 0, st, 1, dst, n, v));
}

}  // namespace dy
