// attn.cu — salient-query attention over the full bidirectional K/V.
//
// For every (sequence, head) the input rows are split into two homogeneous lists:
//   exact rows  (= idx_in):  C = softmax(Q K^T / sqrt(d_h)) V        over all N keys
//   approx rows (input \ idx_in, Alg. 4):
//       pass 1: row max / sum-exp of softmax(Q K^T / sqrt(d_h)) over all N keys (dense scores, D7)
//       pass 2: dC = softmax(...)[:, idx_in] dV over the salient keys only, C = C_cache + dC
// K and V are the merged caches (salient rows already overwritten by qkv_post);
// dV is compact and aligned with the packed idx_in list.
//
// CTA = 4 warps x 16 query rows (64-row q tile), 64-key tiles double-buffered with cp.async,
// bf16 m16n8k16 tensor-core MMA with fp32 accumulation, online softmax in exp2 domain.
// (Round-1 kernel: the SIMT-issued mma.sync path; a tcgen05/TMEM version is the planned upgrade.)
#include "common.cuh"
#include "internal.h"

namespace dy {

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3, const void *p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3, const void *p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void mma16816(float d[4], const uint32_t a[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

constexpr int BQ = 64;
constexpr int BKEY = 64;

template <int HD>
struct AttnSmem {
  static constexpr int LD = HD + 8;  // padded row (16B-aligned, ldmatrix bank-conflict free)
  static constexpr int BYTES = (BQ * LD + 4 * BKEY * LD) * 2;
};

// load a 64-row tile of `width`-wide rows (head slice at column col0) into smem rows [0,64)
template <int HD>
__device__ __forceinline__ void load_rows_tile(bf16 *dst, const bf16 *base, int64_t ld, int col0, const int *rows,
                                               int n_valid, int tid) {
  constexpr int LD = AttnSmem<HD>::LD;
  constexpr int CH = HD / 8;
  for (int e = tid; e < BKEY * CH; e += 128) {
    const int r = e / CH, c = e - r * CH;
    const bool ok = r < n_valid;
    const int64_t row = ok ? rows[r] : 0;
    cp_async16(dst + r * LD + c * 8, base + row * ld + col0 + c * 8, ok);
  }
}
// contiguous key rows [k0, k0+64) of one sequence (row ids s*N + k)
template <int HD>
__device__ __forceinline__ void load_seq_tile(bf16 *dst, const bf16 *base, int64_t ld, int col0, int64_t row0,
                                              int n_valid, int tid) {
  constexpr int LD = AttnSmem<HD>::LD;
  constexpr int CH = HD / 8;
  for (int e = tid; e < BKEY * CH; e += 128) {
    const int r = e / CH, c = e - r * CH;
    const bool ok = r < n_valid;
    cp_async16(dst + r * LD + c * 8, base + (row0 + (ok ? r : 0)) * ld + col0 + c * 8, ok);
  }
}

// S[8][4] = Q(16 x HD, regs) * K_tile^T (64 keys)
template <int HD>
__device__ __forceinline__ void qk_tile(float S[8][4], const uint32_t qf[HD / 16][4], const bf16 *sK, int lane) {
  constexpr int LD = AttnSmem<HD>::LD;
#pragma unroll
  for (int nb = 0; nb < 8; ++nb)
#pragma unroll
    for (int e = 0; e < 4; ++e) S[nb][e] = 0.f;
#pragma unroll
  for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
    for (int nb2 = 0; nb2 < 4; ++nb2) {
      uint32_t b0, b1, b2, b3;
      const int key = nb2 * 16 + (lane / 16) * 8 + (lane % 8);
      const int col = kk * 16 + ((lane / 8) % 2) * 8;
      ldsm_x4(b0, b1, b2, b3, sK + key * LD + col);
      mma16816(S[2 * nb2], qf[kk], b0, b1);
      mma16816(S[2 * nb2 + 1], qf[kk], b2, b3);
    }
  }
}

// O[HD/8][4] += P(16 x 64, regs as bf16) * V_tile(64 x HD)
template <int HD>
__device__ __forceinline__ void pv_tile(float O[HD / 8][4], const float P[8][4], const bf16 *sV, int lane) {
  constexpr int LD = AttnSmem<HD>::LD;
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    uint32_t a[4];
    a[0] = pack2(P[2 * kk][0], P[2 * kk][1]);
    a[1] = pack2(P[2 * kk][2], P[2 * kk][3]);
    a[2] = pack2(P[2 * kk + 1][0], P[2 * kk + 1][1]);
    a[3] = pack2(P[2 * kk + 1][2], P[2 * kk + 1][3]);
#pragma unroll
    for (int dn2 = 0; dn2 < HD / 16; ++dn2) {
      uint32_t b0, b1, b2, b3;
      const int key = kk * 16 + (lane % 8) + ((lane / 8) % 2) * 8;
      const int col = dn2 * 16 + (lane / 16) * 8;
      ldsm_x4_t(b0, b1, b2, b3, sV + key * LD + col);
      mma16816(O[2 * dn2], a, b0, b1);
      mma16816(O[2 * dn2 + 1], a, b2, b3);
    }
  }
}

template <int HD>
__global__ void __launch_bounds__(128) attn_kernel(const AttnArgs a) {
  constexpr int LD = AttnSmem<HD>::LD;
  extern __shared__ __align__(16) uint8_t attn_smem[];
  bf16 *sQ = reinterpret_cast<bf16 *>(attn_smem);
  bf16 *sK = sQ + BQ * LD;          // [2][64][LD]
  bf16 *sV = sK + 2 * BKEY * LD;    // [2][64][LD]

  const int T = gridDim.x / 2;
  const bool exact = blockIdx.x < static_cast<unsigned>(T);
  const int tile = exact ? blockIdx.x : blockIdx.x - T;
  const int h = blockIdx.y, s = blockIdx.z;
  const int *list = exact ? a.ex_rows : a.ap_rows;
  const int *off = exact ? a.ex_off : a.ap_off;
  const int l0 = off[s];
  const int nrows = off[s + 1] - l0;
  const int q0 = tile * BQ;
  if (q0 >= nrows) return;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int g = lane / 4, t4 = lane % 4;
  const int kvh = h / (a.H / a.KVH);
  const int64_t qw = static_cast<int64_t>(a.H) * HD, kw = static_cast<int64_t>(a.KVH) * HD;
  const int N = a.N;
  const float sl2 = a.scale * 1.4426950408889634f;
  const int qrows = min(BQ, nrows - q0);
  const int *qlist = list + l0 + q0;

  // ---- Q tile
  load_rows_tile<HD>(sQ, a.Q, qw, h * HD, qlist, qrows, tid);
  const int64_t seq_row0 = static_cast<int64_t>(s) * N;
  const int nk = (N + BKEY - 1) / BKEY;
  load_seq_tile<HD>(sK, a.K, kw, kvh * HD, seq_row0, min(BKEY, N), tid);
  if (exact) load_seq_tile<HD>(sV, a.V, kw, kvh * HD, seq_row0, min(BKEY, N), tid);
  cp_commit();

  uint32_t qf[HD / 16][4];
  float O[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) O[i][e] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};

  for (int j = 0; j < nk; ++j) {
    const int buf = j & 1;
    if (j + 1 < nk) {
      const int k1 = (j + 1) * BKEY;
      load_seq_tile<HD>(sK + (buf ^ 1) * BKEY * LD, a.K, kw, kvh * HD, seq_row0 + k1, min(BKEY, N - k1), tid);
      if (exact) load_seq_tile<HD>(sV + (buf ^ 1) * BKEY * LD, a.V, kw, kvh * HD, seq_row0 + k1, min(BKEY, N - k1), tid);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (j == 0) {
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
        ldsm_x4(qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3],
                sQ + (warp * 16 + (lane % 16)) * LD + kk * 16 + (lane / 16) * 8);
    }
    float S[8][4];
    qk_tile<HD>(S, qf, sK + buf * BKEY * LD, lane);
    // scale, mask, online softmax
    float mx[2] = {m_r[0], m_r[1]};
#pragma unroll
    for (int nb = 0; nb < 8; ++nb)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = j * BKEY + nb * 8 + 2 * t4 + (e & 1);
        S[nb][e] = key < N ? S[nb][e] * sl2 : -INFINITY;
        mx[e >> 1] = fmaxf(mx[e >> 1], S[nb][e]);
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
    }
    float corr[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      corr[r] = exp2f(m_r[r] - mx[r]);
      m_r[r] = mx[r];
      l_r[r] *= corr[r];
    }
#pragma unroll
    for (int nb = 0; nb < 8; ++nb)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float p = exp2f(S[nb][e] - m_r[e >> 1]);
        S[nb][e] = p;
        l_r[e >> 1] += p;
      }
    if (exact) {
#pragma unroll
      for (int i = 0; i < HD / 8; ++i) {
        O[i][0] *= corr[0];
        O[i][1] *= corr[0];
        O[i][2] *= corr[1];
        O[i][3] *= corr[1];
      }
      pv_tile<HD>(O, S, sV + buf * BKEY * LD, lane);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 1);
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 2);
  }

  if (!exact) {
    // ---- pass 2: salient keys only, P = exp2(s - m) / l, O = P * dV
    const int sb = a.sal_off[s];
    const int ns = a.sal_off[s + 1] - sb;
    const int nks = (ns + BKEY - 1) / BKEY;
    const float inv_l[2] = {1.f / l_r[0], 1.f / l_r[1]};
    if (nks > 0) {
      load_rows_tile<HD>(sK, a.K, kw, kvh * HD, a.sal_rows + sb, min(BKEY, ns), tid);
      load_seq_tile<HD>(sV, a.dV, kw, kvh * HD, sb, min(BKEY, ns), tid);
      cp_commit();
    }
    for (int j = 0; j < nks; ++j) {
      const int buf = j & 1;
      if (j + 1 < nks) {
        const int k1 = (j + 1) * BKEY;
        load_rows_tile<HD>(sK + (buf ^ 1) * BKEY * LD, a.K, kw, kvh * HD, a.sal_rows + sb + k1, min(BKEY, ns - k1),
                           tid);
        load_seq_tile<HD>(sV + (buf ^ 1) * BKEY * LD, a.dV, kw, kvh * HD, sb + k1, min(BKEY, ns - k1), tid);
        cp_commit();
        cp_wait<1>();
      } else {
        cp_wait<0>();
      }
      __syncthreads();
      float S[8][4];
      qk_tile<HD>(S, qf, sK + buf * BKEY * LD, lane);
#pragma unroll
      for (int nb = 0; nb < 8; ++nb)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int key = j * BKEY + nb * 8 + 2 * t4 + (e & 1);
          S[nb][e] = key < ns ? exp2f(S[nb][e] * sl2 - m_r[e >> 1]) * inv_l[e >> 1] : 0.f;
        }
      pv_tile<HD>(O, S, sV + buf * BKEY * LD, lane);
      __syncthreads();
    }
  }

  // ---- epilogue: exact -> O / l ; approx -> C_cache + O
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int qi = warp * 16 + g + r * 8;
    if (qi >= qrows) continue;
    const int64_t row = qlist[qi];
    bf16 *dst = a.C_out + row * qw + h * HD;
    const bf16 *base = a.C_cache + row * qw + h * HD;
    const float il = exact ? 1.f / l_r[r] : 1.f;
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      const int col = i * 8 + 2 * t4;
      float v0 = O[i][2 * r] * il, v1 = O[i][2 * r + 1] * il;
      if (!exact) {
        const __nv_bfloat162 c = *reinterpret_cast<const __nv_bfloat162 *>(base + col);
        v0 += __bfloat162float(c.x);
        v1 += __bfloat162float(c.y);
      }
      *reinterpret_cast<uint32_t *>(dst + col) = pack2(v0, v1);
    }
  }
}

template <int HD>
static int launch_hd(const AttnArgs &a, cudaStream_t st) {
  static bool attr = false;
  const int smem = AttnSmem<HD>::BYTES;
  if (!attr) {
    DY_CUDA(cudaFuncSetAttribute(attn_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  const int T = (a.max_rows_per_seq + BQ - 1) / BQ;
  if (T <= 0) return DYLLM_OK;
  dim3 grid(2 * T, a.H, a.batch);
  attn_kernel<HD><<<grid, 128, smem, st>>>(a);
  DY_CUDA(cudaGetLastError());
  return DYLLM_OK;
}

int attention_launch(const AttnArgs &a, cudaStream_t st) {
  switch (a.hd) {
    case 16: return launch_hd<16>(a, st);
    case 32: return launch_hd<32>(a, st);
    case 64: return launch_hd<64>(a, st);
    case 128: return launch_hd<128>(a, st);
    default:
      set_error("attention: head_dim must be 16, 32, 64 or 128");
      return DYLLM_E_SHAPE;
  }
}

}  // namespace dy
