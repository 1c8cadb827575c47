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
// head_dim 64/128 (LLaDA/Dream): attn_stats_kernel (tcgen05/TMEM, TMA) computes the row max and
// sum-exp of the dense scores of every input row; attn_pv_kernel (bf16 mma.sync) then forms
// P = exp(s - m)/l only where it is multiplied: exact rows x all keys (V), approximate rows x
// salient keys (dV). head_dim 16/32 (tiny parity configs): the single fused online-softmax
// kernel attn_kernel (same math, two passes for approximate rows).
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
  pdl_wait();
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


// =========================================================================== tcgen05 row statistics
// attn_stats_kernel (head_dim 64/128): for every input row r of every (sequence, head),
//   m_r = max_j s_rj,  l_r = sum_j exp2(s_rj - m_r),   s_rj = (q_r . k_j) * scale * log2(e)
// over ALL N keys of the sequence (Alg. 4 lines 1-2: the dense softmax normaliser, D7).
// Work item = (sequence, head, 128-row tile of the step's contiguous input rows). Warp 0: TMA
// (Q tile once per item, 256-key K tiles through a 4-stage ring); warp 1: tcgen05.mma
// 128x256x16 into a double-buffered TMEM score tile; warps 2-5: tcgen05.ld rows -> online
// max / sum-exp (one thread per query row, no shuffles).
constexpr int ST_STAGES = 4;
constexpr int ST_BN = 256;

struct StatsParams {
  int N, row_lo, L, H, KVH, MT, items;
  float sl2;
  float2 *stats;
};

template <int HD>
__global__ void __launch_bounds__(192, 1)
    attn_stats_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                      const StatsParams p) {
  pdl_wait();
  constexpr int KB = HD / 64;
  constexpr int Q_KB_BYTES = 128 * 128;     // 128 rows x 64 bf16
  constexpr int K_BYTES = ST_BN * 128;      // 256 keys x 64 bf16
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t *sQ = smem;                                   // [2][KB][Q_KB_BYTES]
  uint8_t *sK = sQ + 2 * KB * Q_KB_BYTES;               // [ST_STAGES][K_BYTES]
  uint64_t *full = reinterpret_cast<uint64_t *>(sK + ST_STAGES * K_BYTES);
  uint64_t *empty = full + ST_STAGES;
  uint64_t *qfull = empty + ST_STAGES;
  uint64_t *qempty = qfull + 2;
  uint64_t *tfull = qempty + 2;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int NKT = (p.N + ST_BN - 1) / ST_BN;
  const int grp = p.H / p.KVH;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    for (int s = 0; s < ST_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&qfull[s], 1);
      mbar_init(&qempty[s], 1);
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 2 * ST_BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      int it = 0;
      for (int w = blockIdx.x; w < p.items; w += gridDim.x, ++it) {
        const int mt = w % p.MT, sh = w / p.MT, h = sh % p.H, s = sh / p.H;
        const int qb = it & 1;
        mbar_wait(&qempty[qb], ((it >> 1) & 1) ^ 1);
        mbar_expect_tx(&qfull[qb], KB * Q_KB_BYTES);
        for (int kb = 0; kb < KB; ++kb)
          tma_load_2d(sQ + (qb * KB + kb) * Q_KB_BYTES, &tmQ, &qfull[qb], h * HD + kb * 64,
                      s * p.N + p.row_lo + mt * 128);
        const int kvh = h / grp;
        for (int kt = 0; kt < NKT; ++kt)
          for (int kb = 0; kb < KB; ++kb) {
            mbar_wait(&empty[st], ph ^ 1);
            mbar_expect_tx(&full[st], K_BYTES);
            tma_load_2d(sK + st * K_BYTES, &tmK, &full[st], kvh * HD + kb * 64, s * p.N + kt * ST_BN);
            if (++st == ST_STAGES) {
              st = 0;
              ph ^= 1;
            }
          }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_bf16_f32(128, ST_BN);
    int st = 0;
    uint32_t ph = 0;
    int it = 0, tc = 0;
    for (int w = blockIdx.x; w < p.items; w += gridDim.x, ++it) {
      const int qb = it & 1;
      mbar_wait(&qfull[qb], (it >> 1) & 1);
      for (int kt = 0; kt < NKT; ++kt, ++tc) {
        const int acc = tc & 1;
        mbar_wait(&tempty[acc], ((tc >> 1) & 1) ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&full[st], ph);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a0 = smem_u32(sQ + (qb * KB + kb) * Q_KB_BYTES);
            const uint32_t b0 = smem_u32(sK + st * K_BYTES);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_bf16(tmem_base + acc * ST_BN, sw128_kmajor_desc(a0 + k * 32), sw128_kmajor_desc(b0 + k * 32),
                        idesc, (kb | k) != 0);
            umma_commit(&empty[st]);
            if (kb == KB - 1) umma_commit(&tfull[acc]);
          }
          __syncwarp();
          if (++st == ST_STAGES) {
            st = 0;
            ph ^= 1;
          }
        }
      }
      if (lane == 0) umma_commit(&qempty[qb]);
      __syncwarp();
    }
  } else {
    const int quad = warp & 3;
    int tc = 0;
    for (int w = blockIdx.x; w < p.items; w += gridDim.x) {
      const int mt = w % p.MT, sh = w / p.MT, h = sh % p.H, s = sh / p.H;
      float m = -INFINITY, l = 0.f;
      for (int kt = 0; kt < NKT; ++kt, ++tc) {
        const int acc = tc & 1;
        mbar_wait(&tfull[acc], (tc >> 1) & 1);
        tc_fence_after();
        const uint32_t tb = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + acc * ST_BN;
#pragma unroll 1
        for (int c0 = 0; c0 < ST_BN; c0 += 32) {
          float v[32];
          tmem_ld32(tb + c0, v);
          const int kbase = kt * ST_BN + c0;
          float cm = -INFINITY;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            v[j] = (kbase + j < p.N) ? v[j] * p.sl2 : -INFINITY;
            cm = fmaxf(cm, v[j]);
          }
          const float mn = fmaxf(m, cm);
          float add = 0.f;
#pragma unroll
          for (int j = 0; j < 32; ++j) add += exp2f(v[j] - mn);
          l = l * exp2f(m - mn) + add;
          m = mn;
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
      }
      const int r = mt * 128 + quad * 32 + lane;
      if (r < p.L) p.stats[(static_cast<int64_t>(s) * p.N + p.row_lo + r) * p.H + h] = make_float2(m, l);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 2 * ST_BN);
  }
}

// =========================================================================== mma.sync P.V with known stats
// attn_pv_kernel: with (m, l) of every row from attn_stats_kernel, P = exp2(s - m) / l.
//   exact CTAs  : rows of idx_in, keys = all N, O = P V,        C = O
//   approx CTAs : rows input \ idx_in, keys = idx_in, O = P dV, C = C_cache + O   (Alg. 4 lines 3-4)
template <int HD>
__global__ void __launch_bounds__(128) attn_pv_kernel(const AttnArgs a) {
  pdl_wait();
  constexpr int LD = AttnSmem<HD>::LD;
  extern __shared__ __align__(16) uint8_t attn_smem[];
  bf16 *sQ = reinterpret_cast<bf16 *>(attn_smem);
  bf16 *sK = sQ + BQ * LD;
  bf16 *sV = sK + 2 * BKEY * LD;
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
  const int sb = a.sal_off[s];
  const int nkeys = exact ? a.N : a.sal_off[s + 1] - sb;
  if (!exact && nkeys == 0) {  // no salient key: C = C_cache for these rows
    const int qrows = min(BQ, nrows - q0);
    const int64_t qw = static_cast<int64_t>(a.H) * HD;
    for (int e = threadIdx.x; e < qrows * (HD / 8); e += blockDim.x) {
      const int r = e / (HD / 8), c = e - r * (HD / 8);
      const int64_t row = list[l0 + q0 + r];
      *reinterpret_cast<uint4 *>(a.C_out + row * qw + h * HD + c * 8) =
          *reinterpret_cast<const uint4 *>(a.C_cache + row * qw + h * HD + c * 8);
    }
    return;
  }
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int g = lane / 4, t4 = lane % 4;
  const int kvh = h / (a.H / a.KVH);
  const int64_t qw = static_cast<int64_t>(a.H) * HD, kw = static_cast<int64_t>(a.KVH) * HD;
  const float sl2 = a.scale * 1.4426950408889634f;
  const int qrows = min(BQ, nrows - q0);
  const int *qlist = list + l0 + q0;
  const bool warp_active = warp * 16 < qrows;

  load_rows_tile<HD>(sQ, a.Q, qw, h * HD, qlist, qrows, tid);
  const int64_t seq_row0 = static_cast<int64_t>(s) * a.N;
  const bf16 *Vsrc = exact ? a.V : a.dV;
  auto load_kv = [&](int buf, int k0) {
    const int nv = min(BKEY, nkeys - k0);
    if (exact) {
      load_seq_tile<HD>(sK + buf * BKEY * LD, a.K, kw, kvh * HD, seq_row0 + k0, nv, tid);
      load_seq_tile<HD>(sV + buf * BKEY * LD, Vsrc, kw, kvh * HD, seq_row0 + k0, nv, tid);
    } else {
      load_rows_tile<HD>(sK + buf * BKEY * LD, a.K, kw, kvh * HD, a.sal_rows + sb + k0, nv, tid);
      load_seq_tile<HD>(sV + buf * BKEY * LD, Vsrc, kw, kvh * HD, sb + k0, nv, tid);
    }
  };
  load_kv(0, 0);
  cp_commit();
  // row statistics of this thread's two rows
  float mrow[2] = {0.f, 0.f}, ilrow[2] = {0.f, 0.f};
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int qi = warp * 16 + g + r * 8;
    if (qi < qrows) {
      const float2 st = a.stats[static_cast<int64_t>(qlist[qi]) * a.H + h];
      mrow[r] = st.x;
      ilrow[r] = 1.f / st.y;
    }
  }
  uint32_t qf[HD / 16][4];
  float O[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) O[i][e] = 0.f;
  const int nk = (nkeys + BKEY - 1) / BKEY;
  for (int j = 0; j < nk; ++j) {
    const int buf = j & 1;
    if (j + 1 < nk) {
      load_kv(buf ^ 1, (j + 1) * BKEY);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (warp_active) {
      if (j == 0) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          ldsm_x4(qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3],
                  sQ + (warp * 16 + (lane % 16)) * LD + kk * 16 + (lane / 16) * 8);
      }
      float S[8][4];
      qk_tile<HD>(S, qf, sK + buf * BKEY * LD, lane);
#pragma unroll
      for (int nb = 0; nb < 8; ++nb)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int key = j * BKEY + nb * 8 + 2 * t4 + (e & 1);
          S[nb][e] = key < nkeys ? exp2f(S[nb][e] * sl2 - mrow[e >> 1]) * ilrow[e >> 1] : 0.f;
        }
      pv_tile<HD>(O, S, sV + buf * BKEY * LD, lane);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int qi = warp * 16 + g + r * 8;
    if (qi >= qrows) continue;
    const int64_t row = qlist[qi];
    bf16 *dst = a.C_out + row * qw + h * HD;
    const bf16 *base = a.C_cache + row * qw + h * HD;
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      const int col = i * 8 + 2 * t4;
      float v0 = O[i][2 * r], v1 = O[i][2 * r + 1];
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
static int launch_fused(const AttnArgs &a, cudaStream_t st) {
  static DeviceOnce attr;
  const int smem = AttnSmem<HD>::BYTES;
  if (attr.todo()) {
    DY_CUDA(cudaFuncSetAttribute(attn_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr.done();
  }
  const int T = (a.max_rows_per_seq + BQ - 1) / BQ;
  if (T <= 0) return DYLLM_OK;
  dim3 grid(2 * T, a.H, a.batch);
  DY_CUDA(launch_k(attn_kernel<HD>, dim3(grid), dim3(128), smem, st, 1, a));
  DY_CUDA(cudaGetLastError());
  return DYLLM_OK;
}

template <int HD>
static int launch_split(const AttnArgs &a, cudaStream_t st) {
  // 1) tcgen05 row statistics over all input rows
  constexpr int KB = HD / 64;
  const int smem_stats = 1024 + 2 * KB * 128 * 128 + ST_STAGES * ST_BN * 128 + 256;
  static DeviceOnce attr;
  if (attr.todo()) {
    DY_CUDA(cudaFuncSetAttribute(attn_stats_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_stats));
    DY_CUDA(cudaFuncSetAttribute(attn_pv_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 AttnSmem<HD>::BYTES));
    attr.done();
  }
  const int rows_total = a.batch * a.N;
  CUtensorMap tq, tk;
  int rc = make_tmap(&tq, a.Q, rows_total, a.H * HD, 128);
  if (rc) return rc;
  rc = make_tmap(&tk, a.K, rows_total, a.KVH * HD, ST_BN);
  if (rc) return rc;
  StatsParams p;
  p.N = a.N;
  p.row_lo = a.row_lo;
  p.L = a.N - a.row_lo;
  p.H = a.H;
  p.KVH = a.KVH;
  p.MT = (p.L + 127) / 128;
  p.items = a.batch * a.H * p.MT;
  p.sl2 = a.scale * 1.4426950408889634f;
  p.stats = a.stats;
  const int grid = p.items < a.num_sms ? p.items : a.num_sms;
  DY_CUDA(launch_k(attn_stats_kernel<HD>, dim3(grid), dim3(192), smem_stats, st, 1, tq, tk, p));
  DY_CUDA(cudaGetLastError());
  // 2) P.V for exact rows (all keys) and approximate rows (salient keys)
  const int T = (a.max_rows_per_seq + BQ - 1) / BQ;
  dim3 g2(2 * T, a.H, a.batch);
  DY_CUDA(launch_k(attn_pv_kernel<HD>, dim3(g2), dim3(128), AttnSmem<HD>::BYTES, st, 1, a));
  DY_CUDA(cudaGetLastError());
  return DYLLM_OK;
}

bool g_attn_fused_enabled = true;
unsigned long long *g_attn_trace = nullptr;
unsigned long long *g_attn_events = nullptr;

bool attention_writes_delta(int hd) { return hd == 128 && g_attn_fused_enabled; }

int attention_launch(const AttnArgs &a, cudaStream_t st) {
  if (a.hd == 128 && g_attn_fused_enabled) return attention_fused_launch(a, st);
  switch (a.hd) {
    case 16: return launch_fused<16>(a, st);
    case 32: return launch_fused<32>(a, st);
    case 64: return a.stats ? launch_split<64>(a, st) : launch_fused<64>(a, st);
    case 128: return a.stats ? launch_split<128>(a, st) : launch_fused<128>(a, st);
    default:
      set_error("attention: head_dim must be 16, 32, 64 or 128");
      return DYLLM_E_SHAPE;
  }
}

}  // namespace dy
