// gemm.cu — persistent, warp-specialised tcgen05/TMEM GEMM for sm_100a over a device-resident
// row count M (the variable-length salient row set).
//
//   D[M][n] = sum_k A[m][k] * W[n][k]      A: activations (K-major), W: weights [out][in] (K-major)
//
// Roles (192 threads, 1 CTA per SM):
//   warp 0      : TMA producer — one elected lane streams A/W k-blocks (64 bf16 = 128 B wide,
//                 SWIZZLE_128B) into an S-stage shared-memory ring (full/empty mbarriers).
//   warp 1      : TMEM allocator + MMA issuer — one lane issues tcgen05.mma (M=128, N=BN, K=16)
//                 into a double-buffered TMEM accumulator (2 x BN fp32 columns) and commits
//                 stage-release / accumulator-ready barriers with tcgen05.commit.
//   warps 2..5  : epilogue — tcgen05.ld 32x32b.x32 (each warp owns one 32-lane TMEM quadrant),
//                 fused epilogue (bias / residual / SiLU-gate / LM-head max-argmax-sumexp),
//                 bf16 stores straight to global.
// Tiles are scheduled persistently (tile = blockIdx.x + i*gridDim.x) with an n-grouped raster so
// concurrently running CTAs share weight tiles through L2 when M is small (weight-streaming
// regime) and share activation tiles when M is large.
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "internal.h"

namespace dy {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 bytes = one SWIZZLE_128B row
constexpr int kGemmThreads = 192;
constexpr int kGroupN = 8;
constexpr int kPrefetchKb = 8;

template <int BN>
struct GemmCfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (192 * 1024) / STAGE_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;  // double-buffered accumulator
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

struct GemmParams {
  const int *M_ptr;
  int M_cap, N, K;
  bf16 *D;
  int ldd;
  const bf16 *resid;
  int ldr;
  const int *resid_rows;
  const bf16 *bias;
  const int *out_rows;  // nullable: destination row of each output row (fused scatter-back, a8)
  float4 *partials;
  int m_skip_le;
  int excl_col;  // EPI_LMHEAD: column left out of the max / argmax (the mask token, D22), -1: none
};

__device__ __forceinline__ void tile_coords(int t, int num_m, int num_n, int &m, int &n) {
  const int per_group = num_m * kGroupN;
  const int g = t / per_group;
  const int within = t - g * per_group;
  const int gsize = min(kGroupN, num_n - g * kGroupN);
  m = within / gsize;
  n = g * kGroupN + (within - m * gsize);
}

template <int BN, int EPI>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_tcgen05_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const GemmParams p) {
  using C = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t *smem = smem_raw + ((1024 - (raw_addr & 1023)) & 1023);
  uint8_t *smA = smem;
  uint8_t *smB = smem + C::STAGES * C::A_BYTES;
  uint64_t *full_bar = reinterpret_cast<uint64_t *>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t *empty_bar = full_bar + C::STAGES;
  uint64_t *tfull_bar = empty_bar + C::STAGES;
  uint64_t *tempty_bar = tfull_bar + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty_bar + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // setup above overlaps the previous kernel; the whole grid is resident (grid <= #SMs, one CTA
  // per SM), so the next kernel may be released now
  pdl_wait();
  pdl_trigger();

  const int M = p.M_ptr ? min(*p.M_ptr, p.M_cap) : p.M_cap;
  const int num_m = (M + BM - 1) / BM;
  const int num_n = (p.N + BN - 1) / BN;
  const int total = (M <= p.m_skip_le) ? 0 : num_m * num_n;  // small M: the skinny kernel runs
  const int num_kb = p.K / BK;

  if (warp == 0) {
    // ===================== TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int mb, nb;
        tile_coords(t, num_m, num_n, mb, nb);
        // weight tiles: L2 prefetch kPrefetchKb k-blocks ahead of the shared-memory ring
        for (int kb = 0; kb < kPrefetchKb && kb < num_kb; ++kb) tma_prefetch_l2_2d(&tmB, kb * BK, nb * BN);
        for (int kb = 0; kb < num_kb; ++kb) {
          if (kb + kPrefetchKb < num_kb) tma_prefetch_l2_2d(&tmB, (kb + kPrefetchKb) * BK, nb * BN);
          mbar_wait(&empty_bar[stage], phase ^ 1);
          mbar_expect_tx(&full_bar[stage], C::STAGE_BYTES);
          tma_load_2d(smA + stage * C::A_BYTES, &tmA, &full_bar[stage], kb * BK, mb * BM);
          tma_load_2d(smB + stage * C::B_BYTES, &tmB, &full_bar[stage], kb * BK, nb * BN);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer
    constexpr uint32_t idesc = idesc_bf16_f32(BM, BN);
    int stage = 0;
    uint32_t phase = 0;
    int local = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t dtm = tmem_base + acc * BN;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a0 = smem_u32(smA + stage * C::A_BYTES);
          const uint32_t b0 = smem_u32(smB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            umma_bf16(dtm, sw128_kmajor_desc(a0 + k * 32), sw128_kmajor_desc(b0 + k * 32), idesc,
                      (kb | k) != 0);
          }
          umma_commit(&empty_bar[stage]);
          if (kb == num_kb - 1) umma_commit(&tfull_bar[acc]);
        }
        __syncwarp();
        if (++stage == C::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else {
    // ===================== epilogue warps 2..5
    const int quad = warp & 3;
    int local = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
      int mb, nb;
      tile_coords(t, num_m, num_n, mb, nb);
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row = mb * BM + quad * 32 + lane;
      const bool row_ok = row < M;
      const uint32_t tbase = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + acc * BN;
      if constexpr (EPI == EPI_SWIGLU) {
        // tile = [g64 | u64 | g64 | u64] (kGuIl = 64): channels nb*128 + [0,64) and + [64,128)
#pragma unroll 1
        for (int c0 = 0; c0 < BN / 2; c0 += 32) {
          const int gcol = (c0 < kGuIl) ? c0 : c0 + kGuIl;  // gate column in the tile
          float g[32], u[32];
          tmem_ld32(tbase + gcol, g);
          tmem_ld32(tbase + gcol + kGuIl, u);
          if (row_ok) {
            const int col = nb * (BN / 2) + c0;
            bf16 *dst = p.D + static_cast<int64_t>(p.out_rows ? p.out_rows[row] : row) * p.ldd + col;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float o[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float gv = g[q * 8 + j];
                o[j] = gv / (1.f + __expf(-gv)) * u[q * 8 + j];
              }
              reinterpret_cast<uint4 *>(dst)[q] = pack8(o);
            }
          }
        }
      } else if constexpr (EPI == EPI_LMHEAD) {
        // per row and 256-column tile: max and argmax over the columns except the mask token
        // (D22: [M] is never a prediction), sum of exp(z - max) over every column (the
        // probability of the chosen token is normalised over the whole vocabulary)
        float mx = -INFINITY, sm = 0.f, zx = -INFINITY;
        int arg = 0;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          float v[32];
          tmem_ld32(tbase + c0, v);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int col = nb * BN + c0 + j;
            if (col == p.excl_col) {
              zx = v[j];
            } else if (col < p.N) {
              const float z = v[j];
              if (z > mx) {
                sm = sm * __expf(mx - z) + 1.f;
                mx = z;
                arg = col;
              } else {
                sm += __expf(z - mx);
              }
            }
          }
        }
        if (zx > -INFINITY && mx > -INFINITY) sm += __expf(zx - mx);
        if (row_ok) p.partials[static_cast<int64_t>(row) * num_n + nb] = make_float4(mx, sm, __int_as_float(arg), 0.f);
      } else {
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          float v[32];
          tmem_ld32(tbase + c0, v);
          if (row_ok) {
            const int colb = nb * BN + c0;
            bf16 *dst = p.D + static_cast<int64_t>(p.out_rows ? p.out_rows[row] : row) * p.ldd + colb;
            const bf16 *res = nullptr;
            if constexpr (EPI == EPI_RESID) {
              const int rr = p.resid_rows ? p.resid_rows[row] : row;
              res = p.resid + static_cast<int64_t>(rr) * p.ldr + colb;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (colb + q * 8 < p.N) {
                float o[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) o[j] = v[q * 8 + j];
                if (p.bias) {
                  float b[8];
                  unpack8(*reinterpret_cast<const uint4 *>(p.bias + colb + q * 8), b);
#pragma unroll
                  for (int j = 0; j < 8; ++j) o[j] += b[j];
                }
                if constexpr (EPI == EPI_RESID) {
                  float r[8];
                  unpack8(*reinterpret_cast<const uint4 *>(res + q * 8), r);
#pragma unroll
                  for (int j = 0; j < 8; ++j) o[j] += r[j];
                }
                reinterpret_cast<uint4 *>(dst)[q] = pack8(o);
              }
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

int make_tmap(CUtensorMap *m, const void *ptr, int rows, int K, int box_rows) {
  std::call_once(g_encode_once, [] {
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!g_encode) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return DYLLM_E_CUDA;
  }
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(K) * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ") rows=" +
              std::to_string(rows) + " K=" + std::to_string(K));
    return DYLLM_E_CUDA;
  }
  return DYLLM_OK;
}

// 3D view of a [rows][K] bf16 matrix as {64, rows, K/64} (strides: row pitch, 128 B) with box
// {64, box_rows, box_chunks}: one TMA op fetches box_chunks consecutive 64-column chunks of
// box_rows rows, laid out in shared memory as [chunk][row][64] (each chunk a 128B-swizzled
// K-major tile). TMA issue throughput is per operation (~3 ops/us per issuing thread, measured:
// tools/tma_probe.cu), so wide boxes matter more than stage count.
int make_tmap3(CUtensorMap *m, const void *ptr, int rows, int K, int box_rows, int box_chunks) {
  std::call_once(g_encode_once, [] {
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!g_encode) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return DYLLM_E_CUDA;
  }
  cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(K / 64)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(K) * 2, 128};
  cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_rows), static_cast<cuuint32_t>(box_chunks)};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(ptr), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (3d) failed (" + std::to_string(static_cast<int>(r)) + ") rows=" +
              std::to_string(rows) + " K=" + std::to_string(K));
    return DYLLM_E_CUDA;
  }
  return DYLLM_OK;
}

template <int BN, int EPI>
static int launch_t(const GemmCall &g, int num_sms, cudaStream_t st) {
  using C = GemmCfg<BN>;
  auto kern = gemm_tcgen05_kernel<BN, EPI>;
  static DeviceOnce attr_done;
  if (attr_done.todo()) {
    DY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES));
    attr_done.done();
  }
  CUtensorMap ta, tb;
  int rc = make_tmap(&ta, g.A, g.M_cap, g.K, BM);
  if (rc) return rc;
  rc = make_tmap(&tb, g.W, g.N, g.K, BN);
  if (rc) return rc;
  GemmParams p{g.M_ptr, g.M_cap, g.N, g.K, g.D, g.ldd, g.resid, g.ldr, g.resid_rows, g.bias, g.out_rows, g.partials,
               g.m_skip_le, g.excl_col};
  const int max_tiles = ((g.M_cap + BM - 1) / BM) * ((g.N + BN - 1) / BN);
  const int grid = max_tiles < num_sms ? max_tiles : num_sms;
  DY_CUDA(launch_k(kern, dim3(grid), dim3(kGemmThreads), C::SMEM_BYTES, st, 1, ta, tb, p));
  DY_CUDA(cudaGetLastError());
  return DYLLM_OK;
}

int gemm_lmhead_ntiles(int N) { return (N + 255) / 256; }

int gemm_launch(const GemmCall &g, int num_sms, cudaStream_t st) {
  if (g.K % BK != 0 || g.N % 8 != 0 || g.M_cap <= 0) {
    set_error("gemm: unsupported shape M_cap=" + std::to_string(g.M_cap) + " N=" + std::to_string(g.N) +
              " K=" + std::to_string(g.K));
    return DYLLM_E_SHAPE;
  }
  if (g.epi == EPI_SWIGLU && g.N % 256 != 0) {
    set_error("gemm swiglu: N must be a multiple of 256");
    return DYLLM_E_SHAPE;
  }
  // Row counts <= kSkinnyMaxM (16384) go to the 2-CTA weight-stationary kernel. With a device-resident
  // count both kernels are enqueued and each exits unless the count is in its regime.
  if (g.epi == EPI_QKV && !(g_skinny_enabled && skinny_eligible(g) && g.M_cap <= kSkinnyMaxM)) {
    set_error("gemm: the fused QKV epilogue needs the skinny kernel (rows <= 16384, N % 256 == 0)");
    return DYLLM_E_ARG;
  }
  GemmCall s = g;
  if (g_skinny_enabled && skinny_eligible(g)) {
    // every row count up to 16384, the FullStep's included: the CTA-pair 256-row weight tiles move
    // 131 FLOP per L2 byte against the single-CTA 128x256 tiles' 87, and the L2 -> SM operand
    // stream (~12 TB/s, tools/tma_probe.cu) bounds both (M = 15296: QKV 1225 vs 1481 us,
    // gate/up 2417 vs 2862 us, profiles/r2/gemm_15296.txt)
    if (!g.M_ptr && g.M_cap <= kSkinnyMaxM) return gemm_skinny_launch(g, num_sms, st);
    if (g.M_ptr) {
      int rc = gemm_skinny_launch(g, num_sms, st);
      if (rc) return rc;
      if (g.M_cap <= kSkinnyMaxM) return DYLLM_OK;  // the device count can never leave the skinny range
      s.m_skip_le = kSkinnyMaxM;
    }
  }
  switch (s.epi) {
    case EPI_SWIGLU:
      return launch_t<256, EPI_SWIGLU>(s, num_sms, st);
    case EPI_LMHEAD:
      return launch_t<256, EPI_LMHEAD>(s, num_sms, st);
    case EPI_RESID:
      return s.N >= 8192 ? launch_t<256, EPI_RESID>(s, num_sms, st) : launch_t<128, EPI_RESID>(s, num_sms, st);
    default:
      return s.N >= 8192 ? launch_t<256, EPI_BF16>(s, num_sms, st) : launch_t<128, EPI_BF16>(s, num_sms, st);
  }
}

bool g_skinny_enabled = true;
bool g_pdl_enabled = true;

}  // namespace dy
