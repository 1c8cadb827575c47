// gemm_skinny.cu — weight-stationary 2-CTA (cta_group::2) tcgen05 GEMM for the small salient row
// counts of the sparse steps (M <= 512 rows, the weight-streaming
// regime of §8d.3).
//
//   D[m][n] = sum_k A[m][k] * W[n][k]     computed as D^T = W A^T:
//   MMA-M = 256 weight rows of a CTA pair (128 per CTA, its own TMEM lanes),
//   MMA-N = the activation rows (N <= 256 per instruction; two instructions cover M <= 512, each
//           CTA of the pair holding half of them, so every activation byte enters one SM per pair).
// Each weight byte is read by exactly one SM; the accumulator (128 lanes x M columns, <= 512)
// stays in TMEM for the whole K loop. Roles per CTA (192 threads): warp 0 TMA producer (both
// CTAs load their halves; the leader's full barrier counts the bytes of both), warp 1 TMEM
// allocator + (leader only) single-thread tcgen05.mma issuer with multicast commits, warps 2-5
// epilogue from the CTA's own TMEM lanes (bias / residual / SiLU-gate), transposed store.
// The kernel exits immediately when the device-side row count is 0 or > 512 (the standard
// kernel of gemm.cu covers that regime), so both kernels can be enqueued without a host sync.
#include <cudaTypedefs.h>

#include "common.cuh"
#include "internal.h"

namespace dy {

constexpr int SK_STAGES = 4;
constexpr int SK_W_BYTES = 128 * 128;        // 128 weight rows x 64 bf16
constexpr int SK_A_BYTES = 128 * 128;        // 128 activation rows x 64 bf16 (per MMA half)
constexpr int SK_STAGE = SK_W_BYTES + 2 * SK_A_BYTES;
constexpr int SK_XCH = 64 * 33 * 4;          // SwiGLU gate/up exchange buffer
constexpr int SK_SMEM = 1024 + SK_STAGES * SK_STAGE + SK_XCH + 256;
constexpr int SKINNY_MAX_M = kSkinnyMaxM;

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMA 2D load into this CTA's smem, completion counted on the LEADER CTA's barrier
__device__ __forceinline__ void tma_load_2d_pair(void *smem_dst, const void *tmap, uint64_t *bar, int c0, int c1) {
  const uint32_t leader_bar = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t *slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint64_t *bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

struct SkinnyParams {
  const int *M_ptr;
  int M_cap, N, K;
  bf16 *D;
  int ldd;
  const bf16 *resid;
  int ldr;
  const int *resid_rows;
  const bf16 *bias;
};

template <int EPI>
__global__ void __launch_bounds__(192, 1)
    gemm_skinny_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW,
                       const SkinnyParams p) {
  const int M = p.M_ptr ? min(*p.M_ptr, p.M_cap) : p.M_cap;
  if (M <= 0 || M > SKINNY_MAX_M) return;  // uniform across the cluster
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t *stages = smem;
  float *xch = reinterpret_cast<float *>(smem + SK_STAGES * SK_STAGE);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + SK_STAGES * SK_STAGE + SK_XCH);
  uint64_t *empty = full + SK_STAGES;
  uint64_t *tfull = empty + SK_STAGES;
  uint64_t *tempty = tfull + 1;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int items = p.N / 256;
  const int num_kb = p.K / 64;
  const int NA0 = (min(M, 256) + 15) & ~15;
  const int NA1 = M > 256 ? ((M - 256 + 15) & ~15) : 0;
  const uint32_t stage_tx = 2u * (SK_W_BYTES + SK_A_BYTES + (NA1 ? SK_A_BYTES : 0));

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmW);
    for (int s = 0; s < SK_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 2 * 128);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer (both CTAs)
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (int it = pair; it < items; it += npairs) {
        const int wrow = it * 256 + static_cast<int>(rank) * 128;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty[st], ph ^ 1);
          if (rank == 0) mbar_expect_tx(&full[st], stage_tx);
          uint8_t *sb = stages + st * SK_STAGE;
          tma_load_2d_pair(sb, &tmW, &full[st], kb * 64, wrow);
          tma_load_2d_pair(sb + SK_W_BYTES, &tmA, &full[st], kb * 64, static_cast<int>(rank) * (NA0 / 2));
          if (NA1)
            tma_load_2d_pair(sb + SK_W_BYTES + SK_A_BYTES, &tmA, &full[st], kb * 64,
                             256 + static_cast<int>(rank) * (NA1 / 2));
          if (++st == SK_STAGES) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA only)
    if (rank == 0) {
      const uint32_t id0 = idesc_bf16_f32(256, NA0);
      const uint32_t id1 = idesc_bf16_f32(256, NA1 ? NA1 : 16);
      int st = 0;
      uint32_t ph = 0;
      int local = 0;
      for (int it = pair; it < items; it += npairs, ++local) {
        mbar_wait(tempty, (local & 1) ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full[st], ph);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t w0 = smem_u32(stages + st * SK_STAGE);
            const uint32_t a0 = w0 + SK_W_BYTES;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              umma_bf16_pair(tmem_base, sw128_kmajor_desc(w0 + k * 32), sw128_kmajor_desc(a0 + k * 32), id0,
                             (kb | k) != 0);
              if (NA1)
                umma_bf16_pair(tmem_base + 256, sw128_kmajor_desc(w0 + k * 32),
                               sw128_kmajor_desc(a0 + SK_A_BYTES + k * 32), id1, (kb | k) != 0);
            }
            umma_commit_pair(&empty[st]);
            if (kb == num_kb - 1) umma_commit_pair(tfull);
          }
          __syncwarp();
          if (++st == SK_STAGES) {
            st = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else {
    // ===================== epilogue warps 2..5 (both CTAs, own TMEM lanes)
    const int quad = warp & 3;
    const int row = quad * 32 + lane;  // weight row within this CTA's 128
    const uint32_t leader_tempty = mapa_shared(smem_u32(tempty), 0);
    int local = 0;
    for (int it = pair; it < items; it += npairs, ++local) {
      mbar_wait(tfull, local & 1);
      tc_fence_after();
      const uint32_t tb = tmem_base + (static_cast<uint32_t>(quad * 32) << 16);
      const int n_glob = it * 256 + static_cast<int>(rank) * 128 + row;
      for (int j = 0; j < 2; ++j) {
        const int NA = j ? NA1 : NA0;
        for (int c0 = 0; c0 < NA; c0 += 32) {
          float v[32];
          tmem_ld32(tb + j * 256 + c0, v);
          const int m0 = j * 256 + c0;
          if constexpr (EPI == EPI_SWIGLU) {
            // rows [0,64): gate of channels ch0..ch0+63; rows [64,128): up of the same channels
            const int ch = (it * 2 + static_cast<int>(rank)) * 64 + (row & 63);
            if (row >= 64) {
#pragma unroll
              for (int t = 0; t < 32; ++t) xch[(row - 64) * 33 + t] = v[t];
            }
            named_bar_sync(1, 128);
            if (row < 64) {
#pragma unroll
              for (int t = 0; t < 32; ++t) {
                const int m = m0 + t;
                if (m < M) {
                  const float g = v[t], u = xch[row * 33 + t];
                  p.D[static_cast<int64_t>(m) * p.ldd + ch] = f2bf(g / (1.f + __expf(-g)) * u);
                }
              }
            }
            named_bar_sync(1, 128);
          } else {
            const float b = p.bias ? bf2f(p.bias[n_glob]) : 0.f;
#pragma unroll
            for (int t = 0; t < 32; ++t) {
              const int m = m0 + t;
              if (m < M) {
                float o = v[t] + b;
                if constexpr (EPI == EPI_RESID) {
                  const int rr = p.resid_rows ? p.resid_rows[m] : m;
                  o += bf2f(p.resid[static_cast<int64_t>(rr) * p.ldr + n_glob]);
                }
                p.D[static_cast<int64_t>(m) * p.ldd + n_glob] = f2bf(o);
              }
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive_cluster(leader_tempty);
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 512);
  }
}

template <int EPI>
static int launch_skinny_t(const GemmCall &g, int num_sms, cudaStream_t st) {
  auto kern = gemm_skinny_kernel<EPI>;
  static bool attr_done = false;
  if (!attr_done) {
    DY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SK_SMEM));
    DY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
    attr_done = true;
  }
  CUtensorMap ta, tw;
  int rc = make_tmap(&ta, g.A, g.M_cap, g.K, 128);
  if (rc) return rc;
  rc = make_tmap(&tw, g.W, g.N, g.K, 128);
  if (rc) return rc;
  SkinnyParams p{g.M_ptr, g.M_cap, g.N, g.K, g.D, g.ldd, g.resid, g.ldr, g.resid_rows, g.bias};
  const int items = g.N / 256;
  int pairs = num_sms / 2;
  if (pairs > items) pairs = items;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = SK_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DY_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tw, p));
  return DYLLM_OK;
}

bool skinny_eligible(const GemmCall &g) {
  return g.N % 256 == 0 && g.K % 64 == 0 && (g.epi == EPI_BF16 || g.epi == EPI_RESID || g.epi == EPI_SWIGLU);
}

int gemm_skinny_launch(const GemmCall &g, int num_sms, cudaStream_t st) {
  switch (g.epi) {
    case EPI_SWIGLU: return launch_skinny_t<EPI_SWIGLU>(g, num_sms, st);
    case EPI_RESID: return launch_skinny_t<EPI_RESID>(g, num_sms, st);
    default: return launch_skinny_t<EPI_BF16>(g, num_sms, st);
  }
}

}  // namespace dy
