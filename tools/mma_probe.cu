// mma_probe.cu — microbenchmark: issue-to-completion throughput of back-to-back tcgen05.mma
// (kind::f16, bf16 in, fp32 accumulate, cta_group::1) on one SM per CTA, for the operand shapes
// the fused attention kernel uses:
//   SS K-major  M=128 N=128 (S = Q K^T), SS K-major M=128 N=256,
//   TS (A from TMEM) M=128 N=128 with B MN-major (O += P V) and with B K-major.
// One thread issues ITERS MMAs (K = 16 each) on zero-filled 128B-swizzled tiles, commits to an
// mbarrier and waits; cycles / MMA vs. the tcgen05 floor of M*N/256 cycles (B300_MICROARCH.md).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_probe tools/mma_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc_k(uint32_t a) {  // K-major, SWIZZLE_128B, SBO 1024
  return static_cast<uint64_t>((a & 0x3FFFF) >> 4) | (1ull << 16) | (static_cast<uint64_t>(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint64_t desc_mn(uint32_t a, uint32_t lbo) {  // MN-major, SWIZZLE_128B
  return static_cast<uint64_t>((a & 0x3FFFF) >> 4) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (b_mn ? (1u << 16) : 0u) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

// 0: SS N=128, 1: SS N=256, 2: TS N=128 B MN-major, 3: TS N=128 B K-major, 4: SS N=32, 5: SS N=64,
// 6: SS N=32 with A MN-major (the transposed O^T = V^T P^T of the attention's type-4 tiles),
// 7 / 8: SS N=32 from one issuer alternating over 2 / 4 independent accumulators (is the ~73-cycle
// single-issuer rate an accumulate dependency or an issue cost?)
template <int MODE, int NW = 1, bool LANES = false>
__global__ void __launch_bounds__(128, 1) mma_probe(unsigned long long *out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *sm = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(NW) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int issuer = LANES ? threadIdx.x : warp;  // LANES: lanes 0..NW-1 of warp 0 (divergent)
  const uint32_t tm = slot + (issuer % NW) * 128 * (MODE == 4 || MODE == 6 || MODE == 5);
  if (LANES ? threadIdx.x < NW : (threadIdx.x % 32 == 0 && warp < NW)) {
    const uint32_t a = smem_u32(sm), b = a + 32768;
    constexpr int N = MODE == 1 ? 256 : (MODE == 4 || MODE >= 6) ? 32 : MODE == 5 ? 64 : 128;
    constexpr uint32_t id = idesc(128, N, MODE == 2) | (MODE == 6 ? (1u << 15) : 0u);
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t acc = i > 0;
      const int kk = i & 7;
      if (MODE == 6) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                     "l"(desc_mn(a + kk * 2048, 16384)), "l"(desc_k(b + (kk >> 2) * 4096 + (kk & 3) * 32)),
                     "r"(id), "r"(acc)
                     : "memory");
      } else if (MODE == 7 || MODE == 8) {
        const uint32_t dacc = tm + (MODE == 7 ? (i & 1) : (i & 3)) * 32;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dacc),
                     "l"(desc_k(a + (kk >> 2) * 16384 + (kk & 3) * 32)), "l"(desc_k(b + (kk >> 2) * 16384 + (kk & 3) * 32)),
                     "r"(id), "r"(acc)
                     : "memory");
      } else if (MODE <= 1 || MODE == 4 || MODE == 5) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                     "l"(desc_k(a + (kk >> 2) * 16384 + (kk & 3) * 32)), "l"(desc_k(b + (kk >> 2) * 16384 + (kk & 3) * 32)),
                     "r"(id), "r"(acc)
                     : "memory");
      } else {
        const uint64_t bd = MODE == 2 ? desc_mn(b + kk * 2048, 16384) : desc_k(b + (kk >> 2) * 16384 + (kk & 3) * 32);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm),
                     "r"(tm + 384 + kk * 8), "l"(bd), "r"(id), "r"(acc)
                     : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok)
                   : "r"(smem_u32(&bar))
                   : "memory");
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

template <int MODE, int NW = 1, bool LANES = false>
void run(const char *name, int sms, int floor_cyc) {
  unsigned long long *d;
  cudaMalloc(&d, sms * sizeof(unsigned long long));
  const int smem = 96 * 1024 + 1024;
  cudaFuncSetAttribute(mma_probe<MODE, NW, LANES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 8192;
  for (int rep = 0; rep < 2; ++rep) mma_probe<MODE, NW, LANES><<<sms, 128, smem>>>(d, iters);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(unsigned long long) * (sms < 148 ? sms : 148), cudaMemcpyDeviceToHost);
  double mx = 0, sum = 0;
  const int n = sms < 148 ? sms : 148;
  for (int i = 0; i < n; ++i) {
    sum += h[i];
    mx = h[i] > mx ? h[i] : mx;
  }
  printf("%-28s x%d grid=%3d: %.1f cycles/MMA per issuer (mean), %.1f (max CTA); floor %d  -> %.0f%% of floor rate\n", name, NW, sms,
         sum / n / iters, mx / iters, floor_cyc, 100.0 * floor_cyc / (sum / n / iters));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int g : {1, sms}) {
    run<0>("SS K-major M128 N128", g, 64);
    run<1>("SS K-major M128 N256", g, 128);
    run<2>("TS B MN-major M128 N128", g, 64);
    run<3>("TS B K-major M128 N128", g, 64);
    run<4>("SS K-major M128 N32", g, 16);
    run<5>("SS K-major M128 N64", g, 32);
    run<6>("SS A MN-major M128 N32", g, 16);
    run<4, 2>("SS K-major M128 N32", g, 16);
    run<5, 2>("SS K-major M128 N64", g, 32);
    run<4, 4>("SS K-major M128 N32", g, 16);
    run<4, 2, true>("SS N32 2 lanes of 1 warp", g, 16);
    run<7>("SS N32 2 accumulators", g, 16);
    run<8>("SS N32 4 accumulators", g, 16);
  }
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
