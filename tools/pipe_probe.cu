// pipe_probe.cu — microbenchmark: per-SM throughput of MUFU.EX2, a 7-instruction FMA-pipe exp2
// (polynomial), and tcgen05.ld (32x32b.x32) on B200, with W warps per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipe_probe tools/pipe_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2poly(float x) {
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  const float p = fmaf(fmaf(fmaf(0.0555041f, f, 0.2402265f), f, 0.6931472f), f, 1.0f);
  return __int_as_float(__float_as_int(t) * 8388608 + __float_as_int(p));
}

template <int MODE>
__global__ void exp_probe(float *out, int iters) {
  float v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = -0.001f * (threadIdx.x + i);
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float e = MODE == 0 ? ex2f(v[i]) : ex2poly(v[i]);
      acc += e;
      v[i] = v[i] * 0.999f - 0.0001f;
    }
  }
  if (acc == 12345.f) out[threadIdx.x] = acc;
}

__global__ void tmem_probe(float *out, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(&slot)))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t base = slot + (static_cast<uint32_t>((warp & 3) * 32) << 16) + (warp >> 2) * 32;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
          "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
          "=r"(r[30]), "=r"(r[31])
        : "r"(base + (it & 3) * 64));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) acc += __uint_as_float(r[i]);
  }
  if (acc == 12345.f) out[threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(slot) : "memory");
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float *out;
  cudaMalloc(&out, 4096 * sizeof(float));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int mode = 0; mode < 2; ++mode) {
    for (int warps : {4, 8, 16, 32}) {
      float ms = 0;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) exp_probe<0><<<sms, warps * 32>>>(out, iters);
        else exp_probe<1><<<sms, warps * 32>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
      }
      const double per_sm = static_cast<double>(warps) * 32 * iters * 16 / (ms * 1e-3) / 1e9;  // G exps/s/SM
      printf("%s warps/SM=%2d: %.2f Gexp/s/SM = %.1f exp/clk/SM (at %.0f MHz nominal)\n",
             mode == 0 ? "MUFU.EX2" : "poly-exp", warps, per_sm, per_sm * 1e3 / (clk / 1e3), clk / 1e3);
    }
  }
  for (int warps : {4, 8}) {
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      tmem_probe<<<sms, warps * 32>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    const double bytes = static_cast<double>(warps) * 32 * 32 * 4 * iters;  // per SM
    printf("tcgen05.ld x32 warps/SM=%d: %.1f GB/s/SM = %.1f B/clk/SM\n", warps, bytes / (ms * 1e-3) / 1e9,
           bytes / (ms * 1e-3) / (clk * 1e3));
  }
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
