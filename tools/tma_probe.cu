// tma_probe.cu — microbenchmark: per-SM TMA streaming bandwidth vs. stages in flight and box
// shape, from DRAM (1 GiB buffer, no reuse) and from L2 (a 32 MiB buffer re-read). One producer
// thread per CTA issues 2D tiled TMA loads (128B swizzle) into an S-stage ring; a consumer warp
// waits each stage and releases it (no compute), so the loop measures the memory pipeline alone.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_probe tools/tma_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok)
                 : "r"(smem_u32(b)), "r"(ph)
                 : "memory");
}
__device__ __forceinline__ void tma2d(void *dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma3d(void *dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// nprod producer warps (lane 0 each) with private rings of `stages`, 3D box {64, box_rows, halves}
__global__ void __launch_bounds__(256, 1) probe_mp(const __grid_constant__ CUtensorMap tm, int nprod, int stages,
                                                   int box_rows, int halves, int tiles_per_prod, int col_tiles,
                                                   int row_tiles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t *buf = smem + ((1024 - (smem_u32(smem) & 1023)) & 1023);
  const int bytes = box_rows * 128 * halves;
  uint64_t *bars = reinterpret_cast<uint64_t *>(buf + nprod * stages * bytes);
  const int w = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2 * nprod * stages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (w < nprod && threadIdx.x % 32 == 0) {
    uint64_t *full = bars + 2 * w * stages, *empty = full + stages;
    uint8_t *ring = buf + w * stages * bytes;
    int st = 0;
    uint32_t ph = 0;
    for (int i = 0; i < tiles_per_prod; ++i) {
      const long t = (static_cast<long>(blockIdx.x) * nprod + w) + static_cast<long>(i) * gridDim.x * nprod;
      const int ct = static_cast<int>(t % (col_tiles / halves)), rt = static_cast<int>((t / (col_tiles / halves)) % row_tiles);
      mbar_wait(&empty[st], ph ^ 1);
      mbar_expect_tx(&full[st], bytes);
      tma3d(ring + st * bytes, &tm, &full[st], 0, rt * box_rows, ct * halves);
      if (++st == stages) {
        st = 0;
        ph ^= 1;
      }
    }
  } else if (w >= 4 && w - 4 < nprod && threadIdx.x % 32 == 0) {
    const int pw = w - 4;
    uint64_t *full = bars + 2 * pw * stages, *empty = full + stages;
    int st = 0;
    uint32_t ph = 0;
    for (int i = 0; i < tiles_per_prod; ++i) {
      mbar_wait(&full[st], ph);
      mbar_arrive(&empty[st]);
      if (++st == stages) {
        st = 0;
        ph ^= 1;
      }
    }
  }
}

// rows x cols bf16 tensor, box {64 cols, box_rows}; CTA b streams tiles t = b, b + grid, ...
__global__ void __launch_bounds__(64, 1) probe(const __grid_constant__ CUtensorMap tm, int stages, int box_rows,
                                               int tiles_per_cta, int col_tiles, int row_tiles,
                                               unsigned long long *cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t *buf = smem + ((1024 - (smem_u32(smem) & 1023)) & 1023);
  const int bytes = box_rows * 128;
  uint64_t *full = reinterpret_cast<uint64_t *>(buf + stages * bytes);
  uint64_t *empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const unsigned long long t0 = clock64();
  if (threadIdx.x == 0) {
    int st = 0;
    uint32_t ph = 0;
    for (int i = 0; i < tiles_per_cta; ++i) {
      const long t = static_cast<long>(blockIdx.x) + static_cast<long>(i) * gridDim.x;
      const int ct = static_cast<int>(t % col_tiles), rt = static_cast<int>((t / col_tiles) % row_tiles);
      mbar_wait(&empty[st], ph ^ 1);
      mbar_expect_tx(&full[st], bytes);
      tma2d(buf + st * bytes, &tm, &full[st], ct * 64, rt * box_rows);
      if (++st == stages) {
        st = 0;
        ph ^= 1;
      }
    }
  } else if (threadIdx.x == 32) {
    int st = 0;
    uint32_t ph = 0;
    for (int i = 0; i < tiles_per_cta; ++i) {
      mbar_wait(&full[st], ph);
      mbar_arrive(&empty[st]);
      if (++st == stages) {
        st = 0;
        ph ^= 1;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = clock64() - t0;
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void **>(&enc), cudaEnableDefault, &q);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t big_rows = 131072, cols = 4096;  // 1 GiB bf16
  void *dbig = nullptr;
  cudaMalloc(&dbig, big_rows * cols * 2);
  cudaMemset(dbig, 0, big_rows * cols * 2);
  unsigned long long *cyc;
  cudaMalloc(&cyc, sms * sizeof(unsigned long long));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("source box_rows stage_KB stages inflight_KB  GB/s_total  GB/s_per_SM\n");
  for (int src = 0; src < 2; ++src) {
    const size_t rows = src == 0 ? big_rows : 4096;  // 1 GiB (DRAM) vs 32 MiB (L2-resident)
    for (int box_rows : {64, 128, 256}) {
      CUtensorMap tm;
      cuuint64_t dims[2] = {cols, rows};
      cuuint64_t strides[1] = {cols * 2};
      cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
      cuuint32_t es[2] = {1, 1};
      enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dbig, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      const int bytes = box_rows * 128;
      for (int stages : {2, 4, 6, 8, 12}) {
        if (stages * bytes > 200 * 1024) continue;
        const int col_tiles = cols / 64, row_tiles = rows / box_rows;
        const long total_tiles = static_cast<long>(col_tiles) * row_tiles;
        const int per_cta = static_cast<int>(total_tiles / sms / (src == 0 ? 1 : 1));
        const int smem = 1024 + stages * bytes + 256;
        for (int rep = 0; rep < 2; ++rep) {
          cudaEventRecord(e0);
          probe<<<sms, 64, smem>>>(tm, stages, box_rows, src == 0 ? per_cta : per_cta * 8, col_tiles, row_tiles, cyc);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double moved = static_cast<double>(src == 0 ? per_cta : per_cta * 8) * sms * bytes;
        printf("%s %4d %6d %3d %6d  %9.1f  %8.1f\n", src == 0 ? "dram" : "l2  ", box_rows, bytes / 1024, stages,
               stages * bytes / 1024, moved / ms / 1e6, moved / ms / 1e6 / sms);
      }
    }
  }
  // ---- multi-producer + 3D boxes (dims {64, rows, cols/64}, strides {pitch, 128 B})
  cudaFuncSetAttribute(probe_mp, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  printf("\nsource nprod box_rows halves op_KB stages  GB/s_total  GB/s_per_SM  ops/us/SM\n");
  for (int src = 0; src < 2; ++src) {
    const size_t rows = src == 0 ? big_rows : 4096;
    for (int halves : {1, 2, 4}) {
      for (int box_rows : {64, 128, 256}) {
        CUtensorMap tm;
        cuuint64_t dims[3] = {64, rows, cols / 64};
        cuuint64_t strides[2] = {cols * 2, 128};
        cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_rows), static_cast<cuuint32_t>(halves)};
        cuuint32_t es[3] = {1, 1, 1};
        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, dbig, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
          printf("encode failed %d (box %d x %d)\n", r, box_rows, halves);
          continue;
        }
        const int bytes = box_rows * 128 * halves;
        for (int nprod : {1, 2, 4}) {
          const int stages = (180 * 1024) / (bytes * nprod);
          if (stages < 2) continue;
          const int col_tiles = cols / 64, row_tiles = rows / box_rows;
          const long total = static_cast<long>(col_tiles / halves) * row_tiles;
          const int per_prod = static_cast<int>(total / sms / nprod) * (src == 0 ? 1 : 8);
          const int smem = 1024 + nprod * stages * bytes + 2 * nprod * stages * 8 + 64;
          for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            probe_mp<<<sms, 256, smem>>>(tm, nprod, stages, box_rows, halves, per_prod, col_tiles, row_tiles);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
          }
          float ms = 0;
          cudaEventElapsedTime(&ms, e0, e1);
          const double moved = static_cast<double>(per_prod) * nprod * sms * bytes;
          printf("%s %d %4d %d %4d %3d  %9.1f  %8.1f  %6.2f\n", src == 0 ? "dram" : "l2  ", nprod, box_rows, halves,
                 bytes / 1024, stages, moved / ms / 1e6, moved / ms / 1e6 / sms,
                 static_cast<double>(per_prod) * nprod / (ms * 1e3));
        }
      }
    }
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
