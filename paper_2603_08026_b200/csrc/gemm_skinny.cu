// gemm_skinny.cu — weight-stationary 2-CTA (cta_group::2) tcgen05 GEMM for the small salient row
// counts of the sparse steps (M <= 512 rows, the weight-streaming
// regime of §8d.3).
//
//   D[m][n] = sum_k A[m][k] * W[n][k]     computed as D^T = W A^T:
//   MMA-M = 256 weight rows of a CTA pair (128 per CTA, its own TMEM lanes),
//   MMA-N = the activation rows (N <= 256 per instruction; two instructions cover M <= 512, each
//           CTA of the pair holding half of them, so every activation byte enters one SM per pair).
// Each weight byte is read by exactly one SM; the accumulator (128 lanes x M columns, <= 512)
// stays in TMEM for the whole K range of a segment. Work is split stream-K style: the
// (weight block, k-block) space is cut into equal contiguous ranges, one per co-resident SM pair,
// so all 148 SMs stream weights even when N/256 is small (O-proj and FFN-down: 16 blocks).
// A block whose K range spans several pairs is reduced through an fp32 workspace in a fixed
// contributor order (bit-deterministic), each contributor finishing a share of the rows. Roles per CTA (192 threads): warp 0 TMA producer (both
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
constexpr int SK_XCH = 2 * 32 * 128 * 4;     // epilogue transpose tiles: 2 x [32 rows][128 weight rows] fp32
constexpr int kSkRing = SK_STAGES * SK_STAGE / (32 * 128 * 4);  // reduction ring buffers in the stage area
constexpr int SK_SMEM = 1024 + SK_STAGES * SK_STAGE + SK_XCH + 256;
static_assert(12 * 8 + kSkRing * 8 + 4 <= 256, "barrier area");
constexpr int SKINNY_MAX_M = kSkinnyMaxM;
constexpr int kSkPrefetch = 12;   // k-blocks of weight L2 prefetch ahead of the ring
constexpr int kSkMaxContrib = 12;  // <= kSkRing: all partial tiles of one chunk fit in the ring  // split-K contributors per weight block (host-checked)

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
__device__ __forceinline__ void bulk_store(void *gdst, const void *ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_load(void *sdst, const void *gsrc, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(sdst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
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
  float *ws;   // split-K partials: [2*P slots][512 m][256 weight rows] fp32
  int *ctr;    // per (item, rank) arrival counters, zero between launches
  int P;       // pairs taking part in the stream-K partition
  unsigned long long *trace;  // optional [grid][16] globaltimer stamps (debug hook)
  int kpu;     // k-blocks per stream-K unit (K/64 / units per weight block)
};

// Stream-K partition of the (item, k-block) space: pair p owns units [start(p), start(p+1)).
__device__ __forceinline__ int64_t sk_start(int p, int64_t W, int P) { return static_cast<int64_t>(p) * W / P; }
__device__ __forceinline__ int sk_owner(int64_t u, int64_t W, int P) {
  return static_cast<int>((u * P + P - 1) / W);
}
__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void sk_stamp(const SkinnyParams &p, int slot) {
  if (p.trace) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[blockIdx.x * 16 + slot] = t;
  }
}

// One segment = (item, [kb0, kb1)) of a pair's range, in range order.
struct SkSeg {
  int item, kb0, kb1;
};
struct SkIter {
  int64_t u, end;  // unit range [u, end) of the pair
  int upi, kpu;    // units per weight block, k-blocks per unit
  __device__ bool next(SkSeg &s) {
    if (u >= end) return false;
    s.item = static_cast<int>(u / upi);
    const int u0 = static_cast<int>(u - static_cast<int64_t>(s.item) * upi);
    const int64_t left = end - u;
    const int u1 = left < upi - u0 ? u0 + static_cast<int>(left) : upi;
    s.kb0 = u0 * kpu;
    s.kb1 = u1 * kpu;
    u += u1 - u0;
    return true;
  }
};

template <int EPI>
__global__ void __launch_bounds__(192, 1)
    gemm_skinny_kernel(const __grid_constant__ CUtensorMap tmA128, const __grid_constant__ CUtensorMap tmA64,
                       const __grid_constant__ CUtensorMap tmA32, const __grid_constant__ CUtensorMap tmA16,
                       const __grid_constant__ CUtensorMap tmW, const SkinnyParams p) {
  const int M = p.M_ptr ? min(*p.M_ptr, p.M_cap) : p.M_cap;
  if (M <= 0 || M > SKINNY_MAX_M) return;  // uniform across the grid
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t *stages = smem;
  float *xs = reinterpret_cast<float *>(smem + SK_STAGES * SK_STAGE);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + SK_STAGES * SK_STAGE + SK_XCH);
  uint64_t *empty = full + SK_STAGES;
  uint64_t *tfull = empty + SK_STAGES;   // [2]
  uint64_t *tempty = tfull + 2;          // [2]
  uint64_t *rbar = tempty + 2;           // [kSkRing] split-K reduction ring
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(rbar + kSkRing);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const int items = p.N / 256;
  const int num_kb = p.K / 64;
  const int kpu = p.kpu, upi = num_kb / kpu;                 // split granularity (host-chosen)
  const int64_t Wt = static_cast<int64_t>(items) * upi;      // units of the stream-K partition
  // activation rows per MMA, rounded to 32 so that each CTA's half is a multiple of 16 rows
  const int NA0 = (min(M, 256) + 31) & ~31;
  const int NA1 = M > 256 ? ((M - 256 + 31) & ~31) : 0;
  // M <= 256: two 256-column TMEM accumulators (epilogue of segment i overlaps the MMAs of i+1)
  const int nbuf = NA1 ? 1 : 2;
  const uint32_t stage_tx = 2u * (SK_W_BYTES + (NA0 / 2 + NA1 / 2) * 128);
  SkIter iter0{sk_start(pair, Wt, p.P), sk_start(pair + 1, Wt, p.P), upi, kpu};

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA128);
    tma_prefetch_desc(&tmA64);
    tma_prefetch_desc(&tmA32);
    tma_prefetch_desc(&tmA16);
    tma_prefetch_desc(&tmW);
    for (int s = 0; s < SK_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 2 * 128);
    }
    for (int s = 0; s < kSkRing; ++s) mbar_init(&rbar[s], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) sk_stamp(p, 0);

  if (warp == 0) {
    // ===================== TMA producer (both CTAs)
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      SkIter it = iter0;
      SkSeg sg;
      // weight tiles are read once, from DRAM: an L2 prefetch stream runs kSkPrefetch k-blocks
      // ahead of the shared-memory ring so the ring's TMA loads hit L2
      int64_t pf = it.u * kpu;             // k-block space: item * num_kb + kb
      const int64_t pf_end = it.end * kpu;
      auto prefetch_to = [&](int64_t upto) {
        for (; pf < upto && pf < pf_end; ++pf) {
          const int item = static_cast<int>(pf / num_kb);
          const int kb = static_cast<int>(pf - static_cast<int64_t>(item) * num_kb);
          tma_prefetch_l2_2d(&tmW, kb * 64, item * 256 + static_cast<int>(rank) * 128);
        }
      };
      prefetch_to(it.u + kSkPrefetch);
      while (it.next(sg)) {
        const int wrow = sg.item * 256 + static_cast<int>(rank) * 128;
        for (int kb = sg.kb0; kb < sg.kb1; ++kb) {
          prefetch_to(static_cast<int64_t>(sg.item) * num_kb + kb + 1 + kSkPrefetch);
          mbar_wait(&empty[st], ph ^ 1);
          if (rank == 0) mbar_expect_tx(&full[st], stage_tx);
          uint8_t *sb = stages + st * SK_STAGE;
          tma_load_2d_pair(sb, &tmW, &full[st], kb * 64, wrow);
          // this CTA's half of each activation block, in boxes of 128/64/32/16 rows (only the
          // rows the MMA reads; 16-row offsets keep the 128B-swizzle atoms aligned)
          auto load_rows = [&](uint8_t *dst, int r0, int n) {
            const CUtensorMap *maps[4] = {&tmA128, &tmA64, &tmA32, &tmA16};
            int off = 0;
            for (int bi = 0; bi < 4; ++bi) {
              const int box = 128 >> bi;
              while (n - off >= box) {
                tma_load_2d_pair(dst + off * 128, maps[bi], &full[st], kb * 64, r0 + off);
                off += box;
              }
            }
          };
          load_rows(sb + SK_W_BYTES, static_cast<int>(rank) * (NA0 / 2), NA0 / 2);
          if (NA1) load_rows(sb + SK_W_BYTES + SK_A_BYTES, 256 + static_cast<int>(rank) * (NA1 / 2), NA1 / 2);
          if (++st == SK_STAGES) {
            st = 0;
            ph ^= 1;
          }
        }
      }
      sk_stamp(p, 1);
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA only)
    if (rank == 0) {
      const uint32_t id0 = idesc_bf16_f32(256, NA0);
      const uint32_t id1 = idesc_bf16_f32(256, NA1 ? NA1 : 16);
      int st = 0;
      uint32_t ph = 0;
      int local = 0;
      SkIter it = iter0;
      SkSeg sg;
      while (it.next(sg)) {
        const int b = nbuf == 2 ? (local & 1) : 0;
        const uint32_t tph = nbuf == 2 ? ((local >> 1) & 1) : (local & 1);
        const uint32_t acc = tmem_base + b * 256;
        mbar_wait(&tempty[b], tph ^ 1);
        tc_fence_after();
        for (int kb = sg.kb0; kb < sg.kb1; ++kb) {
          mbar_wait(&full[st], ph);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t w0 = smem_u32(stages + st * SK_STAGE);
            const uint32_t a0 = w0 + SK_W_BYTES;
            const uint32_t first = (kb == sg.kb0) ? 1u : 0u;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t accum = (first && k == 0) ? 0u : 1u;
              umma_bf16_pair(acc, sw128_kmajor_desc(w0 + k * 32), sw128_kmajor_desc(a0 + k * 32), id0, accum);
              if (NA1)
                umma_bf16_pair(acc + 256, sw128_kmajor_desc(w0 + k * 32),
                               sw128_kmajor_desc(a0 + SK_A_BYTES + k * 32), id1, accum);
            }
            umma_commit_pair(&empty[st]);
            if (kb == sg.kb1 - 1) umma_commit_pair(&tfull[b]);
          }
          __syncwarp();
          if (++st == SK_STAGES) {
            st = 0;
            ph ^= 1;
          }
        }
        ++local;
      }
      if (lane == 0) sk_stamp(p, 2);
    }
  } else {
    // ===================== epilogue warps 2..5 (both CTAs, own TMEM lanes)
    const int quad = warp & 3;
    const int row = quad * 32 + lane;  // weight row within this CTA's 128
    const int et = threadIdx.x - 64;   // 0..127
    const uint32_t leader_tempty0 = mapa_shared(smem_u32(&tempty[0]), 0);
    const uint32_t leader_tempty1 = mapa_shared(smem_u32(&tempty[1]), 0);
    // Final epilogue of 32 output rows [m0, m0+32) x this CTA's 128 weight rows, read from a
    // [32 m][128 n] fp32 tile in shared memory. Threads are laid out along the weight (= output
    // column) dimension so that the 8-byte bf16 stores (and residual loads) are coalesced.
    // Register slot i holds the float4 at (row m0 + sl_m(i), weight rows sl_n(i)..+3): SwiGLU
    // slots 0-3 gate, 4-7 up (weight rows [0,64) gate, [64,128) up of the same 64 FFN channels).
    constexpr bool kSw = EPI == EPI_SWIGLU;
    const int n4 = kSw ? (et & 15) : (et & 31);
    const int msub = kSw ? (et >> 4) : (et >> 5);
    auto sl_m = [&](int i) { return kSw ? msub + 8 * (i & 3) : msub + 4 * i; };
    auto sl_n = [&](int i) { return kSw ? (i < 4 ? 4 * n4 : 64 + 4 * n4) : 4 * n4; };
    auto store = [&](const float4 r[8], int m0, int item) {
      if constexpr (kSw) {
        const int ch = (item * 2 + static_cast<int>(rank)) * 64 + 4 * n4;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int m = m0 + sl_m(i);
          if (m < M) {
            const float4 g = r[i], u = r[4 + i];
            const float o0 = g.x / (1.f + __expf(-g.x)) * u.x, o1 = g.y / (1.f + __expf(-g.y)) * u.y;
            const float o2 = g.z / (1.f + __expf(-g.z)) * u.z, o3 = g.w / (1.f + __expf(-g.w)) * u.w;
            *reinterpret_cast<uint2 *>(p.D + static_cast<int64_t>(m) * p.ldd + ch) =
                make_uint2(pack2(o0, o1), pack2(o2, o3));
          }
        }
      } else {
        const int n = item * 256 + static_cast<int>(rank) * 128 + 4 * n4;
        float bb[4] = {0.f, 0.f, 0.f, 0.f};
        if (p.bias) {
          const uint2 bv = *reinterpret_cast<const uint2 *>(p.bias + n);
          const float2 b01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&bv.x));
          const float2 b23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&bv.y));
          bb[0] = b01.x; bb[1] = b01.y; bb[2] = b23.x; bb[3] = b23.y;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int m = m0 + sl_m(i);
          if (m < M) {
            float o[4] = {r[i].x + bb[0], r[i].y + bb[1], r[i].z + bb[2], r[i].w + bb[3]};
            if constexpr (EPI == EPI_RESID) {
              const int rr = p.resid_rows ? p.resid_rows[m] : m;
              const uint2 rv = *reinterpret_cast<const uint2 *>(p.resid + static_cast<int64_t>(rr) * p.ldr + n);
              const float2 r01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&rv.x));
              const float2 r23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&rv.y));
              o[0] += r01.x; o[1] += r01.y; o[2] += r23.x; o[3] += r23.y;
            }
            *reinterpret_cast<uint2 *>(p.D + static_cast<int64_t>(m) * p.ldd + n) =
                make_uint2(pack2(o[0], o[1]), pack2(o[2], o[3]));
          }
        }
      }
    };
    // workspace: slot-major, then rank, then [512 m][128 n] fp32, so one 32-row chunk of one
    // CTA's partial is a contiguous 16 KB block (one bulk copy each way)
    auto ws_chunk = [&](int slot, int c) -> float * {
      return p.ws + ((static_cast<int64_t>(slot) * 2 + rank) * 512 + c * 32) * 128;
    };
    // slot of (pair pp, item): side 0 if the pair's range starts inside the item (its first
    // segment), side 1 otherwise (its last segment)
    auto slot_of = [&](int pp, int item) -> int {
      return pp * 2 + (sk_start(pp, Wt, p.P) >= static_cast<int64_t>(item) * upi ? 0 : 1);
    };
    int deferred[2];
    int ndef = 0;
    int local = 0;
    int xb = 0;  // transpose tile double buffer index
    SkIter it = iter0;
    SkSeg sg;
    while (it.next(sg)) {
      const int b = nbuf == 2 ? (local & 1) : 0;
      const uint32_t tph = nbuf == 2 ? ((local >> 1) & 1) : (local & 1);
      mbar_wait(&tfull[b], tph);
      tc_fence_after();
      if (et == 0 && local < 4) sk_stamp(p, 3 + local);
      const uint32_t tb = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + b * 256;
      const bool whole = sg.kb0 == 0 && sg.kb1 == num_kb;  // the segment spans the whole K range
      const int slot = whole ? 0 : slot_of(pair, sg.item);
      const int NAt = NA0 + NA1;
      for (int c0 = 0; c0 < NAt; c0 += 32) {
        // TMEM columns: [0, NA0) hold rows 0.., [256, 256+NA1) hold rows 256..
        const int m0 = c0 < NA0 ? c0 : 256 + (c0 - NA0);
        float *x = xs + xb * (32 * 128);
        float v[32];
        tmem_ld32(tb + (c0 < NA0 ? c0 : 256 + (c0 - NA0)), v);
        if (c0 + 32 >= NAt) {  // accumulator fully read: hand TMEM back to the MMA warp
          tc_fence_before();
          mbar_arrive_cluster(b ? leader_tempty1 : leader_tempty0);
        }
        if (et == 0) bulk_wait_read<1>();  // a bulk store of 2 chunks ago has left x
        named_bar_sync(1, 128);
#pragma unroll
        for (int t = 0; t < 32; ++t) x[t * 128 + row] = v[t];
        if (whole) {
          named_bar_sync(1, 128);
          const float4 *x4 = reinterpret_cast<const float4 *>(x);
          float4 r[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) r[i] = x4[sl_m(i) * 32 + sl_n(i) / 4];
          store(r, m0, sg.item);
        } else {
          // split-K partial: publish the 16 KB tile with one bulk store
          fence_proxy_async();
          named_bar_sync(1, 128);
          if (et == 0) {
            bulk_store(ws_chunk(slot, m0 / 32), x, 32 * 128 * 4);
            bulk_commit();
          }
        }
        xb ^= 1;
      }
      if (!whole) {
        if (et == 0) {
          bulk_wait<0>();   // partial is in global memory (L2)
          fence_proxy_async_global();
          __threadfence();
          atomicAdd(p.ctr + sg.item * 2 + static_cast<int>(rank), 1);
        }
        if (ndef < 2) deferred[ndef++] = sg.item;
      }
      ++local;
    }
    if (et == 0) sk_stamp(p, 7);
    // Reductions of the split blocks (after every segment of this pair is published, so no pair
    // waits while holding unpublished work). Contributor q of nc finishes 32-row chunks
    // q, q+nc, ...: the nc partial tiles of a chunk are streamed into the idle stage ring with
    // bulk copies (kRing buffers of 16 KB) and summed in fixed contributor order
    // (bit-deterministic: the order does not depend on arrival order).
    constexpr int kRing = SK_STAGES * SK_STAGE / (32 * 128 * 4);
    float *ring = reinterpret_cast<float *>(stages);
    int rseq = 0;  // ring buffer sequence number (buffer rseq % kRing, phase (rseq / kRing) & 1)
    for (int di = 0; di < ndef; ++di) {
      const int item = deferred[di];
      const int64_t ib = static_cast<int64_t>(item) * upi;
      const int p_first = sk_owner(ib, Wt, p.P);
      const int nc = sk_owner(ib + upi - 1, Wt, p.P) - p_first + 1;
      const int q = pair - p_first;
      int *ctr = p.ctr + item * 2 + static_cast<int>(rank);
      if (et == 0) {
        while (ld_acquire(ctr) < nc) {
        }
        fence_proxy_async_global();  // generic acquire -> async-proxy (bulk copy) reads
      }
      named_bar_sync(1, 128);
      if (et == 0 && di < 2) sk_stamp(p, 8 + di);
      const int nchunks = (M + 31) / 32;
      const int my = nchunks > q ? (nchunks - q + nc - 1) / nc : 0;  // my chunks
      const int per = kRing / nc;                                      // chunks in flight
      if (per == 0) __trap();                                          // host keeps nc <= kRing
      // issue loads for chunk k of mine into ring sequence rseq + k*nc + qq
      auto issue = [&](int k) {
        const int c = q + k * nc;
        for (int qq = 0; qq < nc; ++qq) {
          const int sq = rseq + k * nc + qq;
          uint64_t *bar = &rbar[sq % kRing];
          mbar_expect_tx(bar, 32 * 128 * 4);
          bulk_load(ring + (sq % kRing) * (32 * 128), ws_chunk(slot_of(p_first + qq, item), c), 32 * 128 * 4, bar);
        }
      };
      if (et == 0) {
        fence_proxy_async();
        for (int k = 0; k < my && k < per; ++k) issue(k);
      }
      for (int k = 0; k < my; ++k) {
        float4 r[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) r[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int qq = 0; qq < nc; ++qq) {
          const int sq = rseq + k * nc + qq;
          mbar_wait(&rbar[sq % kRing], (sq / kRing) & 1);
          const float4 *t4 = reinterpret_cast<const float4 *>(ring + (sq % kRing) * (32 * 128));
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 t = t4[sl_m(i) * 32 + sl_n(i) / 4];
            r[i].x += t.x; r[i].y += t.y; r[i].z += t.z; r[i].w += t.w;
          }
        }
        named_bar_sync(1, 128);  // every thread is done with chunk k's buffers
        if (et == 0 && k + per < my) {
          fence_proxy_async();
          issue(k + per);
        }
        store(r, (q + k * nc) * 32, item);
      }
      rseq += my * nc;
      // second arrival: the last contributor to pass re-arms the counter for the next launch
      if (et == 0 && atomicAdd(ctr, 1) == 2 * nc - 1) atomicExch(ctr, 0);
    }
  }
  if (threadIdx.x == 64) sk_stamp(p, 10);
  tc_fence_before();
  cluster_sync_all();
  if (threadIdx.x == 0) sk_stamp(p, 11);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 512);
  }
}

int skinny_auto_split(int items, int num_kb, int max_pairs);

template <int EPI>
static int launch_skinny_t(const GemmCall &g, int num_sms, cudaStream_t st) {
  auto kern = gemm_skinny_kernel<EPI>;
  static bool attr_done = false;
  static int max_pairs = 0;
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = SK_SMEM;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (!attr_done) {
    DY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SK_SMEM));
    DY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
    // split-K contributors spin on each other: every pair of the grid must be co-resident
    cfg.gridDim = dim3(num_sms);
    int clusters = 0;
    DY_CUDA(cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg));
    max_pairs = clusters < num_sms / 2 ? clusters : num_sms / 2;
    if (max_pairs < 1) {
      set_error("skinny gemm: no co-resident 2-CTA cluster");
      return DYLLM_E_CUDA;
    }
    attr_done = true;
  }
  if (!g.ws || !g.ctr || g.N / 256 * 2 > kSkinnyCtrCap) {
    set_error("skinny gemm: missing split-K workspace or too many weight blocks");
    return DYLLM_E_ARG;
  }
  CUtensorMap ta[4], tw;
  for (int bi = 0; bi < 4; ++bi) {
    int rc = make_tmap(&ta[bi], g.A, g.M_cap, g.K, 128 >> bi);
    if (rc) return rc;
  }
  int rc = make_tmap(&tw, g.W, g.N, g.K, 128);
  if (rc) return rc;
  const int items = g.N / 256, num_kb = g.K / 64;
  // split granularity: units per weight block (S); each unit is num_kb / S k-blocks
  int S = g_skinny_split > 0 ? g_skinny_split : skinny_auto_split(items, num_kb, max_pairs);
  if (S > num_kb) S = num_kb;
  while (num_kb % S) --S;
  const int64_t units = static_cast<int64_t>(items) * S;
  int pairs = max_pairs;
  if (pairs > units) pairs = static_cast<int>(units);
  // every weight block must have <= kSkMaxContrib contributors (its partial tiles share the ring)
  auto max_contrib = [&](int P) {
    int mx = 0;
    for (int i = 0; i < items; ++i) {
      const int64_t a = static_cast<int64_t>(i) * S, b = a + S - 1;
      const int nc = static_cast<int>((b * P + P - 1) / units - (a * P + P - 1) / units) + 1;
      mx = nc > mx ? nc : mx;
    }
    return mx;
  };
  while (pairs > 1 && max_contrib(pairs) > kSkMaxContrib) --pairs;
  SkinnyParams p{g.M_ptr, g.M_cap, g.N, g.K, g.D, g.ldd, g.resid, g.ldr, g.resid_rows, g.bias, g.ws, g.ctr, pairs,
                 g_skinny_trace, num_kb / S};
  cfg.gridDim = dim3(2 * pairs);
  DY_CUDA(cudaLaunchKernelEx(&cfg, kern, ta[0], ta[1], ta[2], ta[3], tw, p));
  return DYLLM_OK;
}

unsigned long long *g_skinny_trace = nullptr;
int g_skinny_split = 0;

// Default split: units per weight block. One unit per pair when there are fewer weight blocks
// than SM pairs (S = pairs / blocks: O-proj and FFN-down, 16 blocks -> S = 4), otherwise no split:
// the fp32 partial round trip through L2 costs more than the imbalance it removes. Measured at
// the LLaDA-8B shapes for M in {100, 410} against S in {1, 2, 4, 8, K/64} (tools/gemm_bench.py
// --split; profiles/).
int skinny_auto_split(int items, int num_kb, int max_pairs) {
  int S = max_pairs / items;
  if (S < 1) S = 1;
  if (S > num_kb) S = num_kb;
  return S;
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
