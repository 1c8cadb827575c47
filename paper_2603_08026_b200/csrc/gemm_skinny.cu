// gemm_skinny.cu — weight-stationary 2-CTA (cta_group::2) tcgen05 GEMM for the salient row
// counts of the sparse steps and the FullStep (M <= 16384 rows; the
// weight-streaming regime of §8d.3 and the tensor-bound range).
//
//   D[m][n] = sum_k A[m][k] * W[n][k]     computed as D^T = W A^T:
//   MMA-M = 256 weight rows of a CTA pair (128 per CTA, its own TMEM lanes),
//   MMA-N = activation rows (N <= 256 per instruction; each CTA of the pair holds half of them,
//           so every activation byte enters one SM per pair).
// A tile is (256-row weight block, activation chunk): M <= 512 -> one chunk of all rows (two
// instructions per k-step above 256 rows, accumulator of M <= 512 TMEM columns); M > 512 ->
// ceil(M/256) equal chunks of <= 256 rows with a double-buffered accumulator. Per SM and k-block
// the pair moves 16 KB of weights + R/2 x 128 B of activations for 128 x R x 64 MACs, which is
// 1.5-2x the arithmetic per byte of a 128 x 256 single-CTA tile: what bounds these GEMMs on
// B200 is the L2 -> SM operand traffic (tools/tma_probe.cu, profiles/r1c_gemm_split_sweep.txt).
// Work is split stream-K style: the (tile, k-block) space is cut into equal contiguous ranges,
// one per co-resident SM pair, so all 148 SMs stream weights even when tiles are few (O-proj and
// FFN-down at M <= 512: 16 tiles).
// A block whose K range spans several pairs is reduced through an fp32 workspace in a fixed
// contributor order (bit-deterministic), each contributor finishing a share of the rows; the
// partials are written and read straight from registers in TMEM-native layout (one 128-byte line
// per thread and 32-row chunk). Roles per CTA (352 threads): warps 0 (weights) and 10
// (activations) TMA producers (both CTAs load their halves; the leader's full barrier counts the
// bytes of both), warp 1 TMEM allocator +
// (leader only) single-thread tcgen05.mma issuer with multicast commits, warps 2-9 epilogue from
// the CTA's own TMEM lanes in two halves of four warps taking alternate 32-column chunks (bias /
// residual / SiLU-gate), transposed through shared memory for coalesced stores.
// The kernel exits immediately when the device-side row count is 0 or > 16384 (the standard
// kernel of gemm.cu covers that regime), so both kernels can be enqueued without a host sync.
#include <cudaTypedefs.h>

#include "common.cuh"
#include "internal.h"

namespace dy {

// A k-block is 128 columns: every operand box is one 3-D TMA op {64 columns, rows, 2 chunks}
// (32 KB for 128 rows), laid out [chunk][rows][64] in shared memory — twice the bytes per TMA
// op of 2-D 64-column boxes, which is what the per-SM L2 -> SM ingest rate depends on
// (tools/tma_probe.cu: 16 KB ops ~44-53 GB/s/SM, 32 KB ops ~71-82 GB/s/SM from L2).
constexpr int SK_KB = 128;                   // k-block width (elements)

constexpr int SK_STAGES = 2;
constexpr int SK_W_BYTES = 128 * 256;        // 128 weight rows x 128 bf16
constexpr int SK_A_BYTES = 128 * 256;        // <= 128 activation rows x 128 bf16 (per MMA half)
constexpr int SK_STAGE = SK_W_BYTES + 2 * SK_A_BYTES;
constexpr int SK_XCH = 2 * 32 * 128 * 4;     // epilogue transpose tiles: one [32 rows][128 weight rows] fp32 per half
constexpr int SK_RING = SK_STAGES * SK_STAGE;  // 192 KB: 2 stages of 96 KB (M in (256, 512]) or 3 of 64 KB
constexpr int SK_MAX_STAGES = 8;           // ring stages sized to the launch's activation rows (below)
constexpr int SK_SMEM = 1024 + SK_RING + SK_XCH + 256;
constexpr int SK_THREADS = 352;              // W producer, MMA, 8 epilogue warps, A producer
constexpr int SKINNY_MAX_M = kSkinnyMaxM;
constexpr int kSkPrefetch = 12;   // k-blocks of weight L2 prefetch ahead of the ring
#ifndef DYLLM_QKV_ROWS
#define DYLLM_QKV_ROWS 1
#endif
constexpr int kQkvRows = DYLLM_QKV_ROWS;  // EPI_QKV: rows whose loads are issued together

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
  __syncwarp();  // bar.sync is .aligned: the warp must be converged
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
  const int *out_rows;  // nullable: destination row of each output row (fused scatter-back, a8)
  float *ws;   // split-K partials: [2*P slots][512 m][256 weight rows] fp32
  int *ctr;    // per (item, rank) arrival counters, zero between launches
  int P_max;   // co-resident pairs of the grid (the partition uses P <= P_max of them)
  unsigned long long *trace;  // optional [grid][16] globaltimer stamps (debug hook)
  int S_force; // test hook: split units per tile (0 = automatic)
  int one_chunk_max;  // largest M kept in ONE activation chunk (two MMAs per k-step above 256
                      // rows, single-buffered accumulator); above: chunks of <= 256 rows
  int chunk_rows;     // test hook: largest rows per activation chunk when chunked (0: 256)
  int krot;           // k-block start offset per weight block (x block index, mod the segment's k-blocks)
  int dbg;            // measurement hook: bit 0 skips the operand TMA loads, bit 1 the MMAs, bit 2 the
                      // epilogue's global stores, bit 3 its shared-memory transpose
  QkvEpi qkv;         // EPI_QKV (a2 + a3 fused)
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
  int64_t u, end;  // unit range [u, end) of the pair (strided: tile u, u + step, ... < end)
  int upi, kpu;    // units per tile, k-blocks per unit
  int64_t step;    // 0: contiguous stream-K range; > 0: whole tiles u, u + step, ...
  __device__ bool next(SkSeg &s) {
    if (u >= end) return false;
    if (step) {
      s.item = static_cast<int>(u);
      s.kb0 = 0;
      s.kb1 = upi * kpu;
      u += step;
      return true;
    }
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

// k-block order of a segment: starts at an offset that depends on the weight block, so that pairs
// running at the same time read different k-blocks of the shared activation rows
__device__ __forceinline__ int sk_rot(const SkSeg &s, int nchunk, int krot) {
  const int n = s.kb1 - s.kb0;
  return n > 0 ? (s.item / nchunk) * krot % n : 0;
}
__device__ __forceinline__ int sk_kb(const SkSeg &s, int j, int rot) {
  const int n = s.kb1 - s.kb0;
  const int q = j + rot;
  return s.kb0 + (q >= n ? q - n : q);
}

// tensor maps: weights (box 128 rows) and activations (box 16 * (i + 1) rows, i = 0..7: one op
// loads exactly a CTA's half of the activation rows of an MMA, whatever the device-side M)
struct SkMaps {
  CUtensorMap w;
  CUtensorMap a[8];
};

__device__ __forceinline__ void tma_load_3d_pair(void *smem_dst, const void *tmap, uint64_t *bar, int c0, int c1,
                                                 int c2) {
  const uint32_t leader_bar = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(leader_bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_l2_3d(const void *tmap, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}

// CH = 64-column chunks per k-block: 2 (128-wide k-blocks, one 32 KB weight op per stage) or 1
// (64-wide k-blocks: half-size stages, twice as many in the same ring)
template <int EPI, int CH>
__global__ void __launch_bounds__(SK_THREADS, 1)
    gemm_skinny_kernel(const __grid_constant__ SkMaps maps, const SkinnyParams p) {
  constexpr int kWBytes = 128 * 128 * CH;  // 128 weight rows x CH chunks of 64 bf16
  constexpr int kRowBytes = 128 * CH;      // one activation row of a stage
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t *stages = smem;
  float *xs = reinterpret_cast<float *>(smem + SK_STAGES * SK_STAGE);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + SK_STAGES * SK_STAGE + SK_XCH);
  uint64_t *empty = full + SK_MAX_STAGES;
  uint64_t *tfull = empty + SK_MAX_STAGES;   // [2]
  uint64_t *tempty = tfull + 2;          // [2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  // setup (independent of the device row count) overlaps the previous kernel of the stream
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&maps.w);
    for (int s = 0; s < SK_MAX_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 2 * 8);  // one arrival per epilogue warp of both CTAs
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();
  pdl_trigger();  // the grid is co-resident (occupancy-sized): the next kernel may launch
  const int M = p.M_ptr ? min(*p.M_ptr, p.M_cap) : p.M_cap;
  if (M <= 0 || M > SKINNY_MAX_M) {  // uniform across the grid: nothing to do
    tc_fence_before();
    cluster_sync_all();
    if (warp == 1) {
      tc_fence_after();
      tmem_dealloc_pair(tmem_base, 512);
    }
    return;
  }
  // Tiles ("items") = (256-row weight block, activation chunk). M <= 512: one chunk holding all
  // rows (two MMAs per k-step when M > 256, single-buffered accumulator); M > 512: ceil(M/256)
  // equal chunks of R <= 256 rows (double-buffered accumulator). Chunks of one weight block are
  // adjacent in tile order, so the pairs working on them at the same time share it through L2.
  // M in (256, 512]: one chunk (two MMAs per k-step, single-buffered accumulator, 2-stage ring)
  // only when that fills the pairs in one round and two chunks would need two rounds
  // (P/2 <= weight blocks < P: the QKV projection); otherwise chunks of <= 256 rows pipeline
  // better (double-buffered accumulator, 3-stage ring). Measured: tools/gemm_bench.py --one-chunk.
  const int nwb = p.N / 256;
  const bool one = p.one_chunk_max >= 0 ? M <= p.one_chunk_max
                                        : (M <= 256 || (M <= 512 && 2 * nwb >= p.P_max && nwb < p.P_max));
  // M > 512 with few weight blocks (O-proj / FFN-down: 16): floor(P / blocks) chunks of up to 512
  // rows, so every tile runs in ONE round over the pairs (256-row chunks would need two rounds:
  // 96 tiles for 74 pairs at M = 1530); else chunks of <= 256 rows (tools/gemm_bench.py --chunk,
  // profiles/r2/skinny/chunk512.txt)
  const int n1 = p.P_max / nwb;
  const bool oneround = p.chunk_rows == 0 && !one && n1 >= 2 && M <= 512 * n1 && M > 512;
  const int crow = oneround ? (M + n1 - 1) / n1 : p.chunk_rows > 0 ? min(p.chunk_rows, 512) : 256;
  const int nchunk = one ? 1 : (M + crow - 1) / crow;
  const int R = nchunk == 1 ? M : (((M + nchunk - 1) / nchunk + 31) & ~31);
  const int items = p.N / 256 * nchunk;
  const int num_kb = p.K / (64 * CH);
  // split granularity (stream-K units per tile), from the device-side M: tiles are cut into
  // S units when there are fewer tiles than pairs (S = pairs / tiles), so all pairs stream
  int upi = p.S_force > 0 ? p.S_force : max(1, p.P_max / items);
  upi = min(upi, num_kb);
  while (num_kb % upi) --upi;
  const int kpu = num_kb / upi;
  const int64_t Wt = static_cast<int64_t>(items) * upi;      // units of the stream-K partition
  const int P = static_cast<int>(min(static_cast<int64_t>(p.P_max), Wt));
  // activation rows per MMA, rounded to 32 so that each CTA's half is a multiple of 16 rows
  // (a chunk of more than 256 rows runs as two MMAs per k-step: rows [0, 256) and [256, R))
  const int NA0 = (min(R, 256) + 31) & ~31;
  const int NA1 = R > 256 ? ((R - 256 + 31) & ~31) : 0;
  // M <= 256: two 256-column TMEM accumulators (epilogue of segment i overlaps the MMAs of i+1)
  const int nbuf = NA1 ? 1 : 2;
  const uint32_t stage_tx = 2u * (kWBytes + (NA0 / 2 + NA1 / 2) * kRowBytes);
  // ring: a stage holds 32 KB of weights + one (or, for M in (256, 512], two) 32 KB activation
  // slots; with one slot the same 192 KB hold 3 stages instead of 2
  // a stage holds the weight box and exactly this launch's activation boxes (the second MMA's rows
  // right after the first's), so fewer activation rows buy a deeper ring: the L2 -> SM latency of
  // the 32 KB boxes is what a 3-stage ring exposes (the k-block time barely depends on the rows)
  const int stage_bytes = (kWBytes + (NA0 / 2) * kRowBytes + (NA1 / 2) * kRowBytes + 1023) & ~1023;
  const int nstages = min(SK_RING / stage_bytes, SK_MAX_STAGES);
  // Unsplit tiles (upi == 1) are dealt round-robin (pair p: tiles p, p + P, ...), so the pairs
  // running at the same time hold consecutive tiles (the activation chunks of one weight block:
  // its HBM read is shared through L2); split tiles use contiguous stream-K ranges.
  SkIter iter0 = upi == 1 ? SkIter{pair < P ? pair : 0, pair < P ? Wt : 0, upi, kpu, P}
                          : SkIter{pair < P ? sk_start(pair, Wt, P) : 0, pair < P ? sk_start(pair + 1, Wt, P) : 0,
                                   upi, kpu, 0};

  if (warp == 10 && lane == 0) {
    tma_prefetch_desc(&maps.a[NA0 / 32 - 1]);
    if (NA1) tma_prefetch_desc(&maps.a[NA1 / 32 - 1]);
  }
  if (threadIdx.x == 0) sk_stamp(p, 0);

  if (warp == 0 || warp == 10) {
    // ===================== TMA producers (both CTAs): warp 0 streams the weight tiles (and the
    // L2 prefetch stream), warp 10 the activation boxes — two issuing threads, since one thread's
    // TMA issue rate (a few small ops per microsecond, tools/tma_probe.cu) would otherwise pace
    // the ring
    const bool wprod = warp == 0;
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      SkIter it = iter0;
      SkSeg sg;
      // weight tiles are read once, from DRAM: an L2 prefetch cursor runs kSkPrefetch k-blocks
      // ahead of the shared-memory ring over the same segment sequence, so the ring's TMA loads
      // hit L2 (only the first activation chunk's pair prefetches a weight block)
      SkIter pit = it;
      SkSeg ps{0, 0, 0};
      int pkb = 0, prot = 0;
      int64_t n_pf = 0, n_ld = 0;
      auto prefetch_ahead = [&]() {
        while (n_pf < n_ld + kSkPrefetch) {
          if (pkb >= ps.kb1) {
            if (!pit.next(ps)) return;
            pkb = ps.kb0;
            prot = sk_rot(ps, nchunk, p.krot);
          }
          if (ps.item % nchunk == 0)
            tma_prefetch_l2_3d(&maps.w, 0, ps.item / nchunk * 256 + static_cast<int>(rank) * 128,
                               sk_kb(ps, pkb - ps.kb0, prot) * CH);
          ++pkb;
          ++n_pf;
        }
      };
      if (wprod) prefetch_ahead();
      while (it.next(sg)) {
        const int wrow = sg.item / nchunk * 256 + static_cast<int>(rank) * 128;
        const int arow = sg.item % nchunk * R;  // first activation row of the tile
        const int rot = sk_rot(sg, nchunk, p.krot);
        for (int j = 0; j < sg.kb1 - sg.kb0; ++j) {
          const int kb = sk_kb(sg, j, rot);
          mbar_wait(&empty[st], ph ^ 1);
          uint8_t *sb = stages + st * stage_bytes;
          if (p.dbg & 1) {
            if (wprod && rank == 0) mbar_arrive(&full[st]);
          } else if (wprod) {
            if (rank == 0) mbar_expect_tx(&full[st], stage_tx);
            tma_load_3d_pair(sb, &maps.w, &full[st], 0, wrow, kb * CH);
            ++n_ld;
            prefetch_ahead();
          } else {
            // this CTA's half of the activation rows of each MMA: one op of exactly that many rows
            tma_load_3d_pair(sb + kWBytes, &maps.a[NA0 / 32 - 1], &full[st], 0,
                             arow + static_cast<int>(rank) * (NA0 / 2), kb * CH);
            if (NA1)
              tma_load_3d_pair(sb + kWBytes + (NA0 / 2) * kRowBytes, &maps.a[NA1 / 32 - 1], &full[st], 0,
                               arow + NA0 + static_cast<int>(rank) * (NA1 / 2), kb * CH);
          }
          if (++st == nstages) {
            st = 0;
            ph ^= 1;
          }
        }
      }
      if (wprod) sk_stamp(p, 1);
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
        const int nkb = sg.kb1 - sg.kb0;
        for (int j = 0; j < nkb; ++j) {
          mbar_wait(&full[st], ph);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t w0 = smem_u32(stages + st * stage_bytes);
            const uint32_t a0 = w0 + kWBytes;
            const uint32_t first = (j == 0) ? 1u : 0u;
            // k-step kk: 64-column chunk kk / 4 (chunk stride = box rows x 128 B), +32 B per 16
#pragma unroll
            for (int kk = 0; kk < ((p.dbg & 2) ? 0 : 4 * CH); ++kk) {
              const uint32_t accum = (first && kk == 0) ? 0u : 1u;
              const uint32_t ko = (kk & 3) * 32, ch = kk >> 2;
              umma_bf16_pair(acc, sw128_kmajor_desc(w0 + ch * (128 * 128) + ko),
                             sw128_kmajor_desc(a0 + ch * (NA0 / 2 * 128) + ko), id0, accum);
              if (NA1)
                umma_bf16_pair(acc + 256, sw128_kmajor_desc(w0 + ch * (128 * 128) + ko),
                               sw128_kmajor_desc(a0 + (NA0 / 2) * kRowBytes + ch * (NA1 / 2 * 128) + ko), id1, accum);
            }
            umma_commit_pair(&empty[st]);
            if (j == nkb - 1) umma_commit_pair(&tfull[b]);
          }
          __syncwarp();
          if (++st == nstages) {
            st = 0;
            ph ^= 1;
          }
        }
        ++local;
      }
      if (lane == 0) sk_stamp(p, 2);
    }
  } else {
    // ===================== epilogue warps 2..9 (both CTAs, own TMEM lanes): two halves of four
    // warps (one per TMEM lane quadrant) take alternate 32-column chunks, so two chunks are in
    // flight per CTA; each warp prefetches its next chunk's TMEM load before storing the current.
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = quad * 32 + lane;        // weight row within this CTA's 128 (= TMEM lane)
    const int et = threadIdx.x - 64;         // 0..255
    const int t = et & 127;                  // thread within the half
    float *x = xs + half * (32 * 128);       // this half's transpose tile [32 m][128 n] fp32
    const uint32_t leader_tempty0 = mapa_shared(smem_u32(&tempty[0]), 0);
    const uint32_t leader_tempty1 = mapa_shared(smem_u32(&tempty[1]), 0);
    // Final epilogue of 32 output rows [m0, m0+32) x this CTA's 128 weight rows, from a
    // [32 m][128 n] fp32 tile in shared memory. Threads are laid out along the weight (= output
    // column) dimension so that the 8-byte bf16 stores (and residual loads) are coalesced.
    // Register slot i holds the float4 at (row m0 + sl_m(i), weight rows sl_n(i)..+3): SwiGLU
    // slots 0-3 gate, 4-7 up (weight rows [0,64) gate, [64,128) up of the same 64 FFN channels).
    constexpr bool kSw = EPI == EPI_SWIGLU;
    // SwiGLU: 16 threads per row x 4 channels (8-byte stores of 4 outputs, gate and up slots);
    // otherwise 16 threads per row x 8 output columns (16-byte stores: a warp writes two rows'
    // 256-byte segments per instruction)
    const int n4 = t & 15;
    const int msub = t >> 4;
    auto sl_m = [&](int i) { return kSw ? msub + 8 * (i & 3) : msub + 8 * (i >> 1); };
    auto sl_n = [&](int i) { return kSw ? (i < 4 ? 4 * n4 : 64 + 4 * n4) : 8 * n4 + 4 * (i & 1); };
    // the output / residual row ids of the four rows a thread stores of a chunk, loaded before the
    // chunk's transpose so that their latency overlaps it (and before any store: D may alias nothing
    // they read, but the compiler cannot know that, and a load written after a store waits for it)
    auto row_ids = [&](int m0, int tile, int orow[4], int rrow[4]) {
      m0 += tile % nchunk * R;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int m = m0 + sl_m(kSw ? i : 2 * i);
        const bool ok = m < M;
        orow[i] = ok && p.out_rows ? __ldg(p.out_rows + m) : m;
        rrow[i] = ok && p.resid_rows ? __ldg(p.resid_rows + m) : m;
      }
    };
    auto store = [&](const float4 r[8], int m0, int tile, const int orow[4], const int rrow[4]) {
      const int item = tile / nchunk;  // weight block (output columns)
      m0 += tile % nchunk * R;         // output rows of the tile's activation chunk
      if constexpr (kSw) {
        const int ch = (item * 2 + static_cast<int>(rank)) * 64 + 4 * n4;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int m = m0 + sl_m(i);
          if (m < M) {
            const float4 g = r[i], u = r[4 + i];
            const float o0 = g.x / (1.f + __expf(-g.x)) * u.x, o1 = g.y / (1.f + __expf(-g.y)) * u.y;
            const float o2 = g.z / (1.f + __expf(-g.z)) * u.z, o3 = g.w / (1.f + __expf(-g.w)) * u.w;
            *reinterpret_cast<uint2 *>(p.D + static_cast<int64_t>(orow[i]) * p.ldd + ch) =
                make_uint2(pack2(o0, o1), pack2(o2, o3));
          }
        }
      } else {
        const int n = item * 256 + static_cast<int>(rank) * 128 + 8 * n4;
        float bb[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (p.bias) {
          const uint4 bv = *reinterpret_cast<const uint4 *>(p.bias + n);
          const uint32_t bw[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&bw[q]));
            bb[2 * q] = f.x;
            bb[2 * q + 1] = f.y;
          }
        }
        // the four residual rows are loaded before the first store (one round trip per chunk)
        uint4 rv[4];
        if constexpr (EPI == EPI_RESID) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            rv[i] = m0 + sl_m(2 * i) < M
                        ? *reinterpret_cast<const uint4 *>(p.resid + static_cast<int64_t>(rrow[i]) * p.ldr + n)
                        : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int m = m0 + sl_m(2 * i);
          if (m < M) {
            const float4 a = r[2 * i], b = r[2 * i + 1];
            float o[8] = {a.x + bb[0], a.y + bb[1], a.z + bb[2], a.w + bb[3],
                          b.x + bb[4], b.y + bb[5], b.z + bb[6], b.w + bb[7]};
            if constexpr (EPI == EPI_RESID) {
              const uint32_t rw[4] = {rv[i].x, rv[i].y, rv[i].z, rv[i].w};
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&rw[q]));
                o[2 * q] += f.x;
                o[2 * q + 1] += f.y;
              }
            }
            *reinterpret_cast<uint4 *>(p.D + static_cast<int64_t>(orow[i]) * p.ldd + n) =
                make_uint4(pack2(o[0], o[1]), pack2(o[2], o[3]), pack2(o[4], o[5]), pack2(o[6], o[7]));
          }
        }
      }
    };
    // EPI_QKV (SURVEY §8 a2 + a3; the a3 kernel qkv_post in kernels.cu does the same from a bf16
    // QKV row): this CTA's 128 weight rows are one head — query head, key head or value head. The
    // thread's 4 rows x 8 head dims of the chunk come from the transposed tile with the bias added;
    // query and key heads are rotated at the row's global position (rotate-half, D10: dims d and
    // d + 64 pair, the partner dims read from the same tile); key rows keep the key they overwrite
    // (Kxo, and Kfi on the row's first write in its statistics epoch); value rows leave
    // dV = V_new - V_cache (read before the overwrite). Loads of two rows, then their stores.
    auto store_qkv = [&](const float4 *x4, int m0, int tile, const int orow[4]) {
      const QkvEpi &q = p.qkv;
      const int item = tile / nchunk;
      m0 += tile % nchunk * R;
      const int hid = item * 2 + static_cast<int>(rank);
      const int kind = hid < q.H ? 0 : hid < q.H + q.KVH ? 1 : 2;  // query / key / value head
      const int hk = kind == 0 ? hid : kind == 1 ? hid - q.H : hid - q.H - q.KVH;
      const int n = 8 * n4, pn = n ^ 64, k0 = n & 63;
      const int wid = (kind == 0 ? q.H : q.KVH) * 128;
      bf16 *__restrict__ cache = kind == 0 ? q.Qc : kind == 1 ? q.Kc : q.Vc;
      bf16 *__restrict__ compact = kind == 0 ? q.Qx : kind == 1 ? q.Kx : nullptr;
      const bool keep_old = kind == 1 && (q.Kxo || q.Kfi);
      float bb[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, bp[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if (p.bias) {
        const int gc = item * 256 + static_cast<int>(rank) * 128;
        unpack8(*reinterpret_cast<const uint4 *>(p.bias + gc + n), bb);
        if (kind < 2) unpack8(*reinterpret_cast<const uint4 *>(p.bias + gc + pn), bp);
      }
#pragma unroll
      for (int kp = 0; kp < 4; kp += kQkvRows) {
        float4 cs[kQkvRows][4];
        uint4 old[kQkvRows];
        bool snap[kQkvRows];
#pragma unroll
        for (int u = 0; u < kQkvRows; ++u) {
          const int k = kp + u;
          const int m = m0 + msub + 8 * k;
          snap[u] = false;
          old[u] = make_uint4(0u, 0u, 0u, 0u);
          if (m < M) {
            const int64_t rid = orow[k];
            if (kind < 2) {
              const float4 *c4 = reinterpret_cast<const float4 *>(q.rope_cs + (rid % q.N) * 64 + k0);
#pragma unroll
              for (int j = 0; j < 4; ++j) cs[u][j] = __ldg(c4 + j);
            }
            if (kind != 0 && (kind == 2 ? q.dV != nullptr : keep_old))
              old[u] = *reinterpret_cast<const uint4 *>(cache + rid * wid + hk * 128 + n);
            if (kind == 1 && q.Kfi) snap[u] = q.snap[m] != 0;
          }
        }
#pragma unroll
        for (int u = 0; u < kQkvRows; ++u) {
          const int k = kp + u;
          const int m = m0 + msub + 8 * k;
          if (m >= M) continue;
          const int64_t rid = orow[k];
          const int xr = (msub + 8 * k) * 32;  // the row within the chunk's transposed tile
          const float4 a = x4[xr + n / 4], b = x4[xr + n / 4 + 1];
          float v[8] = {a.x + bb[0], a.y + bb[1], a.z + bb[2], a.w + bb[3], b.x + bb[4], b.y + bb[5], b.z + bb[6],
                        b.w + bb[7]};
          bf16 *dst = cache + rid * wid + hk * 128 + n;
          if (kind < 2) {
            const float4 pa = x4[xr + pn / 4], pb = x4[xr + pn / 4 + 1];
            const float w[8] = {pa.x + bp[0], pa.y + bp[1], pa.z + bp[2], pa.w + bp[3],
                                pb.x + bp[4], pb.y + bp[5], pb.z + bp[6], pb.w + bp[7]};
            const float *cf = reinterpret_cast<const float *>(cs[u]);
            float y[8];
            // dims d < 64: x_d cos - x_(d+64) sin; dims d >= 64: x_d cos + x_(d-64) sin
#pragma unroll
            for (int j = 0; j < 8; ++j) y[j] = n < 64 ? v[j] * cf[2 * j] - w[j] * cf[2 * j + 1]
                                                      : v[j] * cf[2 * j] + w[j] * cf[2 * j + 1];
            const uint4 yb = pack8(y);
            if (kind == 1) {
              if (q.Kxo) *reinterpret_cast<uint4 *>(q.Kxo + static_cast<int64_t>(m) * wid + hk * 128 + n) = old[u];
              if (snap[u]) *reinterpret_cast<uint4 *>(q.Kfi + rid * wid + hk * 128 + n) = old[u];
            }
            *reinterpret_cast<uint4 *>(dst) = yb;
            if (compact) *reinterpret_cast<uint4 *>(compact + static_cast<int64_t>(m) * wid + hk * 128 + n) = yb;
          } else {
            const uint4 vb = pack8(v);
            if (q.dV) {
              float vn[8], vo[8], dd[8];
              unpack8(vb, vn);
              unpack8(old[u], vo);
#pragma unroll
              for (int j = 0; j < 8; ++j) dd[j] = vn[j] - vo[j];
              *reinterpret_cast<uint4 *>(q.dV + static_cast<int64_t>(m) * wid + hk * 128 + n) = pack8(dd);
            }
            *reinterpret_cast<uint4 *>(dst) = vb;
          }
        }
      }
    };
    // transpose one chunk (thread = weight row `row`, v = its 32 output rows m0..m0+31) through
    // this half's tile and store it. The leading barrier also orders the previous chunk's tile
    // reads before this chunk's writes.
    auto transpose_store = [&](const float v[32], int m0, int item) {
      int orow[4], rrow[4];
      row_ids(m0, item, orow, rrow);
      if (p.dbg & 8) {
        float4 r[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) r[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        if (!(p.dbg & 4) && EPI != EPI_QKV) store(r, m0, item, orow, rrow);
        return;
      }
      named_bar_sync(1 + half, 128);
#pragma unroll
      for (int j = 0; j < 32; ++j) x[j * 128 + row] = v[j];
      named_bar_sync(1 + half, 128);
      const float4 *x4 = reinterpret_cast<const float4 *>(x);
      if constexpr (EPI == EPI_QKV) {
        if (!(p.dbg & 4)) store_qkv(x4, m0, item, orow);
        return;
      }
      float4 r[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) r[i] = x4[sl_m(i) * 32 + sl_n(i) / 4];
      if (!(p.dbg & 4)) store(r, m0, item, orow, rrow);
    };
    // split-K partials, TMEM-native layout: slot-major, then rank, then [16 chunks][8][128 n]
    // float4 (element j of a thread's 32 values at [j / 4][n]), so every warp store / load of one
    // float4 per thread is a contiguous 512-byte line
    auto ws_line = [&](int slot, int c) -> float4 * {
      return reinterpret_cast<float4 *>(p.ws) + (((static_cast<int64_t>(slot) * 2 + rank) * 16 + c) * 8) * 128 + row;
    };
    // slot of (pair pp, item): side 0 if the pair's range starts inside the item (its first
    // segment), side 1 otherwise (its last segment)
    auto slot_of = [&](int pp, int item) -> int {
      return pp * 2 + (sk_start(pp, Wt, P) >= static_cast<int64_t>(item) * upi ? 0 : 1);
    };
    int deferred[2];
    int ndef = 0;
    int local = 0;
    SkIter it = iter0;
    SkSeg sg;
    const int NAt = NA0 + NA1;
    const int nch = NAt / 32;
    auto tcol = [&](int c) { return c * 32 < NA0 ? c * 32 : 256 + (c * 32 - NA0); };  // TMEM column = output row
    while (it.next(sg)) {
      const int b = nbuf == 2 ? (local & 1) : 0;
      const uint32_t tph = nbuf == 2 ? ((local >> 1) & 1) : (local & 1);
      mbar_wait(&tfull[b], tph);
      tc_fence_after();
      if (et == 0 && local < 4) sk_stamp(p, 3 + local);
      const uint32_t tb = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + b * 256;
      const bool whole = sg.kb0 == 0 && sg.kb1 == num_kb;  // the segment spans the whole K range
      const int slot = whole ? 0 : slot_of(pair, sg.item);
      uint32_t ra[32], rb[32];  // current chunk / next chunk (its TMEM load in flight meanwhile)
      if (half < nch) {
        tmem_ld32_issue(tb + tcol(half), ra);
        tmem_ld32_wait(ra);
      }
      for (int c = half; c < nch; c += 2) {
        const bool more = c + 2 < nch;
        if (more) tmem_ld32_issue(tb + tcol(c + 2), rb);
        if (!more) {  // this warp's last read of the accumulator: hand TMEM back to the MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(b ? leader_tempty1 : leader_tempty0);
        }
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(ra[j]);
        if (whole) {
          transpose_store(v, tcol(c), sg.item);
        } else {
          float4 *dst = ws_line(slot, c);
#pragma unroll
          for (int j = 0; j < 8; ++j) dst[j * 128] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        }
        if (more) {
          tmem_ld32_wait(rb);
#pragma unroll
          for (int j = 0; j < 32; ++j) ra[j] = rb[j];
        }
      }
      if (half >= nch) {  // (nch == 1) the idle half still releases its share of the accumulator
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(b ? leader_tempty1 : leader_tempty0);
      }
      if (!whole) {
        __threadfence();
        named_bar_sync(3, 256);
        if (et == 0) atomicAdd(p.ctr + sg.item * 2 + static_cast<int>(rank), 1);
        if (ndef < 2) deferred[ndef++] = sg.item;
      }
      ++local;
    }
    if (et == 0) sk_stamp(p, 7);
    // Reductions of the split blocks (after every segment of this pair is published, so no pair
    // waits while holding unpublished work). Contributor q of nc finishes chunks q, q+nc, ...
    // (alternating between the two halves); each thread sums its 128-byte partial lines of the
    // nc contributors in fixed contributor order (bit-deterministic: the order does not depend on
    // arrival order), then transposes and stores like an unsplit tile.
    for (int di = 0; di < ndef; ++di) {
      const int item = deferred[di];
      const int64_t ib = static_cast<int64_t>(item) * upi;
      const int p_first = sk_owner(ib, Wt, P);
      const int nc = sk_owner(ib + upi - 1, Wt, P) - p_first + 1;
      const int q = pair - p_first;
      int *ctr = p.ctr + item * 2 + static_cast<int>(rank);
      if (et == 0) {
        while (ld_acquire(ctr) < nc) {
        }
      }
      named_bar_sync(3, 256);
      if (et == 0 && di < 2) sk_stamp(p, 8 + di);
      const int my = nch > q ? (nch - q + nc - 1) / nc : 0;  // chunks this pair finishes
      for (int k = half; k < my; k += 2) {
        const int c = q + k * nc;
        float4 acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        // contributors in ascending order, loads of two of them in flight together
        for (int q0 = 0; q0 < nc; q0 += 2) {
          const int nq = nc - q0 < 2 ? nc - q0 : 2;
          float4 tv[2][8];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            if (u < nq) {
              const float4 *src = ws_line(slot_of(p_first + q0 + u, item), c);
#pragma unroll
              for (int j = 0; j < 8; ++j) tv[u][j] = __ldcg(src + j * 128);
            }
          }
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            if (u < nq) {
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                acc[j].x += tv[u][j].x; acc[j].y += tv[u][j].y; acc[j].z += tv[u][j].z; acc[j].w += tv[u][j].w;
              }
            }
          }
        }
        float vr[32];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          vr[4 * j] = acc[j].x; vr[4 * j + 1] = acc[j].y; vr[4 * j + 2] = acc[j].z; vr[4 * j + 3] = acc[j].w;
        }
        transpose_store(vr, tcol(c), item);
      }
      // second arrival: the last contributor to pass re-arms the counter for the next launch
      named_bar_sync(3, 256);
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

template <int EPI, int CH>
static int launch_skinny_t(const GemmCall &g, int num_sms, cudaStream_t st) {
  auto kern = gemm_skinny_kernel<EPI, CH>;
  static DeviceOnce attr_done;
  static int max_pairs_dev[DeviceOnce::kMaxDev] = {};
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(SK_THREADS);
  cfg.dynamicSmemBytes = SK_SMEM;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int dev = DeviceOnce::device();
  int &max_pairs = max_pairs_dev[dev];
  if (attr_done.todo()) {
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
    attr_done.done();
  }
  // split-K counters are used only when tiles < pairs (2 per tile): at most 2 * max_pairs
  if (!g.ws || !g.ctr || 2 * max_pairs > kSkinnyCtrCap) {
    set_error("skinny gemm: missing split-K workspace or counters");
    return DYLLM_E_ARG;
  }
  SkMaps maps;
  for (int i = 0; i < 8; ++i) {
    // boxes taller than the (16-rounded) capacity are never selected: clamp them to stay encodable
    const int cap16 = (g.M_cap + 15) / 16 * 16;
    const int box = 16 * (i + 1) < cap16 ? 16 * (i + 1) : cap16;
    int rc = make_tmap3(&maps.a[i], g.A, g.M_cap, g.K, box, CH);
    if (rc) return rc;
  }
  int rc = make_tmap3(&maps.w, g.W, g.N, g.K, 128, CH);
  if (rc) return rc;
  // the tile count (hence the split and the number of pairs used) depends on the device-side row
  // count: the kernel derives them; the grid is every co-resident pair
  SkinnyParams p{g.M_ptr, g.M_cap, g.N, g.K, g.D, g.ldd, g.resid, g.ldr, g.resid_rows, g.bias, g.out_rows, g.ws, g.ctr,
                 max_pairs,
                 g_skinny_trace, g_skinny_split, g_skinny_one_chunk > 0 ? g_skinny_one_chunk : -1, g_skinny_chunk_rows,
                 g_skinny_krot, g_skinny_dbg, g.qkv};
  if (EPI == EPI_QKV) p.out_rows = g.qkv.idx;  // the epilogue's row ids (loaded ahead of the chunk's transpose)
  DY_CUDA(launch_k(kern, dim3(2 * max_pairs), dim3(SK_THREADS), SK_SMEM, st, 2, maps, p));
  return DYLLM_OK;
}

unsigned long long *g_skinny_trace = nullptr;
int g_skinny_split = 0;
int g_skinny_one_chunk = 0;  // 0: automatic
int g_skinny_chunk_rows = 0;  // 0: 256
int g_skinny_krot = 0;
int g_skinny_dbg = 0;
int g_skinny_kb = 0;  // k-block width: 0 / 128 (default) or 64

bool skinny_eligible(const GemmCall &g) {
  // the epilogue stores 16-byte row segments (8 output columns) and reads bias / residual alike
  const auto a16 = [](const void *q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  return g.N % 256 == 0 && g.K % SK_KB == 0 &&
         (g.epi == EPI_BF16 || g.epi == EPI_RESID || g.epi == EPI_SWIGLU || g.epi == EPI_QKV) &&
         g.ldd % 8 == 0 && a16(g.D) && (!g.resid || (g.ldr % 8 == 0 && a16(g.resid))) && (!g.bias || a16(g.bias));
}

int gemm_skinny_launch(const GemmCall &g, int num_sms, cudaStream_t st) {
  if (g_skinny_kb == 64 && g.epi != EPI_QKV) {
    switch (g.epi) {
      case EPI_SWIGLU: return launch_skinny_t<EPI_SWIGLU, 1>(g, num_sms, st);
      case EPI_RESID: return launch_skinny_t<EPI_RESID, 1>(g, num_sms, st);
      default: return launch_skinny_t<EPI_BF16, 1>(g, num_sms, st);
    }
  }
  switch (g.epi) {
    case EPI_SWIGLU: return launch_skinny_t<EPI_SWIGLU, 2>(g, num_sms, st);
    case EPI_RESID: return launch_skinny_t<EPI_RESID, 2>(g, num_sms, st);
    case EPI_QKV: return launch_skinny_t<EPI_QKV, 2>(g, num_sms, st);
    default: return launch_skinny_t<EPI_BF16, 2>(g, num_sms, st);
  }
}

}  // namespace dy
