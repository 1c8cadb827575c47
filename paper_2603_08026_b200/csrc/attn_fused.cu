// attn_fused.cu — salient-query attention for head_dim 128 (LLaDA/Dream shapes), one persistent
// warp-specialised tcgen05 kernel (Alg. 4, D7).
//
// Work items, per (sequence s, query head h), ordered so that the items of one (s, kv head) run
// side by side and share the K/V tiles through L2:
//   type 1 — 128 consecutive input rows [row_lo + 128 t, ...) of s, read from the Q cache:
//       pass S : row max m and sum-exp l of s_rj = q_r.k_j * scale over ALL N keys (the dense
//                softmax normaliser of Alg. 4 lines 1-2, computed with the merged K);
//       pass P : over the salient keys only (compact K rows of idx_in, Kx), P = exp2(s - m),
//                dC = P dV (Alg. 4 lines 3-4, dV compact, aligned with idx_in);
//       output : approximate rows (not in idx_in): the delta dC / l (C_new = C_cache + dC is
//                formed by the similarity kernel, which reads C_cache anyway — no second read).
//   type 3 — (incremental statistics) a response tile whose cached (m, l) are
//       current: S over the salient keys' new and old K only, l updated by the difference, P dV as
//       in pass P; a row whose l cancels below 2^-14 sends its tile to the dense fixup launch.
//   type 2 — 33..128 exact rows (idx_in, compact new queries Qx) of s, one pass over the N keys:
//       P = exp2(s - ref) with ref = the first tile's row max (a row whose later scores exceed it by
//       more than 2^100 sends the item to the fixup launch, which re-runs it in two passes);
//       O = P V, l = sum P; output C = O / l scattered to the exact rows.
//   type 4 — <= 32 exact rows: type 2 transposed (S^T = K Q^T with the keys on the 128 MMA rows,
//       O^T += V^T P^T with P^T in shared memory), so the exps spread over all 16 softmax warps.
// Roles (640 threads, 1 CTA per SM): warp 0 claims items (decoded once, passed through a 4-slot
// shared-memory queue) and loads Q (double-buffered); warps 0, 18 and 19 load the K / V / dV tiles
// of a unified 4-slot ring in the MMA's consumption order, each every third tile (one 32 KB 3-D TMA
// op per tile; TMA issue throughput is per issuing thread, tools/tma_probe.cu); warp 1 lane 0 issues
// every tcgen05.mma (S = Q K^T into a double-buffered fp32 TMEM tile; P V into a 128x128 fp32 TMEM
// accumulator with P read from TMEM and V as an MN-major smem operand); warps 2-17 are the softmax /
// epilogue warps: four per TMEM lane quadrant, one row per thread, 32 of the 128 key columns of
// each score tile each; P is stored bf16x2-packed into TMEM with tcgen05.st.
#include "common.cuh"

#ifndef DYLLM_FA_X_FIRST
#define DYLLM_FA_X_FIRST 1  // exact-row items claimed first (fa_decode)
#endif
#include "internal.h"

namespace dy {

int g_attn_t4_rows = 32;

// Type-4 tiles (exact-row items of <= 32 rows computed transposed) are compiled only with
// -DDYLLM_FA_T4=1. Measured on one box (tools/gpu_exp62.sh): with them compiled in, the kernel's
// register allocation spills on the other item types' hot loops (76 B vs 12 B) and the attention
// class averages 169 us per launch (type 4 on) against 152 us with the code compiled out; an
// out-of-line type-4 function was slower still (199 us).
#ifndef DYLLM_FA_T4
#define DYLLM_FA_T4 0
#endif

constexpr int FA_BK = 128;                 // keys per tile (MMA N = 128: the Q operand read per
                                           // instruction is amortised over 128 keys)
constexpr int FA_Q_BYTES = 128 * 256;      // 128 rows x 128 bf16: two 64-column halves of 16 KB
constexpr int FA_KV_BYTES = 128 * 256;     // 128 keys x 128 bf16: two 64-column halves of 16 KB
constexpr int FA_QST = 2;
constexpr int FA_KVST = 4;                 // unified K / V / dV tile ring, filled in MMA consumption order
constexpr int FA_DATA = FA_QST * FA_Q_BYTES + FA_KVST * FA_KV_BYTES;
// softmax warps: FA_NG column groups x 4 TMEM lane quadrants; each warp owns 32 rows x FA_CW keys
// of a score tile (and FA_CW head dims of the output)
constexpr int FA_NG = 4;
constexpr int FA_CW = FA_BK / FA_NG;
constexpr int FA_NSW = 4 * FA_NG;           // softmax warps 2 .. 1 + FA_NSW
constexpr int FA_WV = 2 + FA_NSW;           // V / dV producer warp
constexpr int FA_WK2 = 3 + FA_NSW;          // second K producer warp
constexpr int FA_THREADS = 32 * (4 + FA_NSW);
constexpr int FA_XCH = FA_NG * 128 * 8;     // (m, l) per column group per row
constexpr int FA_PF = 3 * 128 * 16;         // row metadata of 3 items in flight (FaRow per row)
constexpr int FA_PT_BYTES = 32 * 256;       // type 4: P^T tile, 32 rows x 128 keys bf16 (K-major, SW128)
constexpr int FA_PT = 2 * FA_PT_BYTES;      // double-buffered
constexpr int FA_X4 = 4 * 4 * 8 * 4;        // type 4: per (column group, quad, row) partial max / sum
constexpr int FA_SMEM = 1024 + FA_DATA + FA_PT + FA_XCH + FA_PF + FA_X4 + 1024;
constexpr int FA_T4_MAX = 32;               // type 4: at most 32 rows (MMA N = 32)
static_assert(FA_CW % 32 == 0, "column groups are whole 32-column TMEM loads");
// TMEM columns: S[2] (2 x 128 fp32), accumulator (128 fp32), P[2] (2 x 64: 128 keys bf16x2-packed,
// the A operand of the P V MMA read straight from TMEM)
constexpr int FA_TMEM_COLS = 512;
constexpr uint32_t FA_ACC_COL = 256;
constexpr uint32_t FA_P_COL = 384;

struct FaParams {
  int N, row_lo, L, H, KVH, grp, MT, XT, items, qw;
  float c;                  // softmax scale * log2(e)
  const int *ex_off;        // [b+1]: exact rows (= salient keys) of each sequence, packed
  const int *ex_rows;       // packed row ids of the exact rows
  const uint32_t *rowflag;  // [b*N]: == tag for the exact rows of this step (type-1 tiles leave them to type 2)
  uint32_t tag;
  const bf16 *C_cache;
  bf16 *C_out;
  int *work_ctr;              // [2] dynamic scheduler: next item, finished CTAs (zero between launches)
  unsigned long long *events; // optional event log of CTAs 0-1 (debug hook): [cta][role][8192]
  float2 *stats;              // [b*N][H] softmax statistics per (row, head): (m c, l = sum 2^(s c - m c))
  int inc;                    // statistics of the response rows are current: incremental tiles allowed
  int resp_lo;                // first response position (L_P)
  int mode;                   // 0 denoising step, 1 fixup list (dense), 2 statistics refresh (no output)
  int *fix;                   // [0] count, [1 ..] ids of incremental tiles whose update cancelled
  int fix_cap;
  int t4max;                  // exact-row items of <= t4max rows run transposed (type 4; 0: never)
  // full-input steps with incremental prompt statistics (SURVEY §8f1 for the prompt rows): row
  // tiles are split at resp_lo (MTp prompt tiles, then the response tiles), and a prompt tile
  // updates its rows' statistics by the keys changed since they were last current (the list U of
  // each sequence: its idx_in rows first, then the keys written by the response-only steps since,
  // compact new keys Kun / snapshot keys Kuo at rows [s*N, s*N + ucnt[s]))
  int MTp;
  int pinc;                   // prompt statistics current up to U: incremental prompt tiles allowed
  const int *ucnt;            // [b] |U| per sequence
  // similarity partials fused into the epilogue: when set, the epilogue reads the
  // cached context C_old of each written row, commits C_new = C_old + dC (approximate rows) or C
  // (exact rows) into C_cache (= C_out) in place, and writes per (row, head) the partial sums
  // (<C_new, C_old>, |C_new|^2, |C_old|^2) over the head's dims, which the selection kernel adds
  // over the heads: the rows are read and written once, by the kernel that produces them
  float4 *cos_part;           // [b*N][H] or nullptr
};
// statistics entry of a row whose tile was handed to the fixup launch (its output was not written;
// the fixup launch recomputes exactly the rows carrying it)
constexpr float FA_PENDING = -1.f;

struct FaItem {
  int s, h, kvh, nrows, q_row, off, nkP, xc;
  int nkS;      // type 3: key count of its new / old key tiles (<= 2 tiles; first row s*N for U, else off)
  bool type2, passP;
  bool inc;     // type 3: incremental statistics (<= 128 salient keys, statistics current up to the
                // changed keys: idx_in for response tiles, U for prompt tiles of full-input steps)
  bool uk;      // type 3 over the U lists (prompt tile) instead of idx_in (Kx / Kxo)
  bool single;  // type 2 in one pass (online softmax); the fixup launch re-runs type 2 in two passes
  bool t4;      // type 2, single pass, <= 32 rows: computed transposed (keys on the MMA rows)
};

// Item decode from its index and the exact-row range (off, e) of its sequence (the producer reads
// those once and passes them through the work queue, so no role stalls on global loads).
// item index -> ((sequence, kv head, group member) index sh, slot t: row tiles 0..MT-1, exact-row
// tiles MT..MT+XT-1). DYLLM_FA_X_FIRST: every exact-row (type 2, the longest) item is claimed
// before any row-tile item, in (sequence, head) order, so the launch ends on short items; the two
// kinds read different key data (full K / V vs the compact changed keys), so nothing shared in L2
// is split. Otherwise the items of one (sequence, head) are adjacent, exact rows last.
__device__ __forceinline__ void fa_decode(const FaParams &p, int w, int &sh, int &t) {
  if (DYLLM_FA_X_FIRST) {
    const int n2 = p.items / (p.MT + p.XT) * p.XT;
    if (w < n2) {
      sh = w / p.XT;
      t = p.MT + w % p.XT;
    } else {
      sh = (w - n2) / p.MT;
      t = (w - n2) % p.MT;
    }
  } else {
    sh = w / (p.MT + p.XT);
    t = w % (p.MT + p.XT);
  }
}
__device__ __forceinline__ FaItem fa_item(const FaParams &p, int w, int off, int e, int nU) {
  FaItem it;
  int sh, t;
  fa_decode(p, w, sh, t);
  const int g = sh % p.grp;
  sh /= p.grp;
  it.kvh = sh % p.KVH;
  it.s = sh / p.KVH;
  it.h = it.kvh * p.grp + g;
  it.off = off;
  it.uk = false;
  it.nkS = e;
  if (t < p.MT) {
    it.type2 = false;
    it.xc = 0;
    const bool prompt = t < p.MTp;
    const int r0 = prompt ? p.row_lo + t * 128 : (p.MTp ? p.resp_lo : p.row_lo) + (t - p.MTp) * 128;
    it.q_row = it.s * p.N + r0;
    it.nrows = min(128, (prompt ? p.resp_lo : p.N) - r0);
    it.passP = e > 0 && p.mode != 2;
    it.nkP = e;
    it.single = false;
    it.t4 = false;
    if (prompt) {
      // the prompt rows' statistics are current up to the keys of U: incremental when U fits in
      // two key tiles (else dense); with no salient key there is no output, only the statistics
      it.inc = p.pinc && p.mode == 0 && e <= FA_BK && nU <= 2 * FA_BK;
      if (it.inc) {
        it.uk = true;
        it.nkS = nU;
        if (nU == 0) it.nrows = 0;  // no key changed since the statistics: nothing to do
      }
    } else {
      it.inc = p.inc && p.mode == 0 && e > 0 && e <= FA_BK && r0 >= p.resp_lo;
      // no salient key in the sequence: the keys did not change, so neither did the statistics
      // (when current) nor the contexts: nothing to do
      if (e == 0 && p.inc && p.mode == 0) it.nrows = 0;
    }
  } else {
    it.type2 = true;
    it.xc = t - p.MT;
    it.q_row = it.off + it.xc * 128;
    it.nrows = min(128, e - it.xc * 128);
    it.passP = true;
    it.nkP = p.N;
    it.inc = false;
    it.single = p.mode != 1;
    it.t4 = DYLLM_FA_T4 && it.single && it.nrows <= p.t4max;
  }
  return it;
}
__device__ __forceinline__ int fa_seq(const FaParams &p, int w) {
  int sh, t;
  fa_decode(p, w, sh, t);
  return sh / p.grp / p.KVH;
}

// UMMA descriptor of an MN-major operand tile written by TMA with 128B swizzle: 64-element
// (128 B) rows along MN, 8-row (K) core groups 1024 B apart (SBO), consecutive 64-element MN
// chunks `lbo` bytes apart (LBO), version 1, SWIZZLE_128B.
__device__ __forceinline__ uint64_t sw128_mn_desc(uint32_t smem_addr, uint32_t lbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr & 0x3FFFF) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}
__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x for x <= 0 on the FMA pipe (the SFU does 16 ex2/clk/SM on B200, measured by
// tools/pipe_probe.cu, and is the softmax bottleneck): x = k + f, k = rint(x) via the 1.5*2^23
// shifter, f in [-1/2, 1/2], 2^f by a cubic fitted for relative error (3e-4, far below bf16's
// 4e-3), 2^k added to the exponent field with one integer multiply-add. x is clamped at -127.
__device__ __forceinline__ float ex2p(float x) {
  x = fmaxf(x, -127.f);
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  const float q = fmaf(fmaf(fmaf(0.05753576f, f, 0.24192697f), f, 0.69278964f), f, 1.0f);
  return __int_as_float(__float_as_int(t) * 8388608 + __float_as_int(q));
}
// Exps per group of 4 computed on the FMA pipe (ex2p) in the dense passes; the rest on MUFU.
// ncu shows the XU pipe near saturation in full-input steps (profiles/r1l_attn_fi_full.md), but
// 2 of 4 measured slower than 1 of 4 (tools/gpu_exp44.sh: full-input step 35.2 vs 34.7 ms).
#ifndef DYLLM_FA_KACT
#define DYLLM_FA_KACT 1  // type 3: warps whose key columns hold no salient key skip their exps
#endif
#ifndef DYLLM_FA_POLY
#define DYLLM_FA_POLY 1
#endif
constexpr int FA_POLY = DYLLM_FA_POLY;
// D[tmem] (+)= A[tmem] * B[smem]^T (kind::f16, A read from tensor memory: M lanes x K/2 packed
// bf16x2 columns)
__device__ __forceinline__ void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// 32 lanes x 16 consecutive 32-bit TMEM columns from registers (thread i -> lane base + i)
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t v[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
// 32 lanes x 32 consecutive 32-bit TMEM columns from registers
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t v[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void fa_wait(uint64_t *bar, uint32_t ph) { mbar_wait(bar, ph); }
// per-row metadata of an item, fetched asynchronously one item ahead (cp.async -> shared memory):
// output row id, its row-kind tag, its cached softmax statistics
struct FaRow {
  int orow;
  uint32_t rf;
  float2 so;
};
__device__ __forceinline__ void cp_async_4(void *smem, const void *gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_8(void *smem, const void *gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// Named barrier of a TMEM lane quadrant's softmax warps. The non-.aligned form: the warps of a
// quadrant reach it from different code paths (e.g. type-3 warps with and without changed keys in
// their columns), which bar.sync (= barrier.sync.aligned) does not allow (compute-sanitizer
// synccheck); each warp is converged when it arrives.
__device__ __forceinline__ void fa_named_sync(int id, int n) {
  __syncwarp();
  asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// debug event log (compiled in with -DDYLLM_ATTN_EVENTS=1, tools/attn_events.py): one 8192-entry
// region per (CTA < 2, role); entry = code << 56 | clock64. With -DDYLLM_ATTN_EVENTS=2 the fourth
// role logs softmax warp 6 (quad 2, column group 1) instead of the V producer
#ifndef DYLLM_ATTN_EVENTS
#define DYLLM_ATTN_EVENTS 0
#endif
constexpr int FA_EV_N = 8192;
struct FaEv {
#if DYLLM_ATTN_EVENTS
  unsigned long long *buf = nullptr;
  int n = 0;
  __device__ __forceinline__ void operator()(int code) {
    if (buf && n < FA_EV_N) buf[n++] = (static_cast<unsigned long long>(code) << 56) | (clock64() & ((1ull << 56) - 1));
  }
  __device__ __forceinline__ void finish() {
    if (buf && n < FA_EV_N) buf[n] = 0;  // terminator (later launches overwrite the same region)
  }
  __device__ __forceinline__ void attach(unsigned long long *b) { buf = b; }
#else
  __device__ __forceinline__ void operator()(int) {}
  __device__ __forceinline__ void finish() {}
  __device__ __forceinline__ void attach(unsigned long long *) {}
#endif
};

// COS: the fused similarity-partials epilogue is compiled in (a separate instance,
// so its registers do not weigh on the default kernel)
template <bool COS>
__global__ void __launch_bounds__(FA_THREADS, 1)
    attn_fused_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmQx,
                      const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                      const __grid_constant__ CUtensorMap tmKx, const __grid_constant__ CUtensorMap tmDV,
                      const __grid_constant__ CUtensorMap tmKxo, const __grid_constant__ CUtensorMap tmKun,
                      const __grid_constant__ CUtensorMap tmKuo, const FaParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t *sQ = smem;                                   // [2][32 KB]
  uint8_t *sKV = sQ + FA_QST * FA_Q_BYTES;              // [4][32 KB] K, V or dV tiles
  uint8_t *sPT = sKV + FA_KVST * FA_KV_BYTES;           // [2][8 KB] type-4 P^T tiles (1024-aligned)
  float2 *xch = reinterpret_cast<float2 *>(sPT + FA_PT);  // [column group][128 rows]
  // similarity partial exchange [item parity][column group][128 rows] (the type-4 P^T tiles' space:
  // type 4 and the fused partials are never built together)
  float4 *cpx = reinterpret_cast<float4 *>(sPT);
  static_assert(DYLLM_FA_T4 == 0 || true, "");
  static_assert(2 * FA_NG * 128 * sizeof(float4) <= FA_PT, "partial exchange fits the P^T space");
  FaRow *rows_s = reinterpret_cast<FaRow *>(reinterpret_cast<uint8_t *>(xch) + FA_XCH);  // [3][128]
  float *x4 = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(rows_s) + FA_PF);  // [4 hh][4 quads][8]
  uint64_t *bars = reinterpret_cast<uint64_t *>(reinterpret_cast<uint8_t *>(x4) + FA_X4);
  uint64_t *q_full = bars, *q_empty = bars + 2;
  uint64_t *kv_full = bars + 4, *kv_empty = bars + 8;   // [FA_KVST]
  uint64_t *s_full = bars + 14, *s_empty = bars + 16;
  uint64_t *p_full = bars + 18, *p_empty = bars + 20;
  uint64_t *acc_full = bars + 22, *acc_empty = bars + 23;
  uint64_t *wq_full = bars + 24, *wq_empty = bars + 28;   // [4] work queue (producer -> other roles)
  int4 *wq = reinterpret_cast<int4 *>(bars + 32);          // [4] (item, off, e, -) ; item -1 = done
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(wq + 4);
  // the queue slots' items, decoded once by the claiming thread (the index arithmetic has three
  // runtime divisions; 500 threads re-deriving it per item was measurable)
  FaItem *wqi = reinterpret_cast<FaItem *>(bars + 48);  // [4]

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int NKT = (p.N + FA_BK - 1) / FA_BK;
  // fixup launch with an empty list (the common case): leave before any setup (no barrier init,
  // no TMEM allocation), so the step's next kernel follows right away
  if (p.mode == 1) {
    pdl_wait();
    if (*reinterpret_cast<volatile const int *>(p.fix) == 0) return;
  }
  // event roles: 0 MMA, 1 softmax warp 2, 2 producer warp 0, 3 V producer
  FaEv ev;
  {
    const int role = warp == 1 ? 0 : warp == 2 ? 1 : warp == 0 ? 2 : warp == (DYLLM_ATTN_EVENTS == 2 ? 6 : FA_WV) ? 3 : -1;
    if (p.events && p.mode == 0 && blockIdx.x < 2 && lane == 0 && role >= 0) ev.attach(p.events + (blockIdx.x * 4 + role) * FA_EV_N);
  }

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmQx);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmKx);
    tma_prefetch_desc(&tmDV);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], FA_NSW);
      mbar_init(&p_full[i], FA_NSW);
      mbar_init(&p_empty[i], 1);
    }
    for (int i = 0; i < FA_KVST; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, FA_NSW);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&wq_full[i], 1);
      mbar_init(&wq_empty[i], 3 + FA_NSW);  // MMA warp, V producer, second K producer, softmax warps
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, FA_TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_trigger();  // grid <= #SMs at one CTA per SM: resident, the next kernel may launch
  // Dynamic scheduling: the producer thread claims items with an atomic counter (items of one
  // (sequence, kv head) stay adjacent in claim order, so concurrently running CTAs share K/V in L2,
  // and heavy exact-row items no longer pile up on fixed CTAs) and passes them to the other roles
  // through a 4-deep shared-memory queue. Consumers: one arrival per warp.
  int wn = 0;  // queue position of this role
  auto next_item = [&](FaItem &it) -> int {
    const int slot = wn & 3;
    fa_wait(&wq_full[slot], (wn >> 2) & 1);
    const int w = wq[slot].x;
    if (w >= 0) it = wqi[slot];
    __syncwarp();
    if (lane == 0) mbar_arrive(&wq_empty[slot]);
    ++wn;
    return w;
  };

  if (warp == 0 || warp == FA_WK2 || warp == FA_WV) {
    // ================================================================ TMA producers. Warp 0 claims
    // items (work queue) and loads Q. All three producer warps walk the same tile sequence — the
    // order in which the MMA warp consumes K / V / dV tiles — and each issues every third tile
    // into the 4-slot ring (ring index g: slot g % 4), tripling the TMA issue rate of one thread
    const int pid = warp == 0 ? 0 : warp == FA_WK2 ? 1 : 2;
    int g = 0;  // ring index of the next tile in consumption order
    auto load_kv = [&](const CUtensorMap *m, int row, int kvh) {
      if (g % 3 == pid && lane == 0) {
        const int ks = g % FA_KVST;
        ev(60);
        fa_wait(&kv_empty[ks], ((g / FA_KVST) & 1) ^ 1);
        ev(61);
        mbar_expect_tx(&kv_full[ks], FA_KV_BYTES);
        tma_load_3d(sKV + ks * FA_KV_BYTES, m, &kv_full[ks], 0, row, kvh * 2);
      }
      ++g;
    };
    // warp 0 claims one item ahead: the queue already holds item i+1 while item i's tiles are
    // issued, and Q of item i+1 is loaded early in item i, so item boundaries cost no claim
    // latency and no exposed Q load
    int wnext = -1;
    FaItem inext;
    auto claim = [&]() {  // warp 0, lane 0: next non-empty item (or -1) into the queue
      ev(62);
      int w, off = 0, e = 0;
      FaItem fi;
      for (;;) {
        w = atomicAdd(&p.work_ctr[0], 1);
        if (p.mode == 1) {  // fixup launch: the listed tiles, processed densely
          const int nfix = p.fix[0];
          if (nfix > p.fix_cap)  // the list overflowed (entries were dropped): every item, densely
            w = w < p.items ? w : -1;
          else
            w = w < nfix ? p.fix[1 + w] : -1;
          if (w < 0) break;
        } else if (w >= p.items) {
          w = -1;
          break;
        }
        const int sq = fa_seq(p, w);
        off = p.ex_off[sq];
        e = p.ex_off[sq + 1] - off;
        fi = fa_item(p, w, off, e, p.pinc ? p.ucnt[sq] : 0);
        if (fi.nrows > 0) break;
      }
      const int slot = wn & 3;
      mbar_wait(&wq_empty[slot], ((wn >> 2) & 1) ^ 1);
      wq[slot] = make_int4(w, off, e, 0);
      if (w >= 0) wqi[slot] = fi;
      mbar_arrive(&wq_full[slot]);
      ev(63);
      ++wn;
      wnext = w;
      inext = fi;
    };
    auto load_q = [&](const FaItem &it, int qi) {
      const int qb = qi & 1;
      ev(64);
      fa_wait(&q_empty[qb], ((qi >> 1) & 1) ^ 1);
      ev(65);
      mbar_expect_tx(&q_full[qb], FA_Q_BYTES);
      tma_load_3d(sQ + qb * FA_Q_BYTES, it.type2 ? &tmQx : &tmQ, &q_full[qb], 0, it.q_row, it.h * 2);
    };
    int qi = 0;
    if (warp == 0 && lane == 0) {
      claim();
      if (wnext >= 0) load_q(inext, 0);
    }
    for (;;) {
      FaItem it;
      int w;
      if (warp == 0) {
        if (lane == 0) {
          w = wnext;
          if (w >= 0) {
            it = inext;
            claim();  // item i+1 into the queue now
          }
        }
        w = __shfl_sync(0xffffffffu, w, 0);
        if (w < 0) break;
        if (lane != 0) it = FaItem{};
      } else {
        w = next_item(it);
        if (w < 0) break;
      }
      const int seq0 = it.s * p.N;
      // Q of the next item is loaded right after this item's first tile is queued
      auto after_first = [&]() {
        if (warp == 0 && lane == 0 && wnext >= 0) load_q(inext, qi + 1);
      };
      if (it.inc) {  // type 3: new keys, the same keys before (tile pairs), then dV
        const CUtensorMap *mn = it.uk ? &tmKun : &tmKx, *mo = it.uk ? &tmKuo : &tmKxo;
        const int nt = (it.nkS + FA_BK - 1) / FA_BK;
        const int kbase = it.uk ? seq0 : it.off;
        for (int j = 0; j < nt; ++j) {
          load_kv(mn, kbase + j * FA_BK, it.kvh);
          if (j == 0) after_first();
          load_kv(mo, kbase + j * FA_BK, it.kvh);
        }
        if (it.passP) load_kv(&tmDV, it.off, it.kvh);
        ++qi;
        continue;
      }
      // pass S (type 1): the N keys
      if (!it.single) {
        for (int kt = 0; kt < NKT; ++kt) {
          load_kv(&tmK, seq0 + kt * FA_BK, it.kvh);
          if (kt == 0) after_first();
        }
      }
      // pass P, in the MMA warp's order: K'(0), K'(1), then K'(j+2), V'(j) for each j (K' = keys of
      // the P tiles, V' = their values: all keys + V for exact rows, salient keys + dV otherwise)
      if (it.passP) {
        const int n2 = (it.nkP + FA_BK - 1) / FA_BK;
        const CUtensorMap *mk = it.type2 ? &tmK : &tmKx, *mv = it.type2 ? &tmV : &tmDV;
        const int r0 = it.type2 ? seq0 : it.off;
        load_kv(mk, r0, it.kvh);
        if (it.single) after_first();
        if (n2 > 1) load_kv(mk, r0 + FA_BK, it.kvh);
        for (int j = 0; j < n2; ++j) {
          if (j + 2 < n2) load_kv(mk, r0 + (j + 2) * FA_BK, it.kvh);
          load_kv(mv, r0 + j * FA_BK, it.kvh);
        }
      }
      ++qi;
    }
  } else if (warp == 1) {
    // ================================================================ MMA issuer: one thread runs
    // the whole role (no per-instruction divergence handling), with every smem descriptor formed
    // once and advanced by constant offsets (the descriptor's address field is addr >> 4)
    if (lane == 0) {
      constexpr uint32_t id_qk = idesc_bf16_f32(128, FA_BK);
      constexpr uint32_t id_pv = idesc_bf16_f32(128, 128) | (1u << 16);  // B (V) MN-major
      // descriptors of slot 0; slot i is + i * (32 KB >> 4) in the address field
      const uint64_t kdesc0 = sw128_kmajor_desc(smem_u32(sKV));
      const uint64_t vdesc0 = sw128_mn_desc(smem_u32(sKV), FA_KV_BYTES / 2);
      const uint64_t qdesc0 = sw128_kmajor_desc(smem_u32(sQ));
      constexpr uint64_t kSlot = FA_KV_BYTES >> 4;
      // K-major operand: k-step kk (16 elements) at +32 B within a 64-column half, halves 16 KB apart
      auto koff = [](int kk) -> uint64_t { return static_cast<uint64_t>(((kk >> 2) * (FA_KV_BYTES / 2) + (kk & 3) * 32) >> 4); };
      int qi = 0, g = 0, sc = 0, pc = 0, ai = 0, wn1 = 0;  // g: K/V ring index
      for (;;) {
        // work queue (single-thread form of next_item)
        const int slot = wn1 & 3;
        fa_wait(&wq_full[slot], (wn1 >> 2) & 1);
        const int qw0 = wq[slot].x;
        FaItem it;
        if (qw0 >= 0) it = wqi[slot];
        mbar_arrive(&wq_empty[slot]);
        ++wn1;
        if (qw0 < 0) break;
        ev(it.inc ? (it.uk ? 4 : 3) : it.type2 ? 2 : 1);
        const int qb = qi & 1;
        fa_wait(&q_full[qb], (qi >> 1) & 1);
        ev(9);
        ++qi;
        const uint64_t qd = qdesc0 + qb * kSlot;
        auto qk = [&]() {
          const int sb = sc & 1;
          ev(10);
          fa_wait(&s_empty[sb], ((sc >> 1) & 1) ^ 1);
          ev(11);
          const int ks = g % FA_KVST;
          fa_wait(&kv_full[ks], (g / FA_KVST) & 1);
          ev(12);
          tc_fence_after();
          const uint64_t kd = kdesc0 + ks * kSlot;
          const uint32_t dst = tmem + sb * FA_BK;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) umma_bf16(dst, qd + koff(kk), kd + koff(kk), id_qk, kk > 0);
          umma_commit(&kv_empty[ks]);
          umma_commit(&s_full[sb]);
          ev(13);
          ++g;
          ++sc;
        };
        auto pv = [&](int j, int n2) {
          const int pb = pc & 1;
          ev(20);
          fa_wait(&p_full[pb], (pc >> 1) & 1);
          ev(21);
          const int vs = g % FA_KVST;
          fa_wait(&kv_full[vs], (g / FA_KVST) & 1);
          if (j == 0) fa_wait(acc_empty, (ai & 1) ^ 1);
          ev(22);
          tc_fence_after();
          const uint64_t vd = vdesc0 + vs * kSlot;
          const uint32_t pa = tmem + FA_P_COL + pb * 64;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)  // 16 keys per MMA: 8 packed TMEM columns of P, 2 KB of V
            umma_bf16_ts(tmem + FA_ACC_COL, pa + kk * 8, vd + static_cast<uint64_t>(kk * 2048 >> 4), id_pv,
                         (j | kk) != 0);
          umma_commit(&kv_empty[vs]);
          umma_commit(&p_empty[pb]);
          if (j == n2 - 1) umma_commit(acc_full);
          ev(23);
          ++g;
          ++pc;
        };
        if (it.inc) {  // type 3: (S_new, S_old) per key tile, then P dV (P from the first new tile)
          const int nt = (it.nkS + FA_BK - 1) / FA_BK;
          for (int j = 0; j < nt; ++j) {
            qk();
            qk();
          }
          if (it.passP) {
            pv(0, 1);
            ++ai;
          }
          umma_commit(&q_empty[qb]);
          continue;
        }
        if (DYLLM_FA_T4 && it.t4) {
          // type 4 (<= 32 exact rows), transposed: S^T = K Q^T (M = 128 keys, N = 32 rows: the K tile
          // is the A operand, the Q tile's first 32 rows the B operand, both K-major as loaded) and
          // O^T += V^T P^T (A = V, MN-major as loaded; B = P^T written by the softmax warps into a
          // K-major shared-memory tile). A quarter of the tensor work of a 128-row tile.
          constexpr uint32_t id_qkT = idesc_bf16_f32(128, FA_T4_MAX);
          constexpr uint32_t id_pvT = idesc_bf16_f32(128, FA_T4_MAX) | (1u << 15);  // A (V) MN-major
          const uint64_t ptdesc0 = sw128_kmajor_desc(smem_u32(sPT));
          auto koffp = [](int kk) -> uint64_t { return static_cast<uint64_t>(((kk >> 2) * (FA_PT_BYTES / 2) + (kk & 3) * 32) >> 4); };
          auto qkT = [&]() {
            const int sb = sc & 1;
            ev(10);
            fa_wait(&s_empty[sb], ((sc >> 1) & 1) ^ 1);
            ev(11);
            const int ks = g % FA_KVST;
            fa_wait(&kv_full[ks], (g / FA_KVST) & 1);
            ev(12);
            tc_fence_after();
            const uint64_t kd = kdesc0 + ks * kSlot;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) umma_bf16(tmem + sb * FA_BK, kd + koff(kk), qd + koff(kk), id_qkT, kk > 0);
            umma_commit(&kv_empty[ks]);
            umma_commit(&s_full[sb]);
            ev(13);
            ++g;
            ++sc;
          };
          auto pvT = [&](int j, int n2) {
            const int pb = pc & 1;
            ev(20);
            fa_wait(&p_full[pb], (pc >> 1) & 1);
            ev(21);
            const int vs = g % FA_KVST;
            fa_wait(&kv_full[vs], (g / FA_KVST) & 1);
            if (j == 0) fa_wait(acc_empty, (ai & 1) ^ 1);
            ev(22);
            tc_fence_after();
            const uint64_t vd = vdesc0 + vs * kSlot;
            const uint64_t pd = ptdesc0 + pb * (FA_PT_BYTES >> 4);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)  // 16 keys per MMA
              umma_bf16(tmem + FA_ACC_COL, vd + static_cast<uint64_t>(kk * 2048 >> 4), pd + koffp(kk), id_pvT,
                        (j | kk) != 0);
            umma_commit(&kv_empty[vs]);
            umma_commit(&p_empty[pb]);
            if (j == n2 - 1) umma_commit(acc_full);
            ev(23);
            ++g;
            ++pc;
          };
          qkT();
          if (NKT > 1) qkT();
          for (int j = 0; j < NKT; ++j) {
            if (j + 2 < NKT) qkT();
            pvT(j, NKT);
          }
          ++ai;
          umma_commit(&q_empty[qb]);
          continue;
        }
        if (!it.single)
          for (int kt = 0; kt < NKT; ++kt) qk();
        if (it.passP) {
          // two score tiles ahead of P V: the score tile j + 2 reuses the S buffer the softmax
          // read tile j out of, so it is issued while the softmax still computes P(j)
          const int n2 = (it.nkP + FA_BK - 1) / FA_BK;
          qk();
          if (n2 > 1) qk();
          for (int j = 0; j < n2; ++j) {
            if (j + 2 < n2) qk();
            pv(j, n2);
          }
          ++ai;
        }
        umma_commit(&q_empty[qb]);
      }
    }
    __syncwarp();
  } else {
    // ================================================================ softmax / epilogue warps
    const int quad = warp & 3;            // TMEM lane quadrant this warp may access
    const int hh = (warp - 2) >> 2;       // which FA_CW columns of a score tile (and head dims)
    const int r = quad * 32 + lane;       // row of the tile
    const uint32_t trow = tmem + (static_cast<uint32_t>(quad * 32) << 16);
    const float c = p.c;
    constexpr int NCH = FA_CW / 32;       // 32-column TMEM loads per warp and tile
    int sc = 0, pc = 0, ai = 0;
    // Row metadata of an item (output row id, row-kind tag, cached softmax statistics): global
    // loads that miss L2 (the weights stream through it every layer). The column-group-0 warps
    // fetch them with cp.async into shared memory one item ahead (the next item is taken from the
    // work queue as soon as the current one starts — the producer claims one ahead), into 3 slots
    // (no warp of a quad lags its group-0 warp by a whole item: they meet at a barrier in each);
    // every thread reads its row's entry only after the item's first quad barrier.
    auto fetch_rows = [&](const FaItem &x, int slot) {
      if (r >= x.nrows) return;
      FaRow *d = rows_s + slot * 128 + r;
      if (p.mode == 1) {  // fixup launch: every row's statistics (FA_PENDING marks the rows to redo)
        const int orow = x.type2 ? p.ex_rows[x.q_row + r] : x.q_row + r;
        d->orow = orow;
        if (!x.type2) cp_async_4(&d->rf, p.rowflag + orow);
        cp_async_8(&d->so, p.stats + static_cast<int64_t>(orow) * p.H + x.h);
      } else if (x.type2) {
        cp_async_4(&d->orow, p.ex_rows + x.q_row + r);
      } else {
        d->orow = x.q_row + r;
        cp_async_4(&d->rf, p.rowflag + x.q_row + r);
        if (x.inc) cp_async_8(&d->so, p.stats + static_cast<int64_t>(x.q_row + r) * p.H + x.h);
        // the contexts this item's epilogue reads (fused similarity partials): into L2 now
        if (COS && p.cos_part && x.passP) {
          const char *cc = reinterpret_cast<const char *>(p.C_cache + static_cast<int64_t>(x.q_row + r) * p.qw + x.h * 128);
          asm volatile("prefetch.global.L2 [%0];" ::"l"(cc));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(cc + 128));
        }
      }
    };
    // The softmax warps hold a queue slot until they finish its item (so the next item can be
    // read in place while the current one runs) and release it at the item's end.
    fa_wait(&wq_full[0], 0);
    int cw = wq[0].x;
    int ii = 0;  // item count of this warp = its queue position
    if (cw >= 0 && hh == 0) fetch_rows(wqi[0], 0);
    while (cw >= 0) {
      // the item, read in place from its queue slot (held until the item ends): no register copy
      // of the decoded item lives across the softmax phases
      const FaItem &it = wqi[ii & 3];
      const int w = cw;
      const int ns = (ii + 1) & 3;
      ev(4);
      fa_wait(&wq_full[ns], ((ii + 1) >> 2) & 1);
      const int nw = wq[ns].x;
      ev(5);
      if (hh == 0) {
        cp_async_wait_all();  // this item's rows (issued one item ago)
        if (nw >= 0) fetch_rows(wqi[ns], (ii + 1) % 3);
      }
      const FaRow *rp = rows_s + (ii % 3) * 128 + r;
      // warps whose 32 rows are all past the item's row count skip the softmax work (they still
      // take part in every barrier; their garbage P rows only reach accumulator rows never stored)
      const bool wact = quad * 32 < it.nrows;
      const bool rvalid = r < it.nrows;
      // (after the item's first quad barrier) type 1 / 3 write approximate rows only (exact rows
      // belong to the type-2 items); statistics entries likewise
      // fixup launch: only the rows the first launch left pending
      auto live = [&]() { return p.mode != 1 || rp->so.y == FA_PENDING; };
      auto write_row = [&]() { return rvalid && (it.type2 || (it.passP && rp->rf != p.tag)) && live(); };
      auto own_stats = [&]() {
        return p.stats != nullptr && rvalid && hh == 0 && (it.type2 || p.mode == 2 || rp->rf != p.tag) && live();
      };
      bool rbad = false;  // this row's tile goes to the fixup launch: no output, statistics pending
      auto srow = [&]() { return static_cast<int64_t>(rp->orow) * p.H + it.h; };
      ev(it.inc ? (it.uk ? 4 : 3) : it.type2 ? 2 : 1);
      float acc[FA_CW];
      float oscale = 1.f;
      if (DYLLM_FA_T4 && it.t4) {
        // ---- type 4: <= 32 exact rows, transposed. S^T in TMEM: lane = key (this thread: key kq of
        // each tile), column = row (this warp: rows n0 .. n0+7). One pass over the N keys as in the
        // single-pass type 2: P = 2^((s - ref) c) with ref = the first tile's row max (reduced over the
        // lanes with an order-preserving integer redux, over the 4 quads through shared memory),
        // written bf16 into the K-major P^T tile (B operand of O^T += V^T P^T); l per row summed per
        // key thread and reduced once at the end. A row whose later scores exceed ref by > 2^100
        // sends the item to the fixup launch (two-pass, as type 2).
        const int kq = quad * 32 + lane;
        const int n0 = hh * 8;
        auto ford = [](float f) { const int i = __float_as_int(f); return i >= 0 ? i : i ^ 0x7fffffff; };
        auto unord = [](int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); };
        float ref[8], lp[8];
        float over = -INFINITY;
#pragma unroll
        for (int i = 0; i < 8; ++i) lp[i] = 0.f;
        for (int j = 0; j < NKT; ++j) {
          const int sb = sc & 1;
          fa_wait(&s_full[sb], (sc >> 1) & 1);
          ++sc;
          const int pb = pc & 1;
          ++pc;
          tc_fence_after();
          float v[8];
          tmem_ld8(trow + sb * FA_BK + n0, v);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&s_empty[sb]);
          const bool kvalid = j * FA_BK + kq < p.N;
          if (j == 0) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int m = __reduce_max_sync(0xffffffffu, ford(kvalid ? v[i] : -INFINITY));
              if (lane == 0) x4[(hh * 4 + quad) * 8 + i] = unord(m);
            }
            fa_named_sync(5 + hh, 128);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              float m = x4[(hh * 4) * 8 + i];
#pragma unroll
              for (int q2 = 1; q2 < 4; ++q2) m = fmaxf(m, x4[(hh * 4 + q2) * 8 + i]);
              ref[i] = m * c;
            }
            fa_named_sync(5 + hh, 128);
          }
          fa_wait(&p_empty[pb], (((pc - 1) >> 1) & 1) ^ 1);
          // P^T element (row n, key kq): half kq / 64, row line n (128 B), 16-byte chunk
          // ((kq % 64) / 8) ^ (n % 8) (128-byte swizzle), 2 bytes at (kq % 8)
          const uint32_t pt = smem_u32(sPT + pb * FA_PT_BYTES + (kq >> 6) * (FA_PT_BYTES / 2)) + (kq & 7) * 2;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int n = n0 + i;
            const float x = kvalid ? fmaf(v[i], c, -ref[i]) : -INFINITY;
            if (n < it.nrows) over = fmaxf(over, x);
            const float pv = ex2f(x);
            lp[i] += pv;
            const __nv_bfloat16 hb = __float2bfloat16_rn(pv);
            const uint32_t addr = pt + n * 128 + ((((kq & 63) >> 3) ^ (n & 7)) << 4);
            asm volatile("st.shared.b16 [%0], %1;" ::"r"(addr), "h"(*reinterpret_cast<const unsigned short *>(&hb)) : "memory");
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_full[pb]);
        }
        fa_wait(acc_full, ai & 1);
        ++ai;
        tc_fence_after();
        float o[8];
        tmem_ld8(trow + FA_ACC_COL + n0, o);   // O^T: lane = head dim kq, columns = rows n0 ..
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty);
        // row sums: lanes (fixed butterfly order), then quads 0..3
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float t = warp_sum(lp[i]);
          if (lane == 0) x4[(hh * 4 + quad) * 8 + i] = t;
        }
        fa_named_sync(5 + hh, 128);
        float L[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float t = x4[(hh * 4) * 8 + i];
#pragma unroll
          for (int q2 = 1; q2 < 4; ++q2) t += x4[(hh * 4 + q2) * 8 + i];
          L[i] = t;
        }
        // every softmax warp reads the rows' output ids fetched by the column-group-0 warp of quad 0
        fa_named_sync(9, 32 * FA_NSW);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int n = n0 + i;
          if (n < it.nrows) {
            const int orr = rows_s[(ii % 3) * 128 + n].orow;
            p.C_out[static_cast<int64_t>(orr) * p.qw + it.h * 128 + kq] = __float2bfloat16_rn(o[i] / L[i]);
            if (p.stats != nullptr && quad == 0 && lane == i)
              p.stats[static_cast<int64_t>(orr) * p.H + it.h] = make_float2(ref[i], L[i]);
          }
        }
        if (__ballot_sync(0xffffffffu, over > 100.f) != 0u && lane == 0) {
          const int pos = atomicAdd(&p.fix[0], 1);
          if (pos < p.fix_cap) p.fix[1 + pos] = w;
        }
      } else if (it.inc) {
        // ---- type 3, incremental statistics (exact up to rounding): only the keys in
        // the item's changed-key list (idx_in for response tiles, U for prompt tiles) differ from
        // the keys this row's statistics (m_old, l_old) were computed with, so
        //   l_new = l_old 2^(m_old - m) - sum_j 2^(s_old_j c - m) + sum_j 2^(s_new_j c - m),
        // with m = max(m_old, max over the first new tile of s_new c); P = 2^(s_new c - m) over the
        // salient keys (the first it.nkP columns of the first new tile) feeds P dV. All exps on MUFU
        // (the removed and added terms must carry no systematic error). A row whose l_new cancels
        // below 2^-14 of l_old (the changed keys held nearly all its attention), or whose later new
        // keys score 2^64 above m, sends its tile to the dense fixup launch.
        float2 so = make_float2(0.f, 1.f);
        const int nt = (it.nkS + FA_BK - 1) / FA_BK;
        float part = 0.f, mref = 0.f;
        bool over = false;
        // the old keys of a tile: their terms leave the normaliser
        auto old_tile = [&](int nvalid) {
          const int sb = sc & 1;
          fa_wait(&s_full[sb], (sc >> 1) & 1);
          ev(43);
          ++sc;
          if (wact && nvalid > 0) {
            tc_fence_after();
            float v[FA_CW];
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) tmem_ld32(trow + sb * FA_BK + hh * FA_CW + ch * 32, v + ch * 32);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[sb]);
            ev(47);
            float sub = 0.f;
#pragma unroll
            for (int t = 0; t < FA_CW; ++t) sub += ex2f(t < nvalid ? fmaf(v[t], c, -mref) : -INFINITY);
            part -= sub;
          } else {
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[sb]);
          }
        };
        {  // ---- tile 0: the new keys (m, P of the salient keys), then the same keys before
          // this warp's valid key columns (the MUFU work follows the changed-key count, not the
          // 128-key tile: warps without one skip their exps)
          const int nvalid = min(FA_CW, it.nkS - hh * FA_CW);
          const bool kact = !DYLLM_FA_KACT || nvalid > 0;
          const int sb = sc & 1;
          ev(40);
          fa_wait(&s_full[sb], (sc >> 1) & 1);
          ev(41);
          ++sc;
          int pb = 0;
          if (it.passP) {
            pb = pc & 1;
            ++pc;
          }
          if (!wact) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[sb]);
            if (it.passP) {
              fa_wait(&p_empty[pb], (((pc - 1) >> 1) & 1) ^ 1);
              __syncwarp();
              if (lane == 0) mbar_arrive(&p_full[pb]);
            }
          } else if (!kact) {  // no changed key in this warp's columns: no exps, P = 0
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[sb]);
            xch[hh * 128 + r].x = -INFINITY;
            fa_named_sync(1 + quad, 32 * FA_NG);
            float mn = -INFINITY;
#pragma unroll
            for (int g2 = 0; g2 < FA_NG; ++g2) mn = fmaxf(mn, xch[g2 * 128 + r].x);
            fa_named_sync(1 + quad, 32 * FA_NG);
            if (rvalid) so = rp->so;
            mref = fmaxf(so.x, mn * c);
            if (it.passP) {
              fa_wait(&p_empty[pb], (((pc - 1) >> 1) & 1) ^ 1);
              tc_fence_after();
              uint32_t pk[16];
#pragma unroll
              for (int t = 0; t < 16; ++t) pk[t] = 0u;
#pragma unroll
              for (int ch = 0; ch < NCH; ++ch) tmem_st16(trow + FA_P_COL + pb * 64 + hh * (FA_CW / 2) + ch * 16, pk);
              tmem_st_wait();
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&p_full[pb]);
            }
          } else {
            tc_fence_after();
            float v[FA_CW];
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) tmem_ld32(trow + sb * FA_BK + hh * FA_CW + ch * 32, v + ch * 32);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[sb]);
            ev(44);
            float tmax = -INFINITY;
#pragma unroll
            for (int t = 0; t < FA_CW; ++t) {
              if (t >= nvalid) v[t] = -INFINITY;
              tmax = fmaxf(tmax, v[t]);
            }
            xch[hh * 128 + r].x = tmax;
            fa_named_sync(1 + quad, 32 * FA_NG);
            float mn = -INFINITY;
#pragma unroll
            for (int g2 = 0; g2 < FA_NG; ++g2) mn = fmaxf(mn, xch[g2 * 128 + r].x);
            fa_named_sync(1 + quad, 32 * FA_NG);
            if (rvalid) so = rp->so;
            mref = fmaxf(so.x, mn * c);
            ev(45);
            if (it.passP) {
              // P over the salient keys (columns < nkP), bf16x2-packed into the P buffer; every
              // valid column's term (masked keys: 2^-inf = 0) enters the normaliser
              const int npv = it.nkP - hh * FA_CW;
              fa_wait(&p_empty[pb], (((pc - 1) >> 1) & 1) ^ 1);
              ev(46);
              tc_fence_after();
#pragma unroll
              for (int ch = 0; ch < NCH; ++ch) {
                uint32_t pk[16];
#pragma unroll
                for (int t = 0; t < 16; ++t) {
                  const int t0 = ch * 32 + 2 * t;
                  const float p0 = ex2f(fmaf(v[t0], c, -mref)), p1 = ex2f(fmaf(v[t0 + 1], c, -mref));
                  part += p0 + p1;
                  pk[t] = pack2(t0 < npv ? p0 : 0.f, t0 + 1 < npv ? p1 : 0.f);
                }
                tmem_st16(trow + FA_P_COL + pb * 64 + hh * (FA_CW / 2) + ch * 16, pk);
              }
              tmem_st_wait();
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&p_full[pb]);
            } else {
#pragma unroll
              for (int t = 0; t < FA_CW; ++t) part += ex2f(fmaf(v[t], c, -mref));
            }
          }
          ev(42);
          old_tile(nvalid);
        }
        for (int jt = 1; jt < nt; ++jt) {  // ---- further tiles of U (prompt tiles): sums only
          const int nvalid = min(FA_CW, it.nkS - (jt * FA_BK + hh * FA_CW));
          const int sb = sc & 1;
          fa_wait(&s_full[sb], (sc >> 1) & 1);
          ++sc;
          if (wact && nvalid > 0) {
            tc_fence_after();
            float v[FA_CW];
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) tmem_ld32(trow + sb * FA_BK + hh * FA_CW + ch * 32, v + ch * 32);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[sb]);
            float add = 0.f, tmax = -INFINITY;
#pragma unroll
            for (int t = 0; t < FA_CW; ++t) {
              const float x = t < nvalid ? fmaf(v[t], c, -mref) : -INFINITY;
              tmax = fmaxf(tmax, x);
              add += ex2f(x);
            }
            over = over || tmax > 64.f;
            part += add;
          } else {
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[sb]);
          }
          old_tile(nvalid);
        }
        float Lnew = 1.f;
        bool bad = false;
        if (wact) {
          ev(48);
          xch[hh * 128 + r].y = over ? NAN : part;  // every column group of the row sees the verdict
          fa_named_sync(1 + quad, 32 * FA_NG);
          ev(49);
          float tot = 0.f;
#pragma unroll
          for (int g2 = 0; g2 < FA_NG; ++g2) tot += xch[g2 * 128 + r].y;
          fa_named_sync(1 + quad, 32 * FA_NG);
          ev(53);
          const float base = so.y * ex2f(so.x - mref);
          Lnew = base + tot;
          bad = !(so.y > 0.f) || !(Lnew > base * 0x1p-14f) || !(Lnew < INFINITY);
          if (own_stats()) p.stats[srow()] = bad ? make_float2(0.f, FA_PENDING) : make_float2(mref, Lnew);
        }
        rbad = bad;
        // a tile with a cancelled row is recomputed densely by the fixup launch (duplicates of a
        // tile id are harmless: the dense recomputation is deterministic); `over` is per column
        // group, so every warp's rows vote
        if (__ballot_sync(0xffffffffu, bad && rvalid && (it.type2 || rp->rf != p.tag)) != 0u && lane == 0) {
          const int pos = atomicAdd(&p.fix[0], 1);
          if (pos < p.fix_cap) p.fix[1 + pos] = w;
        }
        ev(50);
        if (it.passP) {
                    fa_wait(acc_full, ai & 1);
          ev(51);
          ++ai;
          if (wact) {
            tc_fence_after();
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) tmem_ld32(trow + FA_ACC_COL + hh * FA_CW + ch * 32, acc + ch * 32);
            tc_fence_before();
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(acc_empty);
          ev(54);
        }
        oscale = 1.f / Lnew;
      } else if (it.single) {
        // ---- exact rows: one pass over the N keys. P = 2^((s - ref) c) with ONE reference per
        // row, the max of the first key tile (exchanged between the row's column groups once):
        // no per-tile agreement is needed, P may exceed 1 (fp32 / bf16 keep their relative
        // precision at any magnitude). A row whose later scores exceed the reference by more than
        // 2^100 (overflow risk) sends the item to the fixup launch, which re-runs it in two passes.
        float ref = -INFINITY, l = 0.f, over = -INFINITY;
        for (int j = 0; j < NKT; ++j) {
          const int sb = sc & 1;
          ev(40);
          fa_wait(&s_full[sb], (sc >> 1) & 1);
          ev(41);
          ++sc;
          const int pb = pc & 1;
          ++pc;
          if (!wact) {  // the whole quad is past the item's rows: keep the barrier protocol only
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[sb]);
            fa_wait(&p_empty[pb], (((pc - 1) >> 1) & 1) ^ 1);
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[pb]);
            continue;
          }
          tc_fence_after();
          float v[FA_CW];
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) tmem_ld32(trow + sb * FA_BK + hh * FA_CW + ch * 32, v + ch * 32);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&s_empty[sb]);
          const int k0 = j * FA_BK + hh * FA_CW;
          if (k0 + FA_CW > p.N) {
#pragma unroll
            for (int t = 0; t < FA_CW; ++t)
              if (k0 + t >= p.N) v[t] = -INFINITY;
          }
          float tmax = -INFINITY;
#pragma unroll
          for (int t = 0; t < FA_CW; ++t) tmax = fmaxf(tmax, v[t]);
          if (j == 0) {
            // the row reference: max over the first tile (all column groups; key 0 is valid)
            xch[hh * 128 + r].x = tmax;
            fa_named_sync(1 + quad, 32 * FA_NG);
#pragma unroll
            for (int g2 = 0; g2 < FA_NG; ++g2) ref = fmaxf(ref, xch[g2 * 128 + r].x);
          } else {
            over = fmaxf(over, (tmax - ref) * c);
          }
          const float rc = ref * c;
          // P = exp2((s - ref) c), bf16x2-packed into the P buffer; l sums the fp32 values
          fa_wait(&p_empty[pb], (((pc - 1) >> 1) & 1) ^ 1);
          tc_fence_after();
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) {
            uint32_t pk[16];
#pragma unroll
            for (int t = 0; t < 16; ++t) {
              const float x0 = v[ch * 32 + 2 * t], x1 = v[ch * 32 + 2 * t + 1];
              const float p0 = ex2f(fmaf(x0, c, -rc));
              const float p1 = (FA_POLY >= 2 || (t & 1)) ? ex2p(fmaf(x1, c, -rc)) : ex2f(fmaf(x1, c, -rc));
              l += p0 + p1;
              pk[t] = pack2(p0, p1);
            }
            tmem_st16(trow + FA_P_COL + pb * 64 + hh * (FA_CW / 2) + ch * 16, pk);
          }
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_full[pb]);
          ev(42);
        }
        ev(50);
                fa_wait(acc_full, ai & 1);
        ev(51);
        ++ai;
        if (wact) {
          tc_fence_after();
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) tmem_ld32(trow + FA_ACC_COL + hh * FA_CW + ch * 32, acc + ch * 32);
          tc_fence_before();
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty);
        // row normaliser: the column groups' sums share the reference (fixed order 0, 1, ...)
        float L = 0.f;
        if (wact) {
          xch[hh * 128 + r].y = over > 100.f ? NAN : l;  // overflow risk in any column group: the row is redone
          fa_named_sync(1 + quad, 32 * FA_NG);
#pragma unroll
          for (int g2 = 0; g2 < FA_NG; ++g2) L += xch[g2 * 128 + r].y;
          fa_named_sync(1 + quad, 32 * FA_NG);
          rbad = !(L > 0.f && L < INFINITY);
          if (own_stats()) p.stats[srow()] = rbad ? make_float2(0.f, FA_PENDING) : make_float2(ref * c, L);
        }
        oscale = 1.f / L;
        if (__ballot_sync(0xffffffffu, rvalid && rbad) != 0u && lane == 0) {
          const int pos = atomicAdd(&p.fix[0], 1);
          if (pos < p.fix_cap) p.fix[1 + pos] = w;
        }
      } else {
      // ---- pass S: running (m, l) of this column group of the row
      float m = -INFINITY, l = 0.f;
      for (int kt = 0; kt < NKT; ++kt) {
        const int sb = sc & 1;
        ev(30);
        fa_wait(&s_full[sb], (sc >> 1) & 1);
        ev(31);
        ++sc;
        if (!wact) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&s_empty[sb]);
          continue;
        }
        tc_fence_after();
        float v[FA_CW];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) tmem_ld32(trow + sb * FA_BK + hh * FA_CW + ch * 32, v + ch * 32);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[sb]);
        ev(32);
        const int k0 = kt * FA_BK + hh * FA_CW;
        if (k0 + FA_CW > p.N) {  // ragged last tile: mask keys >= N
#pragma unroll
          for (int j = 0; j < FA_CW; ++j)
            if (k0 + j >= p.N) v[j] = -INFINITY;
        }
        float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
        for (int j = 0; j < FA_CW; j += 4) {
          mx0 = fmaxf(mx0, v[j]);
          mx1 = fmaxf(mx1, v[j + 1]);
          mx2 = fmaxf(mx2, v[j + 2]);
          mx3 = fmaxf(mx3, v[j + 3]);
        }
        const float mt = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
        const float mn = fmaxf(m, mt);
        if (mn == -INFINITY) continue;  // every key of this column group masked
        const float mnc = mn * c;
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
        for (int j = 0; j < FA_CW; j += 4) {
          a0 += ex2f(fmaf(v[j], c, -mnc));
          a1 += FA_POLY >= 2 ? ex2p(fmaf(v[j + 1], c, -mnc)) : ex2f(fmaf(v[j + 1], c, -mnc));
          a2 += ex2f(fmaf(v[j + 2], c, -mnc));
          a3 += ex2p(fmaf(v[j + 3], c, -mnc));  // FA_POLY of 4 exps on the FMA pipe
        }
        l = l * ex2f((m - mn) * c) + ((a0 + a1) + (a2 + a3));
        m = mn;
        ev(33);
      }
      // ---- combine the column groups of each row (fixed order: group 0, 1, ...)
      xch[hh * 128 + r] = make_float2(m, l);
      fa_named_sync(1 + quad, 32 * FA_NG);
      float2 hg[FA_NG];
#pragma unroll
      for (int g = 0; g < FA_NG; ++g) hg[g] = xch[g * 128 + r];
      fa_named_sync(1 + quad, 32 * FA_NG);
      float M = -INFINITY;
#pragma unroll
      for (int g = 0; g < FA_NG; ++g) M = fmaxf(M, hg[g].x);
      float Lsum = 0.f;
#pragma unroll
      for (int g = 0; g < FA_NG; ++g) Lsum += hg[g].x == -INFINITY ? 0.f : hg[g].y * ex2f((hg[g].x - M) * c);
      const float Mc = M * c;
      const float inv_l = 1.f / Lsum;
      if (wact && own_stats()) p.stats[srow()] = make_float2(Mc, Lsum);
      // ---- pass P: P = exp2(s - m) into tensor memory for the P V MMA
      oscale = inv_l;
      if (it.passP) {
        const int n2 = (it.nkP + FA_BK - 1) / FA_BK;
        for (int j = 0; j < n2; ++j) {
          const int sb = sc & 1;
          ev(40);
          fa_wait(&s_full[sb], (sc >> 1) & 1);
          ev(41);
          ++sc;
          const int pb = pc & 1;
          ++pc;
          if (!wact) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[sb]);
            fa_wait(&p_empty[pb], (((pc - 1) >> 1) & 1) ^ 1);
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[pb]);
            continue;
          }
          // P = exp2(s - m) for this group's FA_CW keys, bf16x2-packed into the P TMEM buffer
          // (FA_CW / 2 columns per group); the S buffer is released once all chunks are read
          fa_wait(&p_empty[pb], (((pc - 1) >> 1) & 1) ^ 1);
          tc_fence_after();
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) {
            const int k0 = j * FA_BK + hh * FA_CW + ch * 32;
            uint32_t pk[16];
            if (k0 < it.nkP) {
              float v[32];
              tmem_ld32(trow + sb * FA_BK + hh * FA_CW + ch * 32, v);
#pragma unroll
              for (int t = 0; t < 16; ++t) {
                const float e1 = (FA_POLY >= 2 || (t & 1)) ? ex2p(fmaf(v[2 * t + 1], c, -Mc)) : ex2f(fmaf(v[2 * t + 1], c, -Mc));
                const float p0 = (k0 + 2 * t < it.nkP) ? ex2f(fmaf(v[2 * t], c, -Mc)) : 0.f;
                const float p1 = (k0 + 2 * t + 1 < it.nkP) ? e1 : 0.f;
                pk[t] = pack2(p0, p1);
              }
            } else {  // past the salient keys: P = 0, no exps
#pragma unroll
              for (int t = 0; t < 16; ++t) pk[t] = 0u;
            }
            tmem_st16(trow + FA_P_COL + pb * 64 + hh * (FA_CW / 2) + ch * 16, pk);
          }
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&s_empty[sb]);
            mbar_arrive(&p_full[pb]);
          }
          ev(42);
        }
        ev(50);
                fa_wait(acc_full, ai & 1);
        ev(51);
        ++ai;
        if (wact) {
          tc_fence_after();
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) tmem_ld32(trow + FA_ACC_COL + hh * FA_CW + ch * 32, acc + ch * 32);
          tc_fence_before();
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty);
      }
      }  // type 1
      // ---- epilogue: this thread's row, head columns [hh*FA_CW, (hh+1)*FA_CW). Exact rows
      // (type 2): C = O / l. Approximate rows (type 1): the delta dC / l only; the similarity
      // kernel, which reads C_cache anyway, forms C_new = C_cache + dC (no C_cache read here).
      // Stores are made coalesced first: a 4 x 4 transpose of 16-byte chunks inside each group of
      // 4 lanes (two xor-shuffle rounds) leaves lane c of group m holding chunk c of rows
      // 4m .. 4m+3, so each store instruction writes 8 rows x 64 contiguous bytes instead of 32
      // rows x 16 bytes.
      static_assert(FA_CW == 32, "epilogue transpose assumes 4 chunks of 8 head dims per warp");
      {
        const bool wr = write_row() && !rbad;
        const unsigned wmask = (DYLLM_FA_T4 && it.t4) ? 0u : __ballot_sync(0xffffffffu, wr);
        const bool fuse = COS && p.cos_part != nullptr && wact;
        auto shfl4 = [](uint4 v, int m) {
          return make_uint4(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m),
                            __shfl_xor_sync(0xffffffffu, v.z, m), __shfl_xor_sync(0xffffffffu, v.w, m));
        };
        // store 4 chunks of this thread's row slice: a 4 x 4 transpose of 16-byte chunks inside each
        // group of 4 lanes (two xor-shuffle rounds) leaves lane c of group m holding chunk c of rows
        // 4m .. 4m+3, so each store instruction writes 8 rows x 64 contiguous bytes
        auto store_rows = [&](uint4 ch[4]) {
          const bool b0 = lane & 1, b1 = lane & 2;
#pragma unroll
          for (int a = 0; a < 4; a += 2) {  // round 1: chunk pairs (0,1), (2,3) with lane ^ 1
            const uint4 rv = shfl4(b0 ? ch[a] : ch[a + 1], 1);
            if (b0) ch[a] = rv; else ch[a + 1] = rv;
          }
#pragma unroll
          for (int a = 0; a < 2; ++a) {     // round 2: chunk pairs (0,2), (1,3) with lane ^ 2
            const uint4 rv = shfl4(b1 ? ch[a] : ch[a + 2], 2);
            if (b1) ch[a] = rv; else ch[a + 2] = rv;
          }
          const int orow_l = rvalid ? rp->orow : 0;
          const int g4 = lane & ~3;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int src = g4 | k;
            const int orr = __shfl_sync(0xffffffffu, orow_l, src);
            if ((wmask >> src) & 1u)
              *reinterpret_cast<uint4 *>(p.C_out + static_cast<int64_t>(orr) * p.qw + it.h * 128 + hh * FA_CW +
                                         (lane & 3) * 8) = ch[k];
          }
        };
        if (fuse) {
          // ---- fused similarity partials, in the transposed layout (lane: 8 head dims
          // of rows g4..g4+3, coalesced): C_new = C_old + dC rounded as stored (approximate rows) or
          // C (exact rows); partial sums over the dims, then over the 4 lanes of each row, then over
          // the row's four column groups (fixed orders); C_new committed to the C cache (Alg. 3
          // line 16) by the kernel that forms it
          uint4 ch[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            float o[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) o[t] = acc[u * 8 + t] * oscale;
            ch[u] = pack8(o);
          }
          const bool b0 = lane & 1, b1 = lane & 2;
#pragma unroll
          for (int a = 0; a < 4; a += 2) {
            const uint4 rv = shfl4(b0 ? ch[a] : ch[a + 1], 1);
            if (b0) ch[a] = rv; else ch[a + 1] = rv;
          }
#pragma unroll
          for (int a = 0; a < 2; ++a) {
            const uint4 rv = shfl4(b1 ? ch[a] : ch[a + 2], 2);
            if (b1) ch[a] = rv; else ch[a + 2] = rv;
          }
          const int orow_l = rvalid ? rp->orow : 0;
          const int g4 = lane & ~3;
          float pd[4], pa[4], pb[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int src = g4 | k;
            const int orr = __shfl_sync(0xffffffffu, orow_l, src);
            pd[k] = pa[k] = pb[k] = 0.f;
            if ((wmask >> src) & 1u) {
              uint4 *cp = reinterpret_cast<uint4 *>(p.C_out + static_cast<int64_t>(orr) * p.qw + it.h * 128 +
                                                    hh * FA_CW + (lane & 3) * 8);
              float o[8], b8[8];
              unpack8(*cp, b8);
              unpack8(ch[k], o);
              if (!it.type2) {
#pragma unroll
                for (int t = 0; t < 8; ++t) o[t] += b8[t];
                ch[k] = pack8(o);
                unpack8(ch[k], o);
              }
#pragma unroll
              for (int t = 0; t < 8; ++t) {
                pd[k] = fmaf(o[t], b8[t], pd[k]);
                pa[k] = fmaf(o[t], o[t], pa[k]);
                pb[k] = fmaf(b8[t], b8[t], pb[k]);
              }
              *cp = ch[k];
            }
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
#pragma unroll
            for (int o = 1; o <= 2; o <<= 1) {
              pd[k] += __shfl_xor_sync(0xffffffffu, pd[k], o);
              pa[k] += __shfl_xor_sync(0xffffffffu, pa[k], o);
              pb[k] += __shfl_xor_sync(0xffffffffu, pb[k], o);
            }
          }
          const int mk = lane & 3;  // this lane's own row (row layout) is g4 | mk
          float4 *cx = cpx + (ii & 1) * (FA_NG * 128);
          cx[hh * 128 + r] = make_float4(mk == 0 ? pd[0] : mk == 1 ? pd[1] : mk == 2 ? pd[2] : pd[3],
                                         mk == 0 ? pa[0] : mk == 1 ? pa[1] : mk == 2 ? pa[2] : pa[3],
                                         mk == 0 ? pb[0] : mk == 1 ? pb[1] : mk == 2 ? pb[2] : pb[3], 0.f);
          fa_named_sync(1 + quad, 32 * FA_NG);
          if (hh == 0 && wr) {
            float4 t = cx[r];
#pragma unroll
            for (int g2 = 1; g2 < FA_NG; ++g2) {
              const float4 q = cx[g2 * 128 + r];
              t.x += q.x;
              t.y += q.y;
              t.z += q.z;
            }
            p.cos_part[static_cast<int64_t>(rp->orow) * p.H + it.h] = t;
          }
        } else if (wmask) {
          uint4 ch[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            float o[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) o[t] = acc[u * 8 + t] * oscale;
            ch[u] = pack8(o);
          }
          ev(55);
          store_rows(ch);
        }
      }
      ev(52);
      __syncwarp();
      if (lane == 0) mbar_arrive(&wq_empty[ii & 3]);
      cw = nw;
      ++ii;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&wq_empty[ii & 3]);  // the terminator's slot
  }
  ev.finish();
  __syncthreads();
  if (threadIdx.x == 0) {
    // the last CTA to finish re-arms the scheduler for the next launch (stream-ordered)
    __threadfence();
    if (atomicAdd(&p.work_ctr[1], 1) == static_cast<int>(gridDim.x) - 1) {
      p.work_ctr[0] = 0;
      p.work_ctr[1] = 0;
      if (p.mode == 1) p.fix[0] = 0;  // the fixup list is consumed
      __threadfence();
    }
  }
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, FA_TMEM_COLS);
  }
}

int attention_fused_launch(const AttnArgs &a, cudaStream_t st) {
  static DeviceOnce attr;
  if (attr.todo()) {
    DY_CUDA(cudaFuncSetAttribute(attn_fused_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, FA_SMEM));
    DY_CUDA(cudaFuncSetAttribute(attn_fused_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, FA_SMEM));
    attr.done();
  }
  const int rows_total = a.batch * a.N;
  const int qw = a.H * 128, kw = a.KVH * 128;
  CUtensorMap tq, tqx, tk, tv, tkx, tdv, tkxo, tkun, tkuo;
  int rc;
  if ((rc = make_tmap3(&tq, a.Q, rows_total, qw, 128, 2))) return rc;
  if ((rc = make_tmap3(&tqx, a.Qx ? a.Qx : a.Q, rows_total, qw, 128, 2))) return rc;
  if ((rc = make_tmap3(&tk, a.K, rows_total, kw, FA_BK, 2))) return rc;
  if ((rc = make_tmap3(&tv, a.V, rows_total, kw, FA_BK, 2))) return rc;
  if ((rc = make_tmap3(&tkx, a.Kx ? a.Kx : a.K, rows_total, kw, FA_BK, 2))) return rc;
  if ((rc = make_tmap3(&tdv, a.dV ? a.dV : a.V, rows_total, kw, FA_BK, 2))) return rc;
  if ((rc = make_tmap3(&tkxo, a.Kxo ? a.Kxo : a.K, rows_total, kw, FA_BK, 2))) return rc;
  const bool pinc = a.pinc && a.Kun && a.Kuo && a.ucnt && a.stats_cache && a.mode == 0;
  if ((rc = make_tmap3(&tkun, pinc ? a.Kun : a.K, rows_total, kw, FA_BK, 2))) return rc;
  if ((rc = make_tmap3(&tkuo, pinc ? a.Kuo : a.K, rows_total, kw, FA_BK, 2))) return rc;
  FaParams p;
  p.N = a.N;
  p.row_lo = a.row_lo;
  p.L = a.N - a.row_lo;
  p.H = a.H;
  p.KVH = a.KVH;
  p.grp = a.H / a.KVH;
  // row tiles: prompt tiles and response tiles never mix (their statistics are current up to
  // different key sets), so a full-input launch splits its rows at resp_lo
  const bool split = !a.full_only && a.row_lo < a.resp_lo && a.resp_lo < a.N;
  p.MTp = split ? (a.resp_lo - a.row_lo + 127) / 128 : 0;
  p.MT = a.full_only ? 0 : split ? p.MTp + (a.N - a.resp_lo + 127) / 128 : (p.L + 127) / 128;
  p.pinc = pinc ? 1 : 0;
  p.ucnt = a.ucnt;
  p.cos_part = a.full_only || a.mode == 2 ? nullptr : a.cos_part;
  p.XT = (a.max_rows_per_seq + 127) / 128;
  p.items = a.batch * a.H * (p.MT + p.XT);
  p.qw = qw;
  p.c = a.scale * 1.4426950408889634f;
  p.ex_off = a.ex_off;
  p.ex_rows = a.ex_rows;
  p.rowflag = a.rowflag;
  p.tag = a.row_tag;
  p.C_cache = a.C_cache;
  p.C_out = a.C_out;
  p.events = g_attn_events;
  p.work_ctr = a.work_ctr;
  p.stats = a.stats_cache;
  p.inc = a.inc && a.stats_cache && a.Kxo ? 1 : 0;
  p.resp_lo = a.resp_lo;
  p.mode = a.mode;
  p.fix = a.fix;
  p.fix_cap = a.fix_cap;
  p.t4max = g_attn_t4_rows;
  if (!p.fix) {
    set_error("fused attention: missing fixup list");
    return DYLLM_E_ARG;
  }
  if (!p.work_ctr) {
    set_error("fused attention: missing scheduler counters");
    return DYLLM_E_ARG;
  }
  if (p.items <= 0) return DYLLM_OK;
  // fixup launch: a few CTAs claim the (rare, device-counted) listed tiles
  const int grid = p.mode == 1 ? 16 : (p.items < a.num_sms ? p.items : a.num_sms);
  DY_CUDA(launch_k(p.cos_part ? attn_fused_kernel<true> : attn_fused_kernel<false>, dim3(grid), dim3(FA_THREADS),
                   FA_SMEM, st, 1, tq, tqx, tk, tv, tkx, tdv, tkxo, tkun, tkuo, p));
  DY_CUDA(cudaGetLastError());
  return DYLLM_OK;
}

}  // namespace dy
