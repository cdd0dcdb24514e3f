// hygt_gemm.cu -- per-class dense operators on the 5th-generation tensor cores (tcgen05).
//
// Serves two paths of SURVEY.md §8:
//   * a10, the KLT comparison: y = K_c x (klt_forward, statistics.hpp:222-224 -> multiply,
//     matrix.hpp:70-80) and x = K_c^T y (transposed, matrix.hpp:82-88);
//   * a1-a3 at N = 64 / 128 / 256, the HyGT itself as its COMPOSED operator: for a class c the
//     R rounds x log2N passes of Givens rotations (transform.hpp:45-66), the inter-round and
//     final gathers included, are one orthogonal N x N matrix M_c (transform.hpp:100-117
//     builds exactly this matrix column by column). The plan composes M_c once in fp64 from the
//     class's angles, and every row is then y = M_c x (forward) or x = M_c^T y (inverse).
//     At N = 256 the butterfly form needs 32 KB of rotation coefficients per row and direction
//     delivered through the shared-memory/L1 pipe (bound at 37% of HBM); the
//     composed form moves that work onto the tensor cores, whose operand reads bypass the LSU.
//
// Rows are bucketed by class (hygt_bucket). A tile is 128 rows of one class; per tile the
// kernel computes OUT[128 x N] = IN[128 x N] . B^T with B[n][k] (N x K, K-major), B = M_c or
// M_c^T (HyGT) / K_c or K_c^T (KLT).
//
// Precision (the fp32 bar of SURVEY.md c4: relative L2 <= 1e-6): fp16 operands with an exact
// 2-way split on both sides, x = x_hi + x_lo, b = b_hi + b_lo, and three MMAs
// lo.hi + hi.lo + hi.hi accumulated in fp32 in TMEM (the dropped lo.lo term is ~2^-22 relative).
// fp16 has 5 exponent bits, so every row is scaled by a power of two chosen from its own
// max |x| (max |x s| in [2^14, 2^15)) and every class operator by 2^kB (max |b 2^kB| in
// [2^14, 2^15)); both scales are exact and undone in the epilogue. The tensor cores round each
// K step's addition to the running fp32 sum, so per unit the two correction terms of ALL K are
// accumulated first and the main term after them: only its 4 KA K steps round against the
// full-size sum (as with separate accumulators, in half the TMEM).
//
// Kernel structure (one persistent CTA per SM, or a CTA pair per two SMs with tcgen05
// cta_group::2, warp-specialised, all hand-offs on mbarriers; 16 warps = 4 warpgroups whose
// registers are rebalanced with setmaxnreg):
//   warps 0-3   epilogue : TMEM -> registers (tcgen05.ld, lane = row) -> unscale -> swizzled
//                          staging -> coalesced STG rows; fused per-class energy (compensated
//                          fp32 per lane, fp64 at the class flush)
//   warps 4-11  split    : each lane holds its share of a whole tile in registers (one read of
//                          every row): row max -> power-of-two scale -> fp16 hi/lo into the
//                          tile's SWIZZLE_128B K-major A (64-column K atoms); the next tile's
//                          loads of an atom are issued as soon as the atom is converted
//   warp 12     producer : cp.async.bulk of the class's B half-atom stages (L2 resident)
//   warp 13     MMA      : one thread issues tcgen05.mma kind::f16 (M = 128 / 256, N <= 256, K = 16)
//   warp 14     prefetch : L2 prefetch of the rows two tiles ahead (prefetch.global.L2)
//   warp 15     idle     (completes the fourth warpgroup)
//   A tile is issued as NH units of NW output columns (wide: one unit of all N columns), each
//   into one of two TMEM accumulators, so the epilogue of one unit overlaps the next unit's MMAs.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hygt_gpu.h"
#include "hygt_gemm.h"

int hygt_set_error(int status, const char* msg);       // hygt_capi.cu
void hygt_smem_attr(const void* fn, size_t bytes);     // hygt_capi.cu

namespace hygt_gpu {
namespace {

constexpr int GM = 128;           // rows per tile (MMA M)
constexpr int EPI_WARPS = 4;
constexpr int SPLIT_WARPS = 8;
constexpr int PROD_WARP = EPI_WARPS + SPLIT_WARPS;
constexpr int MMA_WARP = PROD_WARP + 1;
constexpr int PF_WARP = MMA_WARP + 1;
constexpr int GEMM_THREADS = (PF_WARP + 2) * 32;  // + one idle warp: four whole warpgroups
// Register rebalancing (setmaxnreg, per warpgroup): 128 per thread at launch (64 K / 512);
// the split warpgroups take what the epilogue and the single-thread roles give back, so that
// a split lane holds its whole share of a tile (up to 128 floats at N = 256).
constexpr int REG_EPI = 128, REG_SPLIT = 160, REG_MISC = 64;
static_assert(REG_EPI + 2 * REG_SPLIT + REG_MISC <= 512, "register pool");
template <int R> __device__ __forceinline__ void regs_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" :: "n"(R)); }
template <int R> __device__ __forceinline__ void regs_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" :: "n"(R)); }
constexpr uint32_t ATOM_BYTES = GM * 128;  // one 64-column fp16 K atom of the A tile (16 KB)

template <int NN, bool PAIR, bool WIDE>
struct Shape {
  static constexpr int KA = NN / 64;                 // K atoms (64 fp16 = one 128 B swizzle row)
  // columns per MMA instruction = per unit: up to 128, or (WIDE, CTA pairs) all N = 256 in one
  // unit, which halves the shared-memory reads of A per tile
  static constexpr int NW = WIDE ? NN : (NN < 128 ? NN : 128);
  static constexpr int NH = NN / NW;                 // units per tile
  static constexpr int BW = PAIR ? NW / 2 : NW;      // B rows (output columns) held by this CTA
  // B stage: one half (hi or lo) of one K atom of one unit (this CTA's BW rows), streamed in
  // the MMA order (per unit: per atom hi, lo for the correction terms, then hi again for the
  // main term): SPT stages per tile
  static constexpr uint32_t STAGE = (uint32_t)BW * 128;
  // N = 256: the epilogue stores straight from tcgen05.ld.16x256b fragments (no staging), which
  // leaves room for a fifth B stage; N <= 128 stages through shared memory (faster there)
  static constexpr bool DIRECT = NN == 256;
  // BRES (one N = 256 unit per tile): the B hi halves of the class stay resident across its
  // tiles (reloaded when the class changes) and only the lo halves stream through the ring
  static constexpr bool BRES = WIDE && NN == 256;
  static constexpr int NB = BRES ? 2 : (STAGE <= 8192 ? 8 : (DIRECT ? 5 : 4));  // B ring stages
  static constexpr int SPT = BRES ? KA : 3 * KA * NH;  // ring stages per tile
  // N <= 128: two 128-row sub-tiles per CTA and tile share every B stage and hand-off, which
  // halves the per-row cost of the pipeline's synchronisation
  static constexpr int SUB = NN <= 128 ? 2 : 1;
  static constexpr int CR = SUB * GM;                 // rows per CTA and tile
  static constexpr int TG = PAIR ? 2 * CR : CR;      // rows per tile (a CTA pair: CR each)
  static constexpr int ABUF = KA * SUB <= 2 ? 2 : 1;  // tiles of A resident (double-buffered if small)
  static constexpr int AS = KA * SUB * ABUF;         // A atom slots (128 rows each)
  static constexpr uint32_t A_OFF = 0;               // A: AS atoms (hi + lo each)
  static constexpr uint32_t BR_OFF = A_OFF + AS * 2 * ATOM_BYTES;          // BRES: KA resident B hi stages
  static constexpr uint32_t B_OFF = BR_OFF + (BRES ? KA * STAGE : 0u);
  static constexpr uint32_t STG_OFF = B_OFF + NB * STAGE;
  static constexpr uint32_t STG_BYTES = DIRECT ? 0 : 32 * 128;  // per epilogue warp: 32 rows x 32 floats (swizzled)
  static constexpr uint32_t FAC_OFF = STG_OFF + EPI_WARPS * STG_BYTES;
  static constexpr int FB = BRES ? 2 : 4;            // row-factor buffers (tiles in flight split -> epilogue)
  static constexpr uint32_t BAR_OFF = FAC_OFF + FB * CR * 4;
  static constexpr uint32_t TE_OFF = BAR_OFF + 512;  // barriers (<= 62 x 8 B) + the TMEM address
  // + [C] u32 per-class cumulative tile counts (tile_end)
  static constexpr uint32_t smem(int classes) { return TE_OFF + 4u * (uint32_t)classes; }
  // TMEM: one fp32 accumulator of NW columns per unit, double-buffered over units
  static constexpr int NBUF = 2;
  static constexpr int ACC = SUB * NW;                // sub-tile s at column s NW
  static constexpr uint32_t TMEM_COLS = NBUF * ACC < 32 ? 32 : NBUF * ACC;
  static constexpr int RG = CR / SPLIT_WARPS / 4;    // 4-row groups per split warp
  static_assert(!WIDE || PAIR || NN <= 128, "N = 256 in one unit needs the CTA pair");
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" :: "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes) : "memory");
}
// CTA-scope acquire, also for the barriers the peer CTA arrives on: what crosses CTAs is
// shared-memory data read by the tensor cores (ordered by fence.proxy.async before the
// arrival) and TMEM (ordered by the tcgen05 fences); a cluster-scope acquire would invalidate
// L1 (CCTL.IVALL) on every wait
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n\tW%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W%=;\n\t}\n"
      :: "r"(smem_u32(b)), "r"(parity) : "memory");
}
// arrive on the barrier at the same offset in CTA `cta` of the cluster (default semantics:
// a cluster-scope release would drain every outstanding global access first)
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* b, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}\n"
      :: "r"(smem_u32(b)), "r"(cta) : "memory");
}
// cluster-scope release / acquire: for data a thread of the other CTA reads with generic
// (DSMEM) loads or TMEM written with tcgen05.st that the peer's MMAs read; used where the
// releasing thread has no global accesses in flight (a release at cluster scope waits for them)
__device__ __forceinline__ void mbar_arrive_remote_release(uint64_t* b, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}\n"
      :: "r"(smem_u32(b)), "r"(cta) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n\tW%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n\t@!P bra W%=;\n\t}\n"
      :: "r"(smem_u32(b)), "r"(parity) : "memory");
}
template <bool PAIR>
__device__ __forceinline__ void tc_commit(uint64_t* b) {
  if constexpr (PAIR)  // the pair's MMAs done: arrive on the barrier in both CTAs
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 :: "r"(smem_u32(b)), "h"((uint16_t)3) : "memory");
  else
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(b)) : "memory");
}
// one tcgen05.mma kind::f16 (M = 128, or 256 over the CTA pair), fp32 accumulate unless acc == 0
template <bool PAIR, int NW>
__device__ __forceinline__ void mma_issue(uint32_t d, uint64_t a, uint64_t b, uint32_t acc);
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id() {
  uint32_t r;
  asm("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_count() {
  uint32_t r;
  asm("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// SWIZZLE_128B K-major UMMA shared-memory descriptor: 8-row x 128 B atoms, 1024 B apart (SBO).
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;            // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;  // SBO
  d |= (uint64_t)1 << 46;            // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;            // SWIZZLE_128B
  return d;
}
// Instruction descriptor: D f32, A/B f16, both K-major, M = m, N = n.
__host__ __device__ constexpr uint32_t idesc_f16(int n, int m = GM) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
template <bool PAIR, int NW>
__device__ __forceinline__ void mma_issue(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  if constexpr (PAIR)  // M = 256: A rows and B columns from both CTAs
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
        :: "r"(d), "l"(a), "l"(b), "r"(idesc_f16(NW, 2 * GM)), "r"(acc));
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
        :: "r"(d), "l"(a), "l"(b), "r"(idesc_f16(NW)), "r"(acc));
}
// One lane of a converged warp (elect.sync). The MMA issuer runs as a whole warp and issues
// from the elected lane: the descriptors then stay in uniform registers and every
// tcgen05.mma is one UTCHMMA, where a lone lane in a divergent branch pays R2UR moves and an
// ELECT loop per instruction (~15 SASS instructions per MMA, which next to the split warps'
// ALU stream limited the N = 256 MMAs to ~280 cycles each instead of 128; tools/microbench_contend.cu)
__device__ __forceinline__ bool elect_one() {
  uint32_t e;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(e));
  return e != 0;
}
// The 4 K steps (16 fp16 = 32 B each: +2 in the descriptors' 16 B address field) of one 64-wide
// K atom, M = 256 over the CTA pair, N = NW: correction terms lo.hi and hi.lo interleaved per K
// step (the first accumulates unless acc0 == 0), or the main term hi.hi alone.
template <int NW>
__device__ __forceinline__ void mma_atom_corr2(uint32_t d, uint64_t alo, uint64_t bhi, uint64_t ahi, uint64_t blo, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 a0, b0, a1, b1;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "mov.b64 a0, %1;\n\tmov.b64 b0, %2;\n\tmov.b64 a1, %3;\n\tmov.b64 b1, %4;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], a0, b0, %6, p;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %6, 1;\n\t"
      "add.s64 a0, a0, 2;\n\tadd.s64 b0, b0, 2;\n\tadd.s64 a1, a1, 2;\n\tadd.s64 b1, b1, 2;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], a0, b0, %6, 1;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %6, 1;\n\t"
      "add.s64 a0, a0, 2;\n\tadd.s64 b0, b0, 2;\n\tadd.s64 a1, a1, 2;\n\tadd.s64 b1, b1, 2;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], a0, b0, %6, 1;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %6, 1;\n\t"
      "add.s64 a0, a0, 2;\n\tadd.s64 b0, b0, 2;\n\tadd.s64 a1, a1, 2;\n\tadd.s64 b1, b1, 2;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], a0, b0, %6, 1;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %6, 1;\n\t}\n"
      :: "r"(d), "l"(alo), "l"(bhi), "l"(ahi), "l"(blo), "r"(acc0), "n"(idesc_f16(NW, 2 * GM)));
}
template <int NW>
__device__ __forceinline__ void mma_atom_main2(uint32_t d, uint64_t ahi, uint64_t bhi) {
  asm volatile(
      "{\n\t.reg .b64 a0, b0;\n\t"
      "mov.b64 a0, %1;\n\tmov.b64 b0, %2;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], a0, b0, %3, 1;\n\t"
      "add.s64 a0, a0, 2;\n\tadd.s64 b0, b0, 2;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], a0, b0, %3, 1;\n\t"
      "add.s64 a0, a0, 2;\n\tadd.s64 b0, b0, 2;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], a0, b0, %3, 1;\n\t"
      "add.s64 a0, a0, 2;\n\tadd.s64 b0, b0, 2;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], a0, b0, %3, 1;\n\t}\n"
      :: "r"(d), "l"(ahi), "l"(bhi), "n"(idesc_f16(NW, 2 * GM)));
}
// swizzled byte offset of 16 B chunk q of row r inside an SW128 atom
__device__ __forceinline__ uint32_t swz(int r, int q) { return (uint32_t)r * 128u + (uint32_t)((q ^ (r & 7)) << 4); }

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float2 unpack_h2(uint32_t u) {
  __half2 h = *reinterpret_cast<__half2*>(&u);
  return __half22float2(h);
}

// Per-row power-of-two scale: max |x s| in [2^14, 2^15) (fp16 max is 65504). Zero rows get 1.
__device__ __forceinline__ float row_scale(float mx) {
  const uint32_t e = __float_as_uint(mx) >> 23;  // biased exponent of max |x|
  if (mx == 0.f) return 1.f;
  int f = 268 - (int)e;                          // 127 + 14 - (e - 127)
  f = f < 1 ? 1 : (f > 254 ? 254 : f);
  return __uint_as_float((uint32_t)f << 23);
}

// end of bucket c (bucket `classes` holds invalid ids); without buckets (one class, no ids) the
// rows are in order: bucket 0 = [0, count)
__device__ __forceinline__ uint64_t seg_at(const GemmParams& P, int c) {
  return P.seg_end ? (uint64_t)__ldg(P.seg_end + c) : (c >= 0 ? P.count : 0ull);
}
__device__ __forceinline__ uint32_t row_at(const GemmParams& P, uint64_t p) {
  return P.idx ? __ldg(P.idx + p) : (uint32_t)p;
}

// tile -> (class, first bucketed position, rows) of this CTA's part of the tile: a tile is TG
// rows of one class; in the CTA-pair variant rank 0 takes its first 128 rows, rank 1 the rest
struct TileMap {
  const uint32_t* tile_end;  // shared: [C] cumulative tile counts
  const GemmParams* P;
  int classes;
  uint32_t tg, part, cr;     // rows per tile, this CTA's offset in the tile (0 or CR), rows per CTA
  const uint32_t* seg_sh = nullptr;  // shared copy of the bucket ends [C] (or nullptr: global seg_end)
  __device__ void of(uint32_t t, int& c, uint64_t& p0, uint32_t& rows) const {
    int lo = 0, hi = classes - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (tile_end[mid] <= t) lo = mid + 1; else hi = mid;
    }
    c = lo;
    const uint32_t first_tile = c ? tile_end[c - 1] : 0u;
    const uint64_t s0 = c ? (seg_sh ? (uint64_t)seg_sh[c - 1] : seg_at(*P, c - 1)) : 0ull;
    const uint64_t s1 = seg_sh ? (uint64_t)seg_sh[c] : seg_at(*P, c);
    p0 = s0 + (uint64_t)(t - first_tile) * tg + part;
    const uint64_t left = s1 > p0 ? s1 - p0 : 0ull;
    rows = left < cr ? (uint32_t)left : cr;
  }
};

// debug trace (hygt_debug_gemm_trace): clock64 of per-tile pipeline events in CTA 0
#define GEMM_TRACE(k, e)                                                   \
  do {                                                                     \
    if (P.trace && blockIdx.x == 0 && (k) < 64) P.trace[(k) * 16 + (e)] = clock64(); \
  } while (0)

template <int NN, bool ENERGY, bool PAIR, bool WIDE>
__global__ void __launch_bounds__(GEMM_THREADS, 1) hygt_gemm_kernel(const GemmParams P) {
  using SH = Shape<NN, PAIR, WIDE>;
  // 1024 B aligned (SWIZZLE_128B atoms); declared shared so every access compiles to LDS/STS
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + SH::BAR_OFF);
  uint64_t* a_full = bars;                     // [AS]  atom written, count SPLIT_WARPS
  uint64_t* a_empty = a_full + SH::AS;         // [AS]  atom read by the tile's last unit (commit)
  uint64_t* b_full = a_empty + SH::AS;         // [NB]  expect_tx
  uint64_t* b_empty = b_full + SH::NB;         // [NB]  tcgen05.commit
  uint64_t* d_full = b_empty + SH::NB;         // [2]   tcgen05.commit
  uint64_t* d_empty = d_full + 2;              // [2]   count EPI_WARPS
  uint64_t* f_full = d_empty + 2;              // [4]   row scales written, count SPLIT_WARPS
  uint64_t* f_empty = f_full + 4;              // [4]   row scales read, count EPI_WARPS
  uint64_t* b_peer = f_empty + 4;              // [NB]  pair: the peer's B half landed (count 1)
  uint64_t* bh_full = b_peer + SH::NB;         // [1]   BRES: the class's resident B hi halves landed (expect_tx)
  uint64_t* bh_empty = bh_full + 1;            // [1]   BRES: the class's last MMAs done (commit)
  uint64_t* bh_peer = bh_empty + 1;            // [1]   BRES, pair: the peer's resident B hi landed
  uint32_t* tmem_sh = reinterpret_cast<uint32_t*>(bh_peer + 1);
  static_assert(SH::AS * 2 + SH::NB * 3 + 15 <= 62, "barrier area");
  static_assert(SH::SUB == 1 || !SH::BRES, "sub-tiles only without resident B");
  uint32_t* tile_end_sh = reinterpret_cast<uint32_t*>(sm + SH::TE_OFF);  // [C]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int C = P.classes;
  // CTA pair (cluster of 2, tcgen05 cta_group::2): rank 0 issues the MMAs of both; every
  // hand-off the MMA issuer waits for is counted on rank 0's barriers, every completion it
  // signals is multicast to both CTAs
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  const uint32_t t_first = PAIR ? cluster_id() : blockIdx.x;
  const uint32_t t_step = PAIR ? cluster_count() : gridDim.x;
  const uint32_t pn = PAIR ? 2u : 1u;  // arrivals per hand-off counted on rank 0
  // per-class cumulative tile counts
  if (warp == 0) {
    uint32_t run = 0;
    for (int c0 = 0; c0 < C; c0 += 32) {
      const int c = c0 + lane;
      uint32_t nt = 0;
      if (c < C) {
        const uint64_t s0 = c ? seg_at(P, c - 1) : 0ull;
        const uint64_t s1 = seg_at(P, c);
        nt = (uint32_t)((s1 - s0 + SH::TG - 1) / SH::TG);
      }
      uint32_t v = nt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (c < C) tile_end_sh[c] = run + v;
      run += __shfl_sync(0xffffffffu, v, 31);
    }
  }
  if (warp == MMA_WARP) {  // in the pair variant both CTAs allocate, with the same warp
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                   :: "r"(smem_u32(tmem_sh)), "r"(SH::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                   :: "r"(smem_u32(tmem_sh)), "r"(SH::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  if (tid == 0) {
    for (int i = 0; i < SH::AS; ++i) { mbar_init(&a_full[i], SPLIT_WARPS * pn); mbar_init(&a_empty[i], 1); }
    for (int i = 0; i < SH::NB; ++i) { mbar_init(&b_full[i], 1); mbar_init(&b_empty[i], 1); mbar_init(&b_peer[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&d_full[i], 1); mbar_init(&d_empty[i], EPI_WARPS * pn); }
    for (int i = 0; i < 4; ++i) { mbar_init(&f_full[i], SPLIT_WARPS); mbar_init(&f_empty[i], EPI_WARPS); }
    mbar_init(bh_full, 1);
    mbar_init(bh_empty, 1);
    mbar_init(bh_peer, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if constexpr (PAIR) cluster_sync(); else __syncthreads();  // barriers initialised in both CTAs
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_sh;
  const TileMap tm{tile_end_sh, &P, C, (uint32_t)SH::TG, rank * (uint32_t)SH::CR, (uint32_t)SH::CR};
  const uint32_t ntiles = C ? tile_end_sh[C - 1] : 0u;
  float* fac = reinterpret_cast<float*>(sm + SH::FAC_OFF);  // [FB][CR] per-row unscale factors
  auto class_of = [&](uint32_t t) {
    int lo = 0, hi = C - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (tile_end_sh[mid] <= t) lo = mid + 1; else hi = mid;
    }
    return lo;
  };

  if (warp == MMA_WARP) {
    // ------------------------------------------------------------------ MMA issuer ----
    regs_dec<REG_MISC>();
    // Per tile, NH units of NW output columns in order, unit u into TMEM buffer u & 1. Per
    // unit the correction terms of all K first (per K atom: lo.hi with the B hi stage, hi.lo
    // with the B lo stage), then the main term hi.hi (B hi again): only the 4 KA main-term K
    // steps round against the full-size sum (the tensor cores round each K step's addition).
    if (PAIR && rank == 1) {
      // the peer forwards "my B half landed" for each stage to rank 0's issuer
      if (lane == 0) {
        uint32_t ib = 0, nload = 0;
        int cur = -1;
        for (uint32_t t = t_first; t < ntiles; t += t_step) {
          if constexpr (SH::BRES) {  // the class's resident B hi halves, once per class change
            const int c = class_of(t);
            if (c != cur) {
              mbar_wait(bh_full, nload & 1);
              mbar_arrive_remote(bh_peer, 0);
              ++nload;
              cur = c;
            }
          }
          for (int s = 0; s < SH::SPT; ++s, ++ib) {
            if ((P.dbg & 1) && ib >= (uint32_t)SH::NB) break;
            const int sb = (int)(ib % SH::NB);
            mbar_wait(&b_full[sb], (ib / SH::NB) & 1);
            mbar_arrive_remote(&b_peer[sb], 0);
          }
        }
      }
    } else if (SH::BRES && PAIR && !(P.dbg & 4)) {
      // One N = 256 unit per tile, issued by the whole (converged) warp from one elected lane
      // (see elect_one). Correction terms (per atom: lo.hi with the resident B hi, hi.lo with
      // the streamed B lo), then the main term hi.hi (resident B hi).
      const bool leader = elect_one();
      uint32_t il = 0, k = 0, nload = 0;
      int cur = -1;
      for (uint32_t t = t_first; t < ntiles; t += t_step, ++k) {
        const int c = class_of(t);
        if (c != cur) {  // the producer loaded this class's B hi halves (one load per change)
          mbar_wait(bh_full, nload & 1);
          mbar_wait(bh_peer, nload & 1);
          ++nload;
          cur = c;
        }
        const int db = (int)(k & 1);
        if (k >= 2) mbar_wait(&d_empty[db], ((k >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (leader) GEMM_TRACE(k, 3);
        const uint32_t dacc = tmem + (uint32_t)(db * SH::ACC);
#pragma unroll 1
        for (int ka = 0; ka < SH::KA; ++ka, ++il) {  // correction terms
          mbar_wait(&a_full[ka], k & 1);
          const int sb = (int)(il % SH::NB);
          const bool b_streamed = !(P.dbg & 1) || il < (uint32_t)SH::NB;  // diagnostic 1: loaded once
          if (b_streamed) {
            mbar_wait(&b_full[sb], (il / SH::NB) & 1);
            mbar_wait(&b_peer[sb], (il / SH::NB) & 1);
          }
          asm volatile("tcgen05.fence::after_thread_sync;");
          __syncwarp();
          if (leader) {
            if (ka < 2) GEMM_TRACE(k, 8 + ka);
            const uint64_t ahi = desc_sw128(smem_u32(sm + SH::A_OFF + (uint32_t)ka * 2 * ATOM_BYTES));
            const uint64_t alo = ahi + (ATOM_BYTES >> 4);
            const uint64_t bhi = desc_sw128(smem_u32(sm + SH::BR_OFF + (uint32_t)ka * SH::STAGE));
            const uint64_t blo = desc_sw128(smem_u32(sm + SH::B_OFF + (uint32_t)sb * SH::STAGE));
            mma_atom_corr2<SH::NW>(dacc, alo, bhi, ahi, blo, (uint32_t)ka);
            if (!(P.dbg & 1)) tc_commit<PAIR>(&b_empty[sb]);
          }
          __syncwarp();
        }
#pragma unroll 1
        for (int ka = 0; ka < SH::KA; ++ka) {  // main term
          if (leader) {
            if (ka < 2) GEMM_TRACE(k, 10 + ka);
            const uint64_t ahi = desc_sw128(smem_u32(sm + SH::A_OFF + (uint32_t)ka * 2 * ATOM_BYTES));
            const uint64_t bhi = desc_sw128(smem_u32(sm + SH::BR_OFF + (uint32_t)ka * SH::STAGE));
            mma_atom_main2<SH::NW>(dacc, ahi, bhi);
            tc_commit<PAIR>(&a_empty[ka]);  // the atom may take the next tile's
          }
          __syncwarp();
        }
        // the class's last tile here: its B hi halves may be replaced once these MMAs are done
        const uint32_t tn = t + t_step;
        const bool last_of_class = tn >= ntiles || class_of(tn) != c;
        if (leader) {
          tc_commit<PAIR>(&d_full[db]);
          if (last_of_class) tc_commit<PAIR>(bh_empty);
          GEMM_TRACE(k, 4);
        }
        __syncwarp();
      }
    } else if (SH::BRES && lane == 0) {
      // One N = 256 unit per tile. Correction terms (per atom: lo.hi with the resident B hi,
      // hi.lo with the streamed B lo), then the main term hi.hi (resident B hi).
      uint32_t il = 0, k = 0, nload = 0;
      int cur = -1;
      for (uint32_t t = t_first; t < ntiles; t += t_step, ++k) {
        const int c = class_of(t);
        if (c != cur) {  // the producer loaded this class's B hi halves (one load per change)
          mbar_wait(bh_full, nload & 1);
          if constexpr (PAIR) mbar_wait(bh_peer, nload & 1);
          ++nload;
          cur = c;
        }
        const int db = (int)(k & 1);
        if (k >= 2) mbar_wait(&d_empty[db], ((k >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        GEMM_TRACE(k, 3);
        const uint32_t dacc = tmem + (uint32_t)(db * SH::ACC);
#pragma unroll 1
        for (int ka = 0; ka < SH::KA; ++ka, ++il) {  // correction terms
          mbar_wait(&a_full[ka], k & 1);
          const int sb = (int)(il % SH::NB);
          mbar_wait(&b_full[sb], (il / SH::NB) & 1);
          if constexpr (PAIR) mbar_wait(&b_peer[sb], (il / SH::NB) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          if (ka < 2) GEMM_TRACE(k, 8 + ka);
          const uint64_t ahi = desc_sw128(smem_u32(sm + SH::A_OFF + (uint32_t)ka * 2 * ATOM_BYTES));
          const uint64_t alo = ahi + (ATOM_BYTES >> 4);
          const uint64_t bhi = desc_sw128(smem_u32(sm + SH::BR_OFF + (uint32_t)ka * SH::STAGE));
          const uint64_t blo = desc_sw128(smem_u32(sm + SH::B_OFF + (uint32_t)sb * SH::STAGE));
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint64_t o = 2u * j;
            mma_issue<PAIR, SH::NW>(dacc, alo + o, bhi + o, (ka | j) ? 1u : 0u);
            mma_issue<PAIR, SH::NW>(dacc, ahi + o, blo + o, 1u);
          }
          tc_commit<PAIR>(&b_empty[sb]);
        }
#pragma unroll 1
        for (int ka = 0; ka < SH::KA; ++ka) {  // main term
          if (ka < 2) GEMM_TRACE(k, 10 + ka);
          const uint64_t ahi = desc_sw128(smem_u32(sm + SH::A_OFF + (uint32_t)ka * 2 * ATOM_BYTES));
          const uint64_t bhi = desc_sw128(smem_u32(sm + SH::BR_OFF + (uint32_t)ka * SH::STAGE));
#pragma unroll
          for (int j = 0; j < 4; ++j) mma_issue<PAIR, SH::NW>(dacc, ahi + 2u * j, bhi + 2u * j, 1u);
          tc_commit<PAIR>(&a_empty[ka]);  // the atom may take the next tile's
        }
        tc_commit<PAIR>(&d_full[db]);
        // the class's last tile here: its B hi halves may be replaced once these MMAs are done
        const uint32_t tn = t + t_step;
        if (tn >= ntiles || class_of(tn) != c) tc_commit<PAIR>(bh_empty);
        GEMM_TRACE(k, 4);
      }
    } else if (!SH::BRES && lane == 0) {
      uint32_t ib = 0, u = 0, k = 0;
      auto wait_stage = [&](uint32_t i) {
        const int sb = (int)(i % SH::NB);
        if (!(P.dbg & 1) || i < (uint32_t)SH::NB) {
          mbar_wait(&b_full[sb], (i / SH::NB) & 1);
          if constexpr (PAIR) mbar_wait(&b_peer[sb], (i / SH::NB) & 1);
        }
        return desc_sw128(smem_u32(sm + SH::B_OFF + (uint32_t)sb * SH::STAGE));
      };
      auto release_stage = [&](uint32_t i) {
        if (!(P.dbg & 1)) tc_commit<PAIR>(&b_empty[i % SH::NB]);
      };
      auto mma = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
        if constexpr (PAIR)  // M = 256: A rows and B columns from both CTAs
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
              :: "r"(d), "l"(a), "l"(b), "r"(idesc_f16(SH::NW, 2 * GM)), "r"(acc));
        else
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
              :: "r"(d), "l"(a), "l"(b), "r"(idesc_f16(SH::NW)), "r"(acc));
      };
      for (uint32_t t = t_first; t < ntiles; t += t_step, ++k) {
        for (int nh = 0; nh < SH::NH; ++nh, ++u) {
          const int db = (int)(u & 1);
          if (u >= 2) mbar_wait(&d_empty[db], ((u >> 1) - 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          if (nh == 0) GEMM_TRACE(k, 3);
          const uint32_t dacc = tmem + (uint32_t)(db * SH::ACC);
          // A atom slot of sub-tile sb, K atom ka; sub-tile sb accumulates at column sb NW
          auto slot = [&](int sb, int ka) { return ((int)(k % SH::ABUF) * SH::SUB + sb) * SH::KA + ka; };
#pragma unroll 1
          for (int ka = 0; ka < SH::KA; ++ka, ib += 2) {  // correction terms
            if (nh == 0)
#pragma unroll
              for (int sb = 0; sb < SH::SUB; ++sb) mbar_wait(&a_full[slot(sb, ka)], (k / SH::ABUF) & 1);
            const uint64_t bhi = wait_stage(ib), blo = wait_stage(ib + 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            if (nh < 2 && ka < 2) GEMM_TRACE(k, 8 + nh * 4 + ka);
#pragma unroll
            for (int sb = 0; sb < SH::SUB; ++sb) {
              // descriptors of the atom's / stage's first K step; the next K step (32 B further)
              // is +2 in the 16 B-unit start-address field (no carry: addresses < 2^18)
              const uint64_t ahi = desc_sw128(smem_u32(sm + SH::A_OFF + (uint32_t)slot(sb, ka) * 2 * ATOM_BYTES));
              const uint64_t alo = ahi + (ATOM_BYTES >> 4);
              const uint32_t d = dacc + (uint32_t)(sb * SH::NW);
#pragma unroll
              for (int j = 0; j < 4; ++j) {  // K = 16 fp16 = 32 B per instruction
                const uint64_t o = 2u * j;
                mma(d, alo + o, bhi + o, (ka | j) ? 1u : 0u);
                mma(d, ahi + o, blo + o, 1u);
              }
            }
            release_stage(ib);
            release_stage(ib + 1);
          }
#pragma unroll 1
          for (int ka = 0; ka < SH::KA; ++ka, ++ib) {  // main term
            const uint64_t bhi = wait_stage(ib);
            asm volatile("tcgen05.fence::after_thread_sync;");
            if (nh < 2 && ka < 2) GEMM_TRACE(k, 10 + nh * 4 + ka);
#pragma unroll
            for (int sb = 0; sb < SH::SUB; ++sb) {
              const uint64_t ahi = desc_sw128(smem_u32(sm + SH::A_OFF + (uint32_t)slot(sb, ka) * 2 * ATOM_BYTES));
              const uint32_t d = dacc + (uint32_t)(sb * SH::NW);
#pragma unroll
              for (int j = 0; j < 4; ++j) mma(d, ahi + 2u * j, bhi + 2u * j, 1u);
            }
            release_stage(ib);
            if (nh == SH::NH - 1)
#pragma unroll
              for (int sb = 0; sb < SH::SUB; ++sb) tc_commit<PAIR>(&a_empty[slot(sb, ka)]);  // may take a later tile's atom
          }
          tc_commit<PAIR>(&d_full[db]);
        }
        GEMM_TRACE(k, 4);
      }
    }
  } else if (warp == PF_WARP) {
    // ------------------------------------------------------------------ row prefetch --
    regs_dec<REG_MISC>();
    // L2 prefetch (prefetch.global.L2, per 128 B line: the LSU path, so the B stage copies in
    // the bulk-copy engine never queue behind this HBM traffic) of the rows of the tile
    // PF_AHEAD steps ahead, paced by the split warps' progress (f_full: row maxima of tile k
    // done), so the split's loads hit L2.
    constexpr int PF_AHEAD = 2;
    auto prefetch_rows = [&](uint32_t tp) {
      if (tp >= ntiles) return;
      int c;
      uint64_t p0;
      uint32_t rows;
      tm.of(tp, c, p0, rows);
      uint32_t id[SH::CR / 32];
#pragma unroll
      for (int i = 0; i < SH::CR / 32; ++i) {
        const uint32_t r = (uint32_t)(lane + 32 * i);
        id[i] = r < rows ? row_at(P, p0 + r) : 0xffffffffu;
      }
#pragma unroll
      for (int i = 0; i < SH::CR / 32; ++i)
        if (id[i] != 0xffffffffu)
#pragma unroll
          for (int l = 0; l < NN / 32; ++l)
            asm volatile("prefetch.global.L2 [%0];" :: "l"(P.x + (size_t)id[i] * NN + l * 32) : "memory");
    };
    if (!(P.dbg & 2)) {
    for (int a = 0; a < PF_AHEAD; ++a) prefetch_rows(t_first + (uint32_t)a * t_step);
    uint32_t k = 0;
    for (uint32_t t = t_first + PF_AHEAD * t_step; t < ntiles; t += t_step, ++k) {
      mbar_wait(&f_full[k % SH::FB], (k / SH::FB) & 1);
      prefetch_rows(t);
    }
    }
  } else if (warp == PROD_WARP) {
    // ------------------------------------------------------------------ B producer ----
    regs_dec<REG_MISC>();
    // Lane 0: the B stages of each unit of each tile, in the MMA's order, into the NB-stage
    // ring.
    if (lane == 0) {
      // global stages: [class][K atom][128-column half][hi | lo] (gemm_build)
      constexpr uint32_t GSTAGE = 2u * (NN < 128 ? NN : 128) * 128, PART = (uint32_t)SH::BW * 128;
      constexpr int GH = NN < 128 ? 1 : NN / 128;
      uint32_t ib = 0, nload = 0;
      int cur = -1;
      for (uint32_t t = t_first; t < ntiles; t += t_step) {
        int c;
        uint64_t p0;
        uint32_t rows;
        tm.of(t, c, p0, rows);
        const unsigned char* src = P.bops + (size_t)c * SH::KA * GH * GSTAGE;
        if constexpr (SH::BRES) {  // class change: the resident B hi halves of this CTA's rows
          if (c != cur) {
            if (nload > 0) mbar_wait(bh_empty, (nload - 1) & 1);  // the previous class's MMAs are done
            mbar_expect_tx(bh_full, SH::KA * SH::STAGE);
            for (int ka = 0; ka < SH::KA; ++ka)
              asm volatile(
                  "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                  :: "r"(smem_u32(sm + SH::BR_OFF + (uint32_t)ka * SH::STAGE)), "l"(src + (size_t)(ka * GH + rank) * GSTAGE),
                     "r"(SH::STAGE), "r"(smem_u32(bh_full)) : "memory");
            ++nload;
            cur = c;
          }
        }
        for (int s = 0; s < SH::SPT; ++s, ++ib) {
            if ((P.dbg & 1) && ib >= (uint32_t)SH::NB) break;
            const int sb = (int)(ib % SH::NB);
            if (ib >= (uint32_t)SH::NB) mbar_wait(&b_empty[sb], ((ib / SH::NB) - 1) & 1);
            mbar_expect_tx(&b_full[sb], SH::STAGE);
            const uint32_t d = smem_u32(sm + SH::B_OFF + (uint32_t)sb * SH::STAGE);
            // stage s of the tile: unit nh; per unit atom r / 2 hi / lo (r < 2 KA), then atom
            // r - 2 KA hi. The unit's B rows of this CTA: with one N = 256 unit per tile and CTA
            // pairs, global half `rank` (all its 128 rows); otherwise global half nh, rows from
            // rank * BW (the layout cta_group::2 expects)
            const int nh = SH::BRES ? 0 : s / (3 * SH::KA), r = s % (3 * SH::KA);
            const int ka = SH::BRES ? s : (r < 2 * SH::KA ? r >> 1 : r - 2 * SH::KA);
            const int part = SH::BRES ? 1 : (r < 2 * SH::KA ? (r & 1) : 0);  // BRES streams the lo halves
            const int gh = (WIDE && NN == 256) ? (int)rank : nh;
            const uint32_t roff = (WIDE && NN == 256) ? 0u : rank * PART;
            const unsigned char* g = src + (size_t)(ka * GH + gh) * GSTAGE + (size_t)part * (GSTAGE / 2) + roff;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                :: "r"(d), "l"(g), "r"(SH::STAGE), "r"(smem_u32(&b_full[sb])) : "memory");
          }
      }
    }
  } else if (warp > PF_WARP) {
    // idle (completes the fourth warpgroup for the register rebalancing)
    regs_dec<REG_MISC>();
  } else if (warp >= EPI_WARPS) {
    // ------------------------------------------------------------------ split warps ---
    regs_inc<REG_SPLIT>();
    const int sw = warp - EPI_WARPS;
    const int g8 = lane >> 3, l8 = lane & 7;  // row within a 4-row group, lane within the row
    // Rows of 4-row group g: one 64-bit store instruction writes 64 B of each of its 4 rows
    // and is served in two 16-lane phases. Rows {0, 4} (lanes 0-15) and {1, 5} (lanes 16-31)
    // of an 8-row block fall in opposite halves of the SWIZZLE_128B pattern, so each phase
    // covers all 32 banks once: 2 wavefronts per instruction, the minimum.
    // (with two sub-tiles, groups 4..7 are the same rows of the second 128-row sub-tile, so
    // every split warp writes into every A atom slot)
    auto row_of_group = [&](int g) {
      const int gb = g & 3, sub = g >> 2;
      const int b16 = (sw * 4 + gb) >> 2, gg = (sw * 4 + gb) & 3;
      return sub * GM + b16 * 16 + (gg & 1) * 2 + (gg >> 1) * 8 + (g8 >> 1) + (g8 & 1) * 4;
    };
    // One pass per tile: each lane holds its 4 row groups x NN / 32 float4 of the tile in
    // registers (the register rebalancing above gives the split warps room for a whole tile),
    // so a row is read from memory once. A tile's loads for K atom ka are issued as soon as the
    // atom ka of the tile HB steps earlier is converted, so they are in flight while the split
    // waits for the MMAs to release the A slots; the prefetch warp's L2 prefetches two tiles
    // ahead shorten their latency.
    constexpr int NV = NN / 32;  // float4 per lane and row group: columns 32 i + 4 l8 .. + 3
    constexpr int HB = 1;  // two tiles in flight at N <= 128 measured slower (N = 64: 62% -> 54%)
    float4 held[HB][SH::RG][NV];
    auto tile_ids = [&](uint32_t t, uint32_t (&ids)[SH::RG]) {
      if (t >= ntiles) {
#pragma unroll
        for (int g = 0; g < SH::RG; ++g) ids[g] = 0xffffffffu;
        return;
      }
      int c;
      uint64_t p0;
      uint32_t rows;
      tm.of(t, c, p0, rows);
#pragma unroll
      for (int g = 0; g < SH::RG; ++g) {
        const int r = row_of_group(g);
        ids[g] = (uint32_t)r < rows ? row_at(P, p0 + r) : 0xffffffffu;
      }
    };
    auto load_part = [&](float4 (&hd)[SH::RG][NV], const uint32_t (&ids)[SH::RG], int i) {  // float4 i of every row group
#pragma unroll
      for (int g = 0; g < SH::RG; ++g)
        hd[g][i] = ids[g] != 0xffffffffu
                       ? __ldcs(reinterpret_cast<const float4*>(P.x + (size_t)ids[g] * NN) + i * 8 + l8)
                       : make_float4(0.f, 0.f, 0.f, 0.f);
    };
#pragma unroll
    for (int hb = 0; hb < HB; ++hb) {
      uint32_t ids[SH::RG];
      tile_ids(t_first + (uint32_t)hb * t_step, ids);
#pragma unroll
      for (int i = 0; i < NV; ++i) load_part(held[hb], ids, i);
    }
    // tile k: convert held[k % HB], then refill it with tile k + HB
    auto do_tile = [&](float4 (&hd)[SH::RG][NV], uint32_t t, uint32_t k) {
      if (sw == 0 && lane == 0) GEMM_TRACE(k, 0);
      uint32_t rnext[SH::RG];
      tile_ids(t + (uint32_t)HB * t_step, rnext);
      // row max -> power-of-two scale
      float scl[SH::RG];
#pragma unroll
      for (int g = 0; g < SH::RG; ++g) {
        float mx = 0.f;
#pragma unroll
        for (int i = 0; i < NV; ++i)
          mx = fmaxf(mx, fmaxf(fmaxf(fabsf(hd[g][i].x), fabsf(hd[g][i].y)), fmaxf(fabsf(hd[g][i].z), fabsf(hd[g][i].w))));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
        scl[g] = row_scale(mx);
      }
      if (sw == 0 && lane == 0) GEMM_TRACE(k, 1);
      {  // row unscale factors for the epilogue: 1 / s (power of two, exact)
        const int fb = (int)(k % SH::FB);
        if (k >= (uint32_t)SH::FB) mbar_wait(&f_empty[fb], ((k / SH::FB) - 1) & 1);  // tile k-FB's factors were read
        if (l8 == 0) {
#pragma unroll
          for (int g = 0; g < SH::RG; ++g) fac[fb * SH::CR + row_of_group(g)] = 1.f / scl[g];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&f_full[fb]);
      }
      // each K atom's 64 columns of every row -> fp16 hi / lo, written as soon as the slot's
      // previous atom was read by the MMAs; one a_full arrival per atom
#pragma unroll
      for (int ka = 0; ka < SH::KA; ++ka) {
#pragma unroll
       for (int sb = 0; sb < SH::SUB; ++sb) {
        const int as = ((int)(k % SH::ABUF) * SH::SUB + sb) * SH::KA + ka;
        if (k >= (uint32_t)SH::ABUF) mbar_wait(&a_empty[as], ((k / SH::ABUF) - 1) & 1);
        if (sw == 0 && lane == 0 && sb == 0 && ka < 2) GEMM_TRACE(k, 12 + 2 * ka);  // atom slot free
        unsigned char* ahi = sm + SH::A_OFF + (uint32_t)as * 2 * ATOM_BYTES;
        unsigned char* alo = ahi + ATOM_BYTES;
#pragma unroll
        for (int g = sb * 4; g < sb * 4 + 4; ++g) {
          const int r = row_of_group(g) & (GM - 1);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float4 v = hd[g][2 * ka + h];
            const float s = scl[g];
            const float a0 = v.x * s, a1 = v.y * s, a2 = v.z * s, a3 = v.w * s;
            const uint32_t h01 = pack_h2(a0, a1), h23 = pack_h2(a2, a3);
            const float2 b01 = unpack_h2(h01), b23 = unpack_h2(h23);
            const uint32_t l01 = pack_h2(a0 - b01.x, a1 - b01.y), l23 = pack_h2(a2 - b23.x, a3 - b23.y);
            // element kk = 32 h + 4 l8 of the atom: chunk q = kk / 8, byte (kk % 8) * 2
            const uint32_t off = swz(r, h * 4 + (l8 >> 1)) + (uint32_t)(l8 & 1) * 8u;
            *reinterpret_cast<uint2*>(ahi + off) = make_uint2(h01, h23);
            *reinterpret_cast<uint2*>(alo + off) = make_uint2(l01, l23);
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic stores -> tensor core reads
        __syncwarp();
        if (lane == 0) {
          if constexpr (PAIR) mbar_arrive_remote(&a_full[as], 0); else mbar_arrive(&a_full[as]);
        }
        if (sw == 0 && lane == 0 && sb == 0 && ka < 2) GEMM_TRACE(k, 13 + 2 * ka);  // atom written
       }
        load_part(hd, rnext, 2 * ka);  // tile k + HB's atom ka, in flight from here
        load_part(hd, rnext, 2 * ka + 1);
      }
      if (sw == 0 && lane == 0) GEMM_TRACE(k, 2);
    };
    uint32_t k = 0;
    for (uint32_t t = t_first; t < ntiles; t += HB * t_step, k += HB) {
      do_tile(held[0], t, k);
      if constexpr (HB == 2) {
        if (t + t_step < ntiles) do_tile(held[HB - 1], t + t_step, k + 1);
      }
    }
    // rows with an invalid class id (bucket C): copied through, the error is flagged by hygt_bucket
    if (C > 0 && P.seg_end) {
      const uint64_t s0 = seg_at(P, C - 1), s1 = seg_at(P, C);
      for (uint64_t p = s0 + (uint64_t)blockIdx.x * SPLIT_WARPS * 4 + sw * 4 + g8; p < s1;
           p += (uint64_t)gridDim.x * SPLIT_WARPS * 4) {
        const uint32_t row = __ldg(P.idx + p);
        const float4* src = reinterpret_cast<const float4*>(P.x + (size_t)row * NN);
        float4* dst = reinterpret_cast<float4*>(P.y + (size_t)row * NN);
        for (int i = l8; i < NN / 4; i += 8) dst[i] = src[i];
      }
    }
  } else {
    if constexpr (SH::DIRECT) {
      // ------------------------------------------------------------------ epilogue ------
      // No staging: per 32-column block two tcgen05.ld.16x256b.x4 (lanes +0 and +16 of the
      // warp's quadrant; the next block's loads in flight) give thread t rows q0 + t/4 + {0, 8,
      // 16, 24} and columns 8 j + 2 (t % 4) + {0, 1} (j < 4): every STG.64 writes 8 rows x 32 B,
      // whole sectors, straight from registers. Energy: each thread sums its 8 columns over its
      // 4 rows in fp32; a shuffle reduce-scatter over the 8 row groups (fp32 partials of 16 rows,
      // the last merge exact) leaves every lane one column of the block summed over the warp's
      // 32 rows, added to a per-lane compensated fp32 accumulator per block; flushed in fp64
      // with atomics when the class changes.
      regs_dec<REG_EPI>();
      const int tq = lane & 3, tg = lane >> 2;  // column pair, row group
      // the column of a block whose energy this lane accumulates (see the reduce-scatter below)
      const int en_col = 8 * (2 * ((lane >> 2) & 1) + ((lane >> 3) & 1)) + 2 * tq + ((lane >> 4) & 1);
      constexpr int NCT = NN / 32;  // column blocks per row
      float ks[ENERGY ? NCT : 1], kc[ENERGY ? NCT : 1];  // per column block: compensated sum (value, error)
  #pragma unroll
      for (int i = 0; i < (ENERGY ? NCT : 1); ++i) ks[i] = kc[i] = 0.f;
      int en_class = -1;
      auto flush_energy = [&]() {
        if (ENERGY && en_class >= 0 && P.energy) {
  #pragma unroll
          for (int i = 0; i < NCT; ++i) {
            const double v = (double)ks[i] + (double)kc[i];
            if (v != 0.0) atomicAdd(P.energy + (size_t)en_class * NN + i * 32 + en_col, v);
            ks[i] = kc[i] = 0.f;
          }
        }
      };
      uint32_t k = 0, u = 0;
      for (uint32_t t = t_first; t < ntiles; t += t_step, ++k) {
        int c;
        uint64_t p0;
        uint32_t rows;
        tm.of(t, c, p0, rows);
        if (ENERGY && c != en_class) {
          flush_energy();
          en_class = c;
        }
        // this thread's rows: warp * 32 + tg + 8 i (i < 4)
        mbar_wait(&f_full[k % SH::FB], (k / SH::FB) & 1);
        const float ucls = __ldg(P.unscale + c);
        float frow[4];
        uint32_t orow[4];
  #pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = warp * 32 + tg + 8 * i;
          frow[i] = fac[(k % SH::FB) * SH::CR + r] * ucls;
          orow[i] = (uint32_t)r < rows ? row_at(P, p0 + r) : 0xffffffffu;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&f_empty[k % SH::FB]);
  #pragma unroll
        for (int nh = 0; nh < SH::NH; ++nh, ++u) {
          const int db = (int)(u & 1);
          mbar_wait(&d_full[db], (u >> 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          if (nh == 0 && warp == 0 && lane == 0) GEMM_TRACE(k, 5);
          // TMEM -> registers for column block cb of the unit's accumulator: v[h][4 j + m],
          // m = 0, 1: row tg + 16 h, columns 8 j + 2 tq + m; m = 2, 3: row tg + 8 + 16 h
          uint32_t v[2][16];
          auto tmem_load = [&](int cb) {
  #pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint32_t taddr = tmem + ((uint32_t)(warp * 32 + 16 * h) << 16) + (uint32_t)(db * SH::ACC + cb * 32);
              asm volatile(
                  "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                  : "=r"(v[h][0]), "=r"(v[h][1]), "=r"(v[h][2]), "=r"(v[h][3]), "=r"(v[h][4]), "=r"(v[h][5]),
                    "=r"(v[h][6]), "=r"(v[h][7]), "=r"(v[h][8]), "=r"(v[h][9]), "=r"(v[h][10]), "=r"(v[h][11]),
                    "=r"(v[h][12]), "=r"(v[h][13]), "=r"(v[h][14]), "=r"(v[h][15])
                  : "r"(taddr));
            }
          };
          constexpr int NCB = SH::NW / 32;
          auto release = [&]() {  // unit accumulator fully read: release it to unit u + 2
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) {
              if constexpr (PAIR) mbar_arrive_remote(&d_empty[db], 0); else mbar_arrive(&d_empty[db]);
            }
          };
          tmem_load(0);
          asm volatile("tcgen05.wait::ld.sync.aligned;");
          if (NCB == 1) release();
          if (P.dbg & 32) {  // diagnostic: accumulators released unread
            if (NCB > 1) release();
            continue;
          }
  #pragma unroll
          for (int cb = 0; cb < NCB; ++cb) {  // unrolled: the energy accumulators are indexed by constants
            // o[i][j][m]: row slot i (row tg + 8 i), column 8 j + 2 tq + m
            float o[4][4][2];
  #pragma unroll
            for (int h = 0; h < 2; ++h)
  #pragma unroll
              for (int j = 0; j < 4; ++j)
  #pragma unroll
                for (int m = 0; m < 2; ++m) {
                  o[2 * h][j][m] = __uint_as_float(v[h][4 * j + m]) * frow[2 * h];
                  o[2 * h + 1][j][m] = __uint_as_float(v[h][4 * j + 2 + m]) * frow[2 * h + 1];
                }
            if (cb + 1 < NCB) tmem_load(cb + 1);  // in flight while this block is stored
            const int col0 = nh * SH::NW + cb * 32;
            if (!(P.dbg & 16)) {
  #pragma unroll
              for (int i = 0; i < 4; ++i)
                if (orow[i] != 0xffffffffu) {
                  float* dst = P.y + (size_t)orow[i] * NN + col0 + 2 * tq;
  #pragma unroll
                  for (int j = 0; j < 4; ++j) __stcs(reinterpret_cast<float2*>(dst + 8 * j), make_float2(o[i][j][0], o[i][j][1]));
                }
            }
            if constexpr (ENERGY) {
              // rows past the tile's end are exact zeros (their A rows are zero): no predicate.
              // q[2 j + m]: column 8 j + 2 tq + m over this thread's 4 rows
              float q[8];
  #pragma unroll
              for (int j = 0; j < 4; ++j)
  #pragma unroll
                for (int m = 0; m < 2; ++m)
                  q[2 * j + m] = fmaf(o[0][j][m], o[0][j][m], fmaf(o[1][j][m], o[1][j][m],
                                 fmaf(o[2][j][m], o[2][j][m], o[3][j][m] * o[3][j][m])));
              // reduce-scatter over the row groups (lane bits 2, 3: fp32, 16 rows), then bit 4
              // (exact merge): lane keeps index 4 b2 + 2 b3 + b4 = column en_col
  #pragma unroll
              for (int w = 4; w >= 2; w >>= 1) {
                const bool up = (lane >> (w == 4 ? 2 : 3)) & 1;
  #pragma unroll
                for (int i = 0; i < w; ++i) {
                  const float send = up ? q[i] : q[i + w];
                  const float keep = up ? q[i + w] : q[i];
                  q[i] = keep + __shfl_xor_sync(0xffffffffu, send, w == 4 ? 4 : 8);
                }
              }
              const bool up = (lane >> 4) & 1;
              const float mine = up ? q[1] : q[0];
              const float other = __shfl_xor_sync(0xffffffffu, up ? q[0] : q[1], 16);
              const float ts = mine + other, tb = ts - mine;
              const float te = (mine - (ts - tb)) + (other - tb);  // ts + te == mine + other exactly
              const int ci = nh * NCB + cb;
              const float sn = ks[ci] + ts, sbp = sn - ks[ci];
              kc[ci] += ((ks[ci] - (sn - sbp)) + (ts - sbp)) + te;
              ks[ci] = sn;
            }
            if (cb + 1 < NCB) {
              asm volatile("tcgen05.wait::ld.sync.aligned;");
              if (cb + 2 == NCB) release();
            }
          }
        }
        if (warp == 0 && lane == 0) GEMM_TRACE(k, 6);
      }
      flush_energy();
    } else {
      // ------------------------------------------------------------------ epilogue ------
      // Thread = row (TMEM lane). Per 32-column block: tcgen05.ld (the next block's load in
      // flight), unscale, swizzled staging [32 rows][32 floats], then coalesced 128-bit stores
      // (8 lanes per row, 4 rows per instruction). Energy: each lane squares its 4 columns of
      // 8 rows in fp32, a shuffle reduce-scatter over the 4 row groups (fp32 partials of 16
      // rows, merged exactly) leaves every lane one column of the block summed over the warp's
      // 32 rows, added to a per-lane compensated fp32 accumulator per block; flushed in fp64
      // with atomics when the class changes.
      regs_dec<REG_EPI>();
      unsigned char* stg = sm + SH::STG_OFF + (uint32_t)warp * SH::STG_BYTES;
      // the column of a block whose energy this lane accumulates (see the reduce-scatter below)
      const int en_col = 4 * (lane & 7) + ((lane >> 3) & 1) * 2 + ((lane >> 4) & 1);
      constexpr int NCT = NN / 32;  // column blocks per row
      float ks[ENERGY ? NCT : 1], kc[ENERGY ? NCT : 1];  // per column block: compensated sum (value, error)
  #pragma unroll
      for (int i = 0; i < (ENERGY ? NCT : 1); ++i) ks[i] = kc[i] = 0.f;
      int en_class = -1;
      auto flush_energy = [&]() {
        if (ENERGY && en_class >= 0 && P.energy) {
  #pragma unroll
          for (int i = 0; i < NCT; ++i) {
            const double v = (double)ks[i] + (double)kc[i];
            if (v != 0.0) atomicAdd(P.energy + (size_t)en_class * NN + i * 32 + en_col, v);
            ks[i] = kc[i] = 0.f;
          }
        }
      };
      uint32_t k = 0, u = 0;
      for (uint32_t t = t_first; t < ntiles; t += t_step, ++k) {
        int c;
        uint64_t p0;
        uint32_t rows;
        tm.of(t, c, p0, rows);
        if (ENERGY && c != en_class) {
          flush_energy();
          en_class = c;
        }
        mbar_wait(&f_full[k % SH::FB], (k / SH::FB) & 1);
        // per sub-tile sb: this lane's row factor (TMEM lane = row sb GM + warp 32 + lane) and
        // the row ids of the 4-row groups it stores (rows sb GM + warp 32 + 4 i + lane / 8)
        const float ucls = __ldg(P.unscale + c);
        float f_rows[SH::SUB];
  #pragma unroll
        for (int sb = 0; sb < SH::SUB; ++sb) f_rows[sb] = fac[(k % SH::FB) * SH::CR + sb * GM + warp * 32 + lane] * ucls;
        __syncwarp();
        if (lane == 0) mbar_arrive(&f_empty[k % SH::FB]);
        uint32_t orow[SH::SUB][8];
  #pragma unroll
        for (int sb = 0; sb < SH::SUB; ++sb)
  #pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int r = sb * GM + warp * 32 + 4 * i + (lane >> 3);
            orow[sb][i] = (uint32_t)r < rows ? row_at(P, p0 + r) : 0xffffffffu;
          }
  #pragma unroll
        for (int nh = 0; nh < SH::NH; ++nh, ++u) {
          const int db = (int)(u & 1);
          mbar_wait(&d_full[db], (u >> 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          if (nh == 0 && warp == 0 && lane == 0) GEMM_TRACE(k, 5);
          // TMEM -> registers for block blk of the unit's accumulator (sub-tile blk / NCB)
          uint32_t v[32];
          auto tmem_load = [&](int blk) {
            const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(db * SH::ACC + blk * 32);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                  "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                  "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                : "r"(taddr));
          };
          constexpr int NCB = SH::NW / 32;       // column blocks per sub-tile
          constexpr int NBLK = SH::SUB * NCB;
          auto release = [&]() {  // unit accumulators fully read: release them to unit u + NBUF
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) {
              if constexpr (PAIR) mbar_arrive_remote(&d_empty[db], 0); else mbar_arrive(&d_empty[db]);
            }
          };
          tmem_load(0);
          asm volatile("tcgen05.wait::ld.sync.aligned;");
          if (NBLK == 1) release();
          if (P.dbg & 32) {  // diagnostic: accumulators released unread
            if (NBLK > 1) release();
            continue;
          }
  #pragma unroll
          for (int blk = 0; blk < NBLK; ++blk) {  // unrolled: the energy accumulators are indexed by constants
            const int sb = blk / NCB, cb = blk % NCB;
            float o[32];
  #pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __uint_as_float(v[i]) * f_rows[sb];
            if (blk + 1 < NBLK) tmem_load(blk + 1);  // in flight while this block is stored
  #pragma unroll
            for (int q = 0; q < 8; ++q)
              *reinterpret_cast<float4*>(stg + swz(lane, q)) = make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
            __syncwarp();
            // coalesced: 8 lanes per row, 4 rows per instruction
            const int col0 = nh * SH::NW + cb * 32;
            // all 8 staging reads into distinct registers first, then the predicated stores: a
            // per-row branch around load + store + energy serialises on the reused registers
            float4 ov[8];
  #pragma unroll
            for (int i = 0; i < 8; ++i) ov[i] = *reinterpret_cast<const float4*>(stg + swz(4 * i + (lane >> 3), lane & 7));
            // rows past the tile's end are exact zeros (their A rows are zero): no predicate needed;
            // squared before the stores, so no register the stores still read is overwritten
            float e0 = 0.f, e1 = 0.f, e2 = 0.f, e3 = 0.f;
            if constexpr (ENERGY) {
  #pragma unroll
              for (int i = 0; i < 8; ++i) {
                e0 = fmaf(ov[i].x, ov[i].x, e0);
                e1 = fmaf(ov[i].y, ov[i].y, e1);
                e2 = fmaf(ov[i].z, ov[i].z, e2);
                e3 = fmaf(ov[i].w, ov[i].w, e3);
              }
            }
            if (!(P.dbg & 16)) {
  #pragma unroll
              for (int i = 0; i < 8; ++i)
                if (orow[sb][i] != 0xffffffffu)
                  __stcs(reinterpret_cast<float4*>(P.y + (size_t)orow[sb][i] * NN + col0) + (lane & 7), ov[i]);
            }
            __syncwarp();  // staging reads done before the next column block overwrites it
            if constexpr (ENERGY) {
              // lanes l and l ^ 8 (row groups g, g ^ 1) keep columns {0,1} / {2,3} of their four
              // (fp32 partials of 16 rows), then l and l ^ 16 keep one of the two: their exact sum
              // (TwoSum) is added to the lane's compensated fp32 accumulator of that column (fp64
              // is only used at the class flush: fp64 adds here stall on the fp64 pipe)
              const bool h1 = (lane >> 3) & 1, h2 = (lane >> 4) & 1;
              const float sa = h1 ? e0 : e2, sb = h1 ? e1 : e3;
              const float ka = (h1 ? e2 : e0) + __shfl_xor_sync(0xffffffffu, sa, 8);
              const float kb = (h1 ? e3 : e1) + __shfl_xor_sync(0xffffffffu, sb, 8);
              const float mine = h2 ? kb : ka;
              const float other = __shfl_xor_sync(0xffffffffu, h2 ? ka : kb, 16);
              const float t = mine + other, tb = t - mine;
              const float te = (mine - (t - tb)) + (other - tb);  // t + te == mine + other exactly
              const int ci = nh * NCB + cb;
              const float sn = ks[ci] + t, sbp = sn - ks[ci];
              kc[ci] += ((ks[ci] - (sn - sbp)) + (t - sbp)) + te;
              ks[ci] = sn;
            }
            if (blk + 1 < NBLK) {
              asm volatile("tcgen05.wait::ld.sync.aligned;");
              if (blk + 2 == NBLK) release();
            }
          }
        }
        if (warp == 0 && lane == 0) GEMM_TRACE(k, 6);
      }
      flush_energy();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if constexpr (PAIR) cluster_sync(); else __syncthreads();  // no peer access after this point
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == MMA_WARP) {
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(SH::TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(SH::TMEM_COLS));
  }
}

// ------------------------------------------------------------------ N = 256: operator in TMEM --
// The N = 256 composed operator with the roles of the two MMA operands swapped ("TS" form):
//   D[out column m][row n] = sum_k OP[m][k] X[n][k]
// A (M = 256 output columns, 128 per CTA of the pair) is the class operator, resident in TMEM
// (tcgen05.mma reads A from TMEM: lane = output column, column j = fp16 pair K 2j, 2j+1); it is
// written once per class change by the epilogue warps with tcgen05.st from the operator stages
// gemm_build lays out. B (N = 128 data rows per tile, 64 per CTA) is the split's fp16 hi / lo
// tile in shared memory, SWIZZLE_128B K-major, with TS_DBUF tiles resident. Per tile 48 MMAs
// (M = 256, N = 128, K = 16): the correction terms OPhi.Xlo and OPlo.Xhi over all K first,
// then the main term OPhi.Xhi (as in the SS form, only the main term's K steps round against
// the full-size sum).
// Against the SS form (hygt_gemm_kernel with a resident B hi and a streamed B lo, 56% of HBM):
//   * the epilogue thread owns one output column, so every store instruction writes 32
//     consecutive columns of one row = one whole 128 B line (the SS form's tcgen05.ld.16x256b
//     fragments stored 8 rows x 32 B per instruction, and those 4x more L1 wavefronts starved
//     the split warps' shared-memory stores: tools/trace_summary.py, DBG 16);
//   * the split runs TS_DBUF tiles ahead of the MMAs (the SS form had one A buffer and the
//     split and MMAs advanced atom by atom), and no B operand streams through shared memory;
//   * the per-column energy is a per-thread sum (no cross-lane reduction).
namespace ts {
constexpr int TR = 128;                       // rows per tile (MMA N, both CTAs)
constexpr int CR = 64;                        // rows per CTA and tile
constexpr int KA = 4;                         // K atoms of 64
constexpr uint32_t HALF = CR * 128;           // one K atom, hi or lo, of this CTA's rows (8 KB)
constexpr uint32_t TILE = KA * 2 * HALF;      // 64 KB
constexpr int DBUF = 3;                       // data tiles resident
constexpr int FB = 4;                         // row tables (tiles in flight split -> epilogue)
constexpr uint32_t TAB_OFF = DBUF * TILE;     // [FB][TR] {row factor, row id}
constexpr uint32_t BAR_OFF = TAB_OFF + FB * TR * 8;
constexpr uint32_t TE_OFF = BAR_OFF + 256;    // + [C] u32 tile_end, [C] u32 bucket ends
constexpr uint32_t smem(int classes) { return TE_OFF + 8u * (uint32_t)classes; }
constexpr uint32_t OPHI = 0, OPLO = 128, DCOL = 256;  // TMEM columns: operator hi / lo, 2 accumulators of 128
constexpr int RG = CR / SPLIT_WARPS / 4;     // 4-row groups per split lane
}  // namespace ts
// registers per thread after setmaxnreg: the split holds half the tile the SS form's does, the
// epilogue keeps two 32-column TMEM loads and the energy in flight
constexpr int TS_REG_EPI = 160, TS_REG_SPLIT = 144;
static_assert(TS_REG_EPI + 2 * TS_REG_SPLIT + REG_MISC <= 512, "register pool");
namespace ts {
static_assert(RG == 2, "split layout");
}  // namespace ts

// 4 K steps (one 64-wide K atom) of D += A(TMEM) . B(smem)^T, M = 256 over the pair, N = 128
__device__ __forceinline__ void mma_ts_atom(uint32_t d, uint32_t a, uint64_t b, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 b0;\n\t.reg .b32 a0;\n\t"
      "setp.ne.b32 p, %3, 0;\n\t"
      "mov.b32 a0, %1;\n\tmov.b64 b0, %2;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [a0], b0, %4, p;\n\t"
      "add.s32 a0, a0, 8;\n\tadd.s64 b0, b0, 2;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [a0], b0, %4, 1;\n\t"
      "add.s32 a0, a0, 8;\n\tadd.s64 b0, b0, 2;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [a0], b0, %4, 1;\n\t"
      "add.s32 a0, a0, 8;\n\tadd.s64 b0, b0, 2;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [a0], b0, %4, 1;\n\t}\n"
      :: "r"(d), "r"(a), "l"(b), "r"(acc0), "n"(idesc_f16(ts::TR, 2 * GM)));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      :: "r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
         "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]),
         "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]),
         "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
// Tiles of one CTA in increasing order: the class index only moves forward, so the lookup is
// an incremental scan of the shared tile_end / bucket-end tables (no binary search per tile)
struct TileCursor {
  const uint32_t* tile_end;  // shared [C]
  const uint32_t* seg;       // shared [C]: bucket ends
  int classes;
  uint32_t tg, part, cr;
  int c = 0;
  __device__ __forceinline__ int cls(uint32_t t) {
    while (c < classes - 1 && tile_end[c] <= t) ++c;
    return c;
  }
  __device__ __forceinline__ void of(uint32_t t, int& cc, uint64_t& p0, uint32_t& rows) {
    cc = cls(t);
    const uint32_t first_tile = cc ? tile_end[cc - 1] : 0u;
    const uint64_t s0 = cc ? (uint64_t)seg[cc - 1] : 0ull, s1 = seg[cc];
    p0 = s0 + (uint64_t)(t - first_tile) * tg + part;
    const uint64_t left = s1 > p0 ? s1 - p0 : 0ull;
    rows = left < cr ? (uint32_t)left : cr;
  }
};
// store a float2 at the same shared-memory offset in CTA `cta` of the cluster
__device__ __forceinline__ void st_dsmem_f2(float2* p, uint32_t cta, float2 v) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, %1;\n\tst.shared::cluster.v2.f32 [ra], {%2, %3};\n\t}\n"
      :: "r"(smem_u32(p)), "r"(cta), "f"(v.x), "f"(v.y) : "memory");
}

template <bool ENERGY>
__global__ void __launch_bounds__(GEMM_THREADS, 1) hygt_gemm_ts_kernel(const GemmParams P) {  // clusters of 2
  constexpr int NN = 256;
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + ts::BAR_OFF);
  uint64_t* x_full = bars;                  // [DBUF] data tile written (rank 0: count 2 SPLIT_WARPS)
  uint64_t* x_empty = x_full + ts::DBUF;    // [DBUF] data tile read by the MMAs (commit, both CTAs)
  uint64_t* d_full = x_empty + ts::DBUF;    // [2]    accumulator done (commit, both CTAs)
  uint64_t* d_empty = d_full + 2;           // [2]    accumulator read (rank 0: count 2 EPI_WARPS)
  uint64_t* f_split = d_empty + 2;          // [FB]   this CTA's half of the row table written (count SPLIT_WARPS)
  uint64_t* f_full = f_split + ts::FB;      // [FB]   row table complete (count 2: the relays of both CTAs)
  uint64_t* f_empty = f_full + ts::FB;      // [FB]   row table read (count 2 EPI_WARPS: both epilogues)
  uint64_t* op_full = f_empty + ts::FB;     // [1]    class operator in TMEM (rank 0: count 2 EPI_WARPS)
  uint32_t* tmem_sh = reinterpret_cast<uint32_t*>(op_full + 1);
  static_assert((2 * ts::DBUF + 4 + 3 * ts::FB + 1) * 8 + 4 <= 256, "barrier area");
  uint32_t* tile_end_sh = reinterpret_cast<uint32_t*>(sm + ts::TE_OFF);
  uint32_t* seg_sh = tile_end_sh + P.classes;  // [C] bucket ends
  // [FB][TR] row table {row factor (1 / row scale x class unscale), row id (bits)}: rows
  // rank 64 .. written by this CTA's split, the other half copied in by the peer's relay warp;
  // read by this CTA's epilogue
  float2* tab = reinterpret_cast<float2*>(sm + ts::TAB_OFF);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int C = P.classes;
  const uint32_t rank = cluster_rank(), peer = rank ^ 1u;
  const uint32_t t_first = cluster_id(), t_step = cluster_count();
  if (warp == 0) {  // per-class cumulative tile counts (tiles of TR rows), bucket ends
    uint32_t run = 0;
    for (int c0 = 0; c0 < C; c0 += 32) {
      const int c = c0 + lane;
      uint32_t nt = 0;
      if (c < C) {
        const uint64_t s0 = c ? seg_at(P, c - 1) : 0ull, s1 = seg_at(P, c);
        nt = (uint32_t)((s1 - s0 + ts::TR - 1) / ts::TR);
        seg_sh[c] = (uint32_t)s1;
      }
      uint32_t v = nt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (c < C) tile_end_sh[c] = run + v;
      run += __shfl_sync(0xffffffffu, v, 31);
    }
  }
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(tmem_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < ts::DBUF; ++i) { mbar_init(&x_full[i], 2 * SPLIT_WARPS); mbar_init(&x_empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&d_full[i], 1); mbar_init(&d_empty[i], 2 * EPI_WARPS); }
    for (int i = 0; i < ts::FB; ++i) {
      mbar_init(&f_split[i], SPLIT_WARPS);
      mbar_init(&f_full[i], 2);
      mbar_init(&f_empty[i], 2 * EPI_WARPS);
    }
    mbar_init(op_full, 2 * EPI_WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_sh;
  const uint32_t ntiles = C ? tile_end_sh[C - 1] : 0u;

  if (warp == MMA_WARP) {
    // ------------------------------------------------------------------ MMA issuer ----
    regs_dec<REG_MISC>();
    if (rank == 0) {  // the whole warp, one elected lane issues (see elect_one)
      const bool leader = elect_one();
      TileCursor cur_t{tile_end_sh, seg_sh, C, 0, 0, 0};
      uint32_t k = 0, nop = 0;
      int cur = -1;
      for (uint32_t t = t_first; t < ntiles; t += t_step, ++k) {
        const int c = cur_t.cls(t);
        if (c != cur) {  // both CTAs' epilogues wrote this class's operator into TMEM
          mbar_wait(op_full, nop & 1);
          ++nop;
          cur = c;
        }
        const int db = (int)(k & 1), xb = (int)(k % ts::DBUF);
        if (k >= 2) mbar_wait(&d_empty[db], ((k >> 1) - 1) & 1);
        mbar_wait(&x_full[xb], (k / ts::DBUF) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        __syncwarp();
        if (leader) {
          GEMM_TRACE(k, 3);
          const uint32_t dacc = tmem + ts::DCOL + (uint32_t)db * ts::TR;
          const uint64_t xd = desc_sw128(smem_u32(sm + (uint32_t)xb * ts::TILE));
          constexpr uint64_t ATOM = (2 * ts::HALF) >> 4, LO = ts::HALF >> 4;  // descriptor address units
#pragma unroll
          for (int ka = 0; ka < ts::KA; ++ka)  // OPhi . Xlo
            mma_ts_atom(dacc, tmem + ts::OPHI + 32u * ka, xd + ka * ATOM + LO, (uint32_t)ka);
#pragma unroll
          for (int ka = 0; ka < ts::KA; ++ka)  // OPlo . Xhi
            mma_ts_atom(dacc, tmem + ts::OPLO + 32u * ka, xd + ka * ATOM, 1u);
#pragma unroll
          for (int ka = 0; ka < ts::KA; ++ka)  // OPhi . Xhi
            mma_ts_atom(dacc, tmem + ts::OPHI + 32u * ka, xd + ka * ATOM, 1u);
          tc_commit<true>(&x_empty[xb]);
          tc_commit<true>(&d_full[db]);
          GEMM_TRACE(k, 4);
        }
        __syncwarp();
      }
    }
  } else if (warp == PF_WARP) {
    // ------------------------------------------------------------------ row prefetch --
    regs_dec<REG_MISC>();
    // L2 prefetch of this CTA's rows of the tile 2 steps ahead, paced by the split (f_full)
    TileCursor cur_t{tile_end_sh, seg_sh, C, (uint32_t)ts::TR, rank * (uint32_t)ts::CR, (uint32_t)ts::CR};
    auto prefetch_rows = [&](uint32_t tp) {
      if (tp >= ntiles) return;
      int c;
      uint64_t p0;
      uint32_t rows;
      cur_t.of(tp, c, p0, rows);
      uint32_t id[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const uint32_t r = (uint32_t)(lane + 32 * i);
        id[i] = r < rows ? row_at(P, p0 + r) : 0xffffffffu;
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
        if (id[i] != 0xffffffffu)
#pragma unroll
          for (int l = 0; l < NN / 32; ++l)
            asm volatile("prefetch.global.L2 [%0];" :: "l"(P.x + (size_t)id[i] * NN + l * 32) : "memory");
    };
    if (!(P.dbg & 2)) {
      constexpr int PF_AHEAD = 2;
      for (int a = 0; a < PF_AHEAD; ++a) prefetch_rows(t_first + (uint32_t)a * t_step);
      uint32_t k = 0;
      for (uint32_t t = t_first + PF_AHEAD * t_step; t < ntiles; t += t_step, ++k) {
        mbar_wait(&f_full[k % ts::FB], (k / ts::FB) & 1);
        prefetch_rows(t);
      }
    }
  } else if (warp == PROD_WARP) {
    // ------------------------------------------------------------------ row-table relay
    regs_dec<REG_MISC>();
    // Per tile: once this CTA's split wrote its half of the row table (f_split), copy the half
    // into the peer's table over DSMEM and signal both tables' f_full, the peer's with a
    // cluster-scope release: the release (a memory barrier) waits only for these stores, not
    // for the split warps' global loads in flight.
    const float2* mine = tab + rank * ts::CR;
    uint32_t k = 0;
    for (uint32_t t = t_first; t < ntiles; t += t_step, ++k) {
      const int fb = (int)(k % ts::FB);
      mbar_wait(&f_split[fb], (k / ts::FB) & 1);
#pragma unroll
      for (int i = 0; i < ts::CR / 32; ++i) {
        const float2* e = mine + fb * ts::TR + 32 * i + lane;
        st_dsmem_f2(const_cast<float2*>(e), peer, *e);
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&f_full[fb]);
        mbar_arrive_remote_release(&f_full[fb], peer);
      }
    }
  } else if (warp > PROD_WARP) {
    regs_dec<REG_MISC>();  // idle (keeps the warpgroups whole for the register rebalancing)
  } else if (warp >= EPI_WARPS) {
    // ------------------------------------------------------------------ split warps ---
    regs_inc<TS_REG_SPLIT>();
    const int sw = warp - EPI_WARPS;
    const int g8 = lane >> 3, l8 = lane & 7;
    // rows of 4-row group g (the conflict-free STS.64 pattern of hygt_gemm_kernel)
    auto row_of_group = [&](int g) {
      const int i = sw * ts::RG + g, b16 = i >> 2, gg = i & 3;
      return b16 * 16 + (gg & 1) * 2 + (gg >> 1) * 8 + (g8 >> 1) + (g8 & 1) * 4;
    };
    constexpr int NV = NN / 32;
    float4 held[ts::RG][NV];
    TileCursor cur_t{tile_end_sh, seg_sh, C, (uint32_t)ts::TR, rank * (uint32_t)ts::CR, (uint32_t)ts::CR};
    // row ids of this CTA's rows of tile t (and its class)
    auto tile_ids = [&](uint32_t t, uint32_t (&ids)[ts::RG]) {
      if (t >= ntiles) {
#pragma unroll
        for (int g = 0; g < ts::RG; ++g) ids[g] = 0xffffffffu;
        return 0;
      }
      int c;
      uint64_t p0;
      uint32_t rows;
      cur_t.of(t, c, p0, rows);
#pragma unroll
      for (int g = 0; g < ts::RG; ++g) {
        const int r = row_of_group(g);
        ids[g] = (uint32_t)r < rows ? row_at(P, p0 + r) : 0xffffffffu;
      }
      return c;
    };
    auto load_part = [&](const uint32_t (&ids)[ts::RG], int i) {
#pragma unroll
      for (int g = 0; g < ts::RG; ++g)
        held[g][i] = ids[g] != 0xffffffffu
                         ? __ldcs(reinterpret_cast<const float4*>(P.x + (size_t)ids[g] * NN) + i * 8 + l8)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
    };
    uint32_t ids[ts::RG];
    int cls = tile_ids(t_first, ids);
#pragma unroll
    for (int i = 0; i < NV; ++i) load_part(ids, i);
    uint32_t k = 0;
    for (uint32_t t = t_first; t < ntiles; t += t_step, ++k) {
      if (sw == 0 && lane == 0) GEMM_TRACE(k, 0);
      float scl[ts::RG];
#pragma unroll
      for (int g = 0; g < ts::RG; ++g) {
        float mx = 0.f;
#pragma unroll
        for (int i = 0; i < NV; ++i)
          mx = fmaxf(mx, fmaxf(fmaxf(fabsf(held[g][i].x), fabsf(held[g][i].y)), fmaxf(fabsf(held[g][i].z), fabsf(held[g][i].w))));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
        scl[g] = row_scale(mx);
      }
      if (sw == 0 && lane == 0) GEMM_TRACE(k, 1);
      {  // this CTA's rows of the row table (the relay warp copies them to the peer)
        const int fb = (int)(k % ts::FB);
        const float ucls = __ldg(P.unscale + cls);
        if (k >= (uint32_t)ts::FB) mbar_wait(&f_empty[fb], ((k / ts::FB) - 1) & 1);  // both epilogues done with fb
        if (l8 == 0) {
#pragma unroll
          for (int g = 0; g < ts::RG; ++g)
            tab[fb * ts::TR + rank * ts::CR + row_of_group(g)] = make_float2(ucls / scl[g], __uint_as_float(ids[g]));
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&f_split[fb]);
      }
      uint32_t rnext[ts::RG];
      const int cnext = tile_ids(t + t_step, rnext);
      const int xb = (int)(k % ts::DBUF);
      if (k >= (uint32_t)ts::DBUF) mbar_wait(&x_empty[xb], ((k / ts::DBUF) - 1) & 1);
      if (sw == 0 && lane == 0) GEMM_TRACE(k, 12);
      unsigned char* xt = sm + (uint32_t)xb * ts::TILE;
#pragma unroll
      for (int ka = 0; ka < ts::KA; ++ka) {
        unsigned char* xhi = xt + (uint32_t)ka * 2 * ts::HALF;
        unsigned char* xlo = xhi + ts::HALF;
#pragma unroll
        for (int g = 0; g < ts::RG; ++g) {
          const int r = row_of_group(g);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float4 v = held[g][2 * ka + h];
            const float s = scl[g];
            const float a0 = v.x * s, a1 = v.y * s, a2 = v.z * s, a3 = v.w * s;
            const uint32_t h01 = pack_h2(a0, a1), h23 = pack_h2(a2, a3);
            const float2 b01 = unpack_h2(h01), b23 = unpack_h2(h23);
            const uint32_t l01 = pack_h2(a0 - b01.x, a1 - b01.y), l23 = pack_h2(a2 - b23.x, a3 - b23.y);
            const uint32_t off = swz(r, h * 4 + (l8 >> 1)) + (uint32_t)(l8 & 1) * 8u;
            *reinterpret_cast<uint2*>(xhi + off) = make_uint2(h01, h23);
            *reinterpret_cast<uint2*>(xlo + off) = make_uint2(l01, l23);
          }
        }
        load_part(rnext, 2 * ka);  // the next tile's atom ka, in flight from here
        load_part(rnext, 2 * ka + 1);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic stores -> tensor core reads
      __syncwarp();
      if (lane == 0) {
        if (rank == 0) mbar_arrive(&x_full[xb]); else mbar_arrive_remote(&x_full[xb], 0);
      }
      if (sw == 0 && lane == 0) GEMM_TRACE(k, 2);
#pragma unroll
      for (int g = 0; g < ts::RG; ++g) ids[g] = rnext[g];
      cls = cnext;
    }
    // rows with an invalid class id (bucket C): copied through, the error is flagged by hygt_bucket
    if (C > 0 && P.seg_end) {
      const uint64_t s0 = seg_at(P, C - 1), s1 = seg_at(P, C);
      for (uint64_t p = s0 + (uint64_t)blockIdx.x * SPLIT_WARPS * 4 + sw * 4 + g8; p < s1;
           p += (uint64_t)gridDim.x * SPLIT_WARPS * 4) {
        const uint32_t row = __ldg(P.idx + p);
        const float4* src = reinterpret_cast<const float4*>(P.x + (size_t)row * NN);
        float4* dst = reinterpret_cast<float4*>(P.y + (size_t)row * NN);
        for (int i = l8; i < NN / 4; i += 8) dst[i] = src[i];
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue ------
    // Thread = output column m = rank 128 + warp 32 + lane (TMEM lane). Per tile, per block of
    // 32 rows one tcgen05.ld.32x32b.x32 (the next block's in flight); per row one broadcast
    // LDS.64 of {row factor, row id} from the row table the splits of both CTAs filled, and
    // one STG.32 per warp = one whole 128 B line. Energy: the thread's column summed in fp32
    // per 16 rows, compensated (TwoSum) across blocks, fp64 atomics at the class flush. On a
    // class change first the class operator: this thread's output row of the operator stages
    // (hi and lo, de-swizzled) into TMEM lane m with tcgen05.st.
    regs_inc<TS_REG_EPI>();
    const uint32_t col = rank * 128u + (uint32_t)(warp * 32 + lane);
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    float* ycol = P.y + col;
    float ks = 0.f, kc = 0.f;
    int cur = -1;
    auto flush_energy = [&]() {
      if (ENERGY && cur >= 0 && P.energy) {
        const double v = (double)ks + (double)kc;
        if (v != 0.0) atomicAdd(P.energy + (size_t)cur * NN + col, v);
        ks = kc = 0.f;
      }
    };
    // operator stages (gemm_build): [C][KA][2 halves][hi | lo][128 rows x 128 B, SW128]
    constexpr uint32_t GSTAGE = 2u * 128 * 128;
    const uint32_t orow = (uint32_t)(warp * 32 + lane);  // row of this CTA's half (= rank)
    TileCursor cur_t{tile_end_sh, seg_sh, C, 0, 0, 0};
    uint32_t k = 0;
    for (uint32_t t = t_first; t < ntiles; t += t_step, ++k) {
      const int c = cur_t.cls(t);
      if (c != cur) {
        flush_energy();
        // the previous tile's accumulator was waited for (d_full): every MMA that read the
        // previous operator is complete, and the MMAs of this tile wait for op_full
        asm volatile("tcgen05.fence::after_thread_sync;");
        const unsigned char* src = P.bops + (size_t)c * ts::KA * 2 * GSTAGE + (size_t)rank * GSTAGE + (size_t)orow * 128;
#pragma unroll 1
        for (int part = 0; part < 2; ++part) {  // hi, lo
#pragma unroll 1
          for (int ka = 0; ka < ts::KA; ++ka) {
            const uint4* s4 = reinterpret_cast<const uint4*>(src + (size_t)ka * 2 * GSTAGE + (size_t)part * (GSTAGE / 2));
            uint32_t v[32];
#pragma unroll
            for (int q = 0; q < 8; ++q) {  // chunk q (K 8q .. 8q + 7) sits at 16 B slot q ^ (row & 7)
              const uint4 u = __ldg(s4 + (q ^ (orow & 7)));
              v[4 * q] = u.x; v[4 * q + 1] = u.y; v[4 * q + 2] = u.z; v[4 * q + 3] = u.w;
            }
            tmem_st32(tmem + lane_base + (part ? ts::OPLO : ts::OPHI) + 32u * ka, v);
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) {
          if (rank == 0) mbar_arrive(op_full); else mbar_arrive_remote_release(op_full, 0);
        }
        cur = c;
      }
      const int fb = (int)(k % ts::FB), db = (int)(k & 1);
      mbar_wait_cluster(&f_full[fb], (k / ts::FB) & 1);  // pairs with the relays' cluster release
      mbar_wait(&d_full[db], (k >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (warp == 0 && lane == 0) GEMM_TRACE(k, 5);
      const uint32_t dbase = tmem + lane_base + ts::DCOL + (uint32_t)db * ts::TR;
      const float2* tk = tab + fb * ts::TR;
      uint32_t v[2][32];
      tmem_ld32(dbase, v[0]);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        if (i + 1 < 4) tmem_ld32(dbase + 32u * (i + 1), v[(i + 1) & 1]);
        if (i == 3) {  // accumulator read: release it to tile k + 2
          asm volatile("tcgen05.fence::before_thread_sync;");
          __syncwarp();
          if (lane == 0) {
            if (rank == 0) mbar_arrive(&d_empty[db]); else mbar_arrive_remote(&d_empty[db], 0);
          }
        }
        if (P.dbg & 32) continue;
        float e0 = 0.f, e1 = 0.f;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float2 fe = tk[32 * i + j];  // broadcast
          const uint32_t rid = __float_as_uint(fe.y);
          const float val = __uint_as_float(v[i & 1][j]) * fe.x;
          if (ENERGY) {
            if (j & 1) e1 = fmaf(val, val, e1); else e0 = fmaf(val, val, e0);
          }
          if (rid != 0xffffffffu && !(P.dbg & 16)) __stcs(ycol + (size_t)rid * NN, val);
        }
        if (ENERGY) {  // rows past the tile's end are exact zeros (their B rows are zero)
          const float ts_ = e0 + e1, tb = ts_ - e0;
          const float te = (e0 - (ts_ - tb)) + (e1 - tb);
          const float sn = ks + ts_, sbp = sn - ks;
          kc += ((ks - (sn - sbp)) + (ts_ - sbp)) + te;
          ks = sn;
        }
      }
      __syncwarp();
      if (lane == 0) {  // row table fb read: both splits may refill it
        mbar_arrive(&f_empty[fb]);
        mbar_arrive_remote(&f_empty[fb], peer);
      }
      if (warp == 0 && lane == 0) GEMM_TRACE(k, 6);
    }
    flush_energy();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync();  // no peer access after this point
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == MMA_WARP) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" :: "r"(tmem));
}

// ---------------------------------------------------------------- host: operand builder ----
// Round to nearest even fp16 (bits) from fp64, no double rounding.
uint16_t half_rn(double v) {
  const uint16_t sign = std::signbit(v) ? 0x8000u : 0u;
  double a = std::fabs(v);
  if (a == 0.0) return sign;
  if (!(a < 65520.0)) return (uint16_t)(sign | 0x7c00u);
  int ex = 0;
  std::frexp(a, &ex);
  int E = ex - 1;  // a in [2^E, 2^(E+1))
  if (E < -14) {   // subnormal: units of 2^-24
    const double q = std::nearbyint(std::ldexp(a, 24));
    return (uint16_t)(sign | (uint16_t)q);  // q == 1024 becomes the smallest normal
  }
  double q = std::nearbyint((std::ldexp(a, -E) - 1.0) * 1024.0);
  if (q >= 1024.0) {
    q = 0.0;
    ++E;
  }
  if (E > 15) return (uint16_t)(sign | 0x7c00u);
  return (uint16_t)(sign | (uint16_t)((E + 15) << 10) | (uint16_t)q);
}
double half_to_double(uint16_t h) {
  const int e = (h >> 10) & 31, m = h & 1023;
  const double v = e == 0 ? std::ldexp((double)m, -24) : std::ldexp(1.0 + m / 1024.0, e - 15);
  return (h & 0x8000u) ? -v : v;
}

}  // namespace

int gemm_smem_bytes(int n) {
  switch (n) {
    case 64: return (int)std::max(Shape<64, true, true>::smem(HYGT_GEMM_MAX_CLASSES), Shape<64, true, false>::smem(HYGT_GEMM_MAX_CLASSES));
    case 128: return (int)std::max(Shape<128, true, true>::smem(HYGT_GEMM_MAX_CLASSES), Shape<128, true, false>::smem(HYGT_GEMM_MAX_CLASSES));
    case 256: return (int)std::max(Shape<256, true, false>::smem(HYGT_GEMM_MAX_CLASSES), ts::smem(HYGT_GEMM_MAX_CLASSES));
    default: return 0;
  }
}

bool gemm_supported(int n, int classes) {
  return (n == 64 || n == 128 || n == 256) && classes >= 1 && classes <= HYGT_GEMM_MAX_CLASSES;
}

// ops[c] = B_c (N x K row-major fp64): out[row] = B_c in[row]. Builds the per-class hi/lo fp16
// stages in the SW128 K-major layout the kernel streams, and the per-class unscale 2^-kB.
int gemm_build(int n, int classes, const double* ops, GemmOperands& out) {
  if (!gemm_supported(n, classes)) return hygt_set_error(HYGT_ERR_ARGUMENT, "gemm: unsupported shape");
  const int nw = n < 128 ? n : 128, ka = n / 64, nh = n / nw;
  const size_t stage = (size_t)2 * nw * 128, per_class = stage * ka * nh;
  std::vector<unsigned char> host(per_class * classes, 0);
  std::vector<float> unscale(classes);
  for (int c = 0; c < classes; ++c) {
    const double* b = ops + (size_t)c * n * n;
    double mx = 0;
    for (size_t i = 0; i < (size_t)n * n; ++i) mx = std::max(mx, std::fabs(b[i]));
    if (!std::isfinite(mx)) return hygt_set_error(HYGT_ERR_ARGUMENT, "gemm: non-finite operator");
    int kb = 0;
    if (mx > 0) {
      int ex = 0;
      std::frexp(mx, &ex);  // mx in [2^(ex-1), 2^ex)
      kb = 15 - ex;         // mx 2^kb in [2^14, 2^15)
    }
    unscale[c] = (float)std::ldexp(1.0, -kb);
    unsigned char* dst = host.data() + per_class * c;
    for (int a = 0; a < ka; ++a)
      for (int h = 0; h < nh; ++h) {
        unsigned char* st = dst + stage * (size_t)(a * nh + h);
        for (int r = 0; r < nw; ++r)
          for (int kk = 0; kk < 64; ++kk) {
            const double v = std::ldexp(b[(size_t)(h * nw + r) * n + a * 64 + kk], kb);
            const uint16_t hi = half_rn(v);
            const uint16_t lo = half_rn(v - half_to_double(hi));
            const int q = kk / 8;
            const size_t off = (size_t)r * 128 + (size_t)((q ^ (r & 7)) << 4) + (size_t)(kk % 8) * 2;
            std::memcpy(st + off, &hi, 2);
            std::memcpy(st + stage / 2 + off, &lo, 2);
          }
      }
  }
  gemm_release(out);
  out.n = n;
  out.classes = classes;
  if (cudaMalloc(&out.d_ops, host.size()) != cudaSuccess || cudaMalloc(&out.d_unscale, classes * sizeof(float)) != cudaSuccess) {
    gemm_release(out);
    cudaGetLastError();
    return hygt_set_error(HYGT_ERR_CUDA, "gemm: cudaMalloc failed");
  }
  if (cudaMemcpy(out.d_ops, host.data(), host.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(out.d_unscale, unscale.data(), classes * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess) {
    gemm_release(out);
    return hygt_set_error(HYGT_ERR_CUDA, "gemm: upload failed");
  }
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&out.num_sms, cudaDevAttrMultiProcessorCount, dev);
  if (out.num_sms <= 0) out.num_sms = 148;
  return HYGT_OK;
}

void gemm_release(GemmOperands& g) {
  cudaFree(g.d_ops);
  cudaFree(g.d_unscale);
  g.d_ops = nullptr;
  g.d_unscale = nullptr;
}

namespace {
template <int NN, bool E, bool PAIR, bool WIDE>
int launch_one(const GemmParams& P, int num_sms, cudaStream_t st) {
  using SH = Shape<NN, PAIR, WIDE>;
  const auto fn = hygt_gemm_kernel<NN, E, PAIR, WIDE>;
  const uint32_t smem = (SH::smem(P.classes) + 15u) & ~15u;
  hygt_smem_attr(reinterpret_cast<const void*>(fn), smem);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  cfg.gridDim = dim3(PAIR ? (unsigned)(num_sms / 2 * 2) : (unsigned)num_sms);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = PAIR ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, fn, P);
  return e == cudaSuccess ? HYGT_OK : hygt_set_error(HYGT_ERR_CUDA, cudaGetErrorString(e));
}
template <bool E>
int launch_ts(const GemmParams& P, int num_sms, cudaStream_t st) {
  const auto fn = hygt_gemm_ts_kernel<E>;
  const uint32_t smem = (ts::smem(P.classes) + 15u) & ~15u;
  hygt_smem_attr(reinterpret_cast<const void*>(fn), smem);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  cfg.gridDim = dim3((unsigned)(num_sms / 2 * 2));
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, fn, P);
  return e == cudaSuccess ? HYGT_OK : hygt_set_error(HYGT_ERR_CUDA, cudaGetErrorString(e));
}
template <int NN>
int launch_n(const GemmParams& P, int grid, bool pair, bool wide, bool tsf, cudaStream_t st) {
  // N = 256 with CTA pairs: the operator-in-TMEM form (hygt_gemm_ts_kernel)
  if (NN == 256 && pair && tsf) return P.energy ? launch_ts<true>(P, grid, st) : launch_ts<false>(P, grid, st);
  // wide: one unit of all N columns per tile, merged accumulator (N = 256 only with CTA pairs)
  // (the resident B hi halves at N = 256 leave room for at most 384 classes' tile table)
  if (pair && wide && (NN != 256 || P.classes <= 384))
    return P.energy ? launch_one<NN, true, true, true>(P, grid, st) : launch_one<NN, false, true, true>(P, grid, st);
  if constexpr (NN <= 128) {
    if (wide)
      return P.energy ? launch_one<NN, true, false, true>(P, grid, st) : launch_one<NN, false, false, true>(P, grid, st);
  }
  if (pair) return P.energy ? launch_one<NN, true, true, false>(P, grid, st) : launch_one<NN, false, true, false>(P, grid, st);
  return P.energy ? launch_one<NN, true, false, false>(P, grid, st) : launch_one<NN, false, false, false>(P, grid, st);
}
}  // namespace

unsigned long long* g_gemm_trace = nullptr;  // debug hook (hygt_debug_gemm_trace)

int gemm_run(const GemmOperands& g, const float* x, float* y, const uint32_t* idx,
             const uint32_t* seg_end, uint64_t count, double* energy, cudaStream_t st) {
  if (!count) return HYGT_OK;
  GemmParams P{};
  P.trace = g_gemm_trace;
  P.dbg = g.dbg;
  P.x = x;
  P.y = y;
  P.idx = idx;
  P.seg_end = seg_end;
  P.classes = g.classes;
  P.count = count;
  P.bops = g.d_ops;
  P.unscale = g.d_unscale;
  P.energy = energy;
  const uint64_t tiles = (count + GM - 1) / GM + (uint64_t)g.classes;
  const bool pair = g.pair && g.num_sms >= 2;
  const int grid = (int)std::min<uint64_t>((uint64_t)g.num_sms, pair ? 2 * ((tiles + 1) / 2) : tiles);
  switch (g.n) {
    case 64: return launch_n<64>(P, grid, pair, g.wide, g.ts, st);
    case 128: return launch_n<128>(P, grid, pair, g.wide, g.ts, st);
    case 256: return launch_n<256>(P, grid, pair, g.wide, g.ts, st);
    default: return hygt_set_error(HYGT_ERR_ARGUMENT, "gemm: unsupported N");
  }
}

}  // namespace hygt_gpu

// Debug hook (not part of the public header): per-tile clock64 events of CTA 0 of the next
// tensor-core launches are written to dev[k * 8 + e] (k < 64; e: 0/1/2 split pass-1 start /
// pass-1 end / atoms written, 3/4 MMA start / committed, 5/6 epilogue start / end); nullptr off.
extern "C" void hygt_debug_gemm_trace(void* dev) {
  hygt_gpu::g_gemm_trace = static_cast<unsigned long long*>(dev);
}
