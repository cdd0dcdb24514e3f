// hygt_corr_tc.cu -- per-class second moments sum_c += r r^T (SURVEY.md §8 f3,
// CorrelationAccumulator::add, statistics.hpp:63-99) on the 5th-generation tensor cores,
// N = 64, 128 and 256.
//
// Exactness. The reference accumulates r_i r_j in fp64, and fp32 samples make every product exact
// there; the parity bar is 1e-12 of the largest sum. Floating-point tensor-core inputs cannot
// carry that, integers can: within a run of tiles of one class, column i of every row is taken to
// fixed point relative to a per-column power of two 2^E_i > max |r_i| (X = rint(r 2^(54 - E_i)),
// |X| < 2^54, exact for every sample above 2^(E_i - 30), rounded at 2^(E_i - 55) below) and split
// into 7 balanced base-256 digits d_0 .. d_6 in [-128, 127] (d_0 most significant). Then
//   X_i X_j = sum_{p,q} d_p(i) d_q(j) 256^(12 - p - q),
// and the kernel accumulates, per level L = p + q <= 6, D_L = sum_rows sum_{p+q=L} d_p(i) d_q(j)
// with tcgen05.mma.kind::i8 into int32 TMEM accumulators: exact (|D_L| < 2^31 for up to 128
// tiles). The dropped levels L > 6 and the rounding of small samples contribute below
// 2^-54 of max|r_i| max|r_j| per product. At a flush (class change, an exponent re-base when a
// tile exceeds the run's scale, every 128 tiles, the end) the levels are combined in fp64,
// sum_L D_L 2^(-8L) 2^(E_i + E_j - 12), and added to the class's fp64 sums.
//
// Digits. X comes from two exact power-of-two FMULs (r 2^a 2^b, a + b = 54 - E_i) and one
// F2I.S64; the digits are the bytes of (X + C) ^ C with C = 0x80 in each of the 7 bytes
// (X + C = sum (d_p + 128) 256^(6-p), each d_p + 128 in [0, 255]): 7 instructions per sample.
// Byte permutes (PRMT) then transpose 16 rows into each digit slice.
//
// Operands: digit p of column i is row i of a digit slice, K = the tile's 128 rows, SWIZZLE_128B
// K-major. A tile is 128 bucketed rows of one class; one CTA per SM (N = 64) or per SM and role.
//   N = 64 (one symmetric 64-column block): only the digit pairs p <= q are multiplied, two per
//           MMA (A = two adjacent digit slices, M = 128; B = one slice, N = 64): 8 MMAs x 4 K
//           steps per tile, one 64-column TMEM block each (the table at s64_pos below).
//   N = 128 / 256 (64-column blocks I != J, one "role" per CTA): A = [digit p of block I ;
//           digit p of block J] (M = 128), B = digit q of block J (the second half of A's stack q,
//           no extra copy). One MMA gives output blocks (I, J) in TMEM lanes 0-63 and (J, J) in
//           lanes 64-127, level p + q in column block p + q: 28 MMAs x 4 K steps per tile. TMEM
//           (448 of 512 columns for 7 levels x 64) holds one such pair per SM, so the upper block
//           triangle is covered by roles (N = 256: (0,1) (1,2) (2,3) (3,0) give every off-diagonal
//           block next to a diagonal one, (0,2) (1,3) the last two off-diagonal blocks); the CTAs of
//           the roles walk the same row range together, so the rows come from L2 after the first.
// Warps: 8 (N = 64) or 16 (8 per block) split warps -- lane l holds columns l and l + 32 of 16
// rows of its block, per-column maxima, the run's exponents, the digits, and the flushes (warp w
// reads TMEM lane quadrant w % 4) -- and one MMA warp issuing from one thread.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../../include/hygt_gpu.h"
#include "hygt_corr_tc.h"

int hygt_set_error(int status, const char* msg);  // hygt_capi.cu
void hygt_smem_attr(const void* fn, size_t bytes);

namespace hygt_gpu {
namespace {

constexpr int CN = 64;             // columns per block
constexpr int KT = 128;            // rows per tile (MMA K)
constexpr int NDIG = 7;            // digits per sample
constexpr uint32_t SLICE = CN * 128;  // 64 rows x 128 B (K = 128 int8)
constexpr int MAX_RUN_TILES = 128;    // int32 headroom: |D_L| <= 7 * 128 * 128^2 per tile < 2^31 / 146
constexpr int HEADROOM = 2;  // bits of a run's exponents above the first tile's column maxima

// N = 64 (one symmetric 64 x 64 block): G_qp = G_pq^T, so only the 16 digit pairs p <= q, p + q <= 6
// are multiplied, two per MMA: A = two digit slices adjacent in shared memory (M = 128), B = one
// slice (N = 64). With the slices stored in the order 0 1 3 2 4 6 5 the 16 pairs are covered
// exactly by 8 MMAs (x 4 K steps; found by exhaustive search over slice orders), each into its own
// 64-column TMEM block (8 x 64 = all 512 columns), so every (block, lane half) holds one pair:
//   block : A lower, A upper, B   -> lanes 0-63         | lanes 64-127
//     0   :    2        4     2   -> (2,2) level 4 diag | (2,4) level 6
//     1   :    0        1     5   -> (0,5) level 5      | (1,5) level 6
//     2   :    0        1     0   -> (0,0) level 0 diag | (0,1) level 1
//     3   :    1        3     1   -> (1,1) level 2 diag | (1,3) level 4
//     4   :    3        2     0   -> (0,3) level 3      | (0,2) level 2
//     5   :    4        6     0   -> (0,4) level 4      | (0,6) level 6
//     6   :    3        2     3   -> (3,3) level 6 diag | (2,3) level 5
//     7   :    2        4     1   -> (1,2) level 3      | (1,4) level 5
// The flush forms U = sum over the off-diagonal pairs + half the diagonal pairs (weights
// 2^(-8 level)) and adds U(i, j) to sum(i, j) and to sum(j, i): U + U^T is the full product.
// (packed nibbles: constexpr functions are usable in device code, constexpr arrays are not)
__host__ __device__ constexpr int s64_pos(int p) { return (0x5642310u >> (4 * p)) & 15; }  // digit -> slice position
__host__ __device__ constexpr int s64_a(int m) { return (0x23431002u >> (4 * m)) & 15; }   // lower digit of A (the upper follows it)
__host__ __device__ constexpr int s64_b(int m) { return (0x13001052u >> (4 * m)) & 15; }
static_assert(s64_pos(2) == 3 && s64_pos(3) == 2 && s64_pos(5) == 6 && s64_pos(6) == 5 && s64_a(0) == 2 && s64_a(5) == 4 &&
              s64_a(7) == 2 && s64_b(1) == 5 && s64_b(6) == 3 && s64_b(7) == 1, "N = 64 pair schedule");
// level of the pair in (lane half, block) and whether the lower half's pair is a diagonal one (p = q)
__constant__ int c_s64_level[2][8] = {{4, 5, 0, 2, 3, 4, 6, 3}, {6, 6, 1, 4, 2, 6, 5, 5}};
__constant__ bool c_s64_diag[8] = {true, false, true, true, false, false, true, false};

// Kernel geometry: PR = false -> N = 64 digit stacks; PR = true -> block-pair roles (N = 128 / 256)
template <bool PR>
struct Geo {
  static constexpr int SW = PR ? 16 : 8;                     // split warps
  // N = 64: a dedicated MMA warp. Pairs: no MMA warp (a 17th warp would put 5 warps on one SM
  // sub-partition and cap registers at 96); split warps 0-3, one per sub-partition, issue the
  // MMAs of their accumulator levels ({0, 6}, {1, 5}, {2, 4}, {3}: 8, 8, 8, 4 digit pairs).
  static constexpr int MMA_W = PR ? 0 : SW;                 // warp that allocates TMEM
  static constexpr int NISSUE = PR ? 4 : 1;                 // MMA-issuing threads (commits per tile)
  static constexpr int THREADS = (PR ? SW : SW + 1) * 32;
  static constexpr int NB = PR ? 2 : 1;                      // 64-column blocks per CTA
  static constexpr uint32_t PSTRIDE = PR ? 2 * SLICE : SLICE;  // bytes between digit p and p + 1
  static constexpr uint32_t BUF = NDIG * PSTRIDE;
  static constexpr uint32_t CEX_OFF = 2 * BUF;              // [NB][64 cols][8 groups] u8 exponent fields
  static constexpr uint32_t EXP_OFF = CEX_OFF + NB * CN * 8;  // [NB * 64] int run exponents
  static constexpr uint32_t MISC_OFF = EXP_OFF + NB * CN * 4;
  static constexpr uint32_t BAR_OFF = MISC_OFF + 64;
  // N = 64: the raw fp32 rows of two tiles (cp.async, one tile ahead of the split)
  static constexpr uint32_t XRAW_OFF = (BAR_OFF + 64 + 127) / 128 * 128;
  static constexpr uint32_t XRAW_TILE = KT * CN * 4;
  static constexpr uint32_t SMEM = PR ? BAR_OFF + 64 : XRAW_OFF + 2 * XRAW_TILE;
  static constexpr int FCOLS = CN / (SW / 4);               // flush columns per warp
};
static_assert(Geo<true>::SMEM <= 232448 && Geo<false>::SMEM <= 232448, "shared memory");

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint64_t umax64(uint64_t a, uint64_t b) { return a > b ? a : b; }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" :: "r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile("{\n\t.reg .pred P;\n\tW%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W%=;\n\t}\n"
               :: "r"(su32(b)), "r"(parity) : "memory");
}
template <int SW>
__device__ __forceinline__ void split_sync() { asm volatile("bar.sync 1, %0;" :: "n"(SW * 32) : "memory"); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
constexpr uint32_t DESC_HI = (uint32_t)(((uint64_t)(1024 >> 4) << 32 | (uint64_t)1 << 46 | (uint64_t)2 << 61) >> 32);
// D s32, A and B signed 8-bit, both K-major, N = 64, M = 128
constexpr uint32_t IDESC_I8 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(CN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
__device__ __forceinline__ uint32_t swz(int r, int q) { return (uint32_t)r * 128u + (uint32_t)((q ^ (r & 7)) << 4); }
__device__ __forceinline__ float pow2f(int k) { return __int_as_float((k + 127) << 23); }  // k in [-126, 127]

// The digit bytes of X = rint(x 2^(54 - E)), |x| < 2^E, f1 f2 = 2^(54 - E) (both exact
// power-of-two scalings): low word = d_6 .. d_3 (byte 0 = d_6, the least significant), high
// word = d_2 .. d_0.
__device__ __forceinline__ void digit_bytes(float x, float f1, float f2, uint32_t& zl, uint32_t& zh) {
  const long long X = __float2ll_rn((x * f1) * f2);
  const uint64_t y = (uint64_t)X + 0x0080808080808080ull;
  zl = (uint32_t)y ^ 0x80808080u;
  zh = (uint32_t)(y >> 32) ^ 0x00808080u;
}

struct Seg {  // the CTA's next tile: class f, positions [p0, p0 + rows)
  int f;
  uint64_t p0;
  uint32_t rows;
};

// Role r of the block-pair layout: blocks I != J; `off` = write block (I, J) (and its mirror),
// `diag` = write block (J, J).
struct Role {
  int I, J;
  bool off, diag;
};
__device__ __forceinline__ Role role_of(int n, int r) {
  if (n == 128) return Role{r, 1 - r, r == 0, true};
  constexpr int I[6] = {0, 1, 2, 3, 0, 1}, J[6] = {1, 2, 3, 0, 2, 3};
  return Role{I[r], J[r], true, r < 4};
}
__host__ __device__ constexpr int roles_of(int n) { return n == 64 ? 1 : n == 128 ? 2 : 6; }

template <bool PR>
__global__ void __launch_bounds__(Geo<PR>::THREADS, 1) corr_tc_kernel(const CorrTcParams P) {
  using G = Geo<PR>;
  constexpr int SW = G::SW;
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* cex = sm + G::CEX_OFF;
  int* erun = reinterpret_cast<int*>(sm + G::EXP_OFF);
  volatile int* flag = reinterpret_cast<volatile int*>(sm + G::MISC_OFF);  // [k & 1] flush vote, [2+b] fresh[b]
  uint64_t* a_full = reinterpret_cast<uint64_t*>(sm + G::BAR_OFF);   // [2] split warps -> MMA
  uint64_t* a_empty = a_full + 2;                                     // [2] MMA commit -> split
  uint32_t* tmem_sh = reinterpret_cast<uint32_t*>(a_empty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const int n = P.n;
  const int nroles = roles_of(n);
  const int role_id = PR ? (int)(blockIdx.x % (unsigned)nroles) : 0;
  const Role role = PR ? role_of(n, role_id) : Role{0, 0, true, true};
  const uint64_t beg = (uint64_t)(blockIdx.x / (unsigned)nroles) * P.cta_span;
  const uint64_t end = umin64(beg + P.cta_span, P.count);
  const int C = P.idx ? P.classes : 1;
  auto seg_end = [&](int f) -> uint64_t { return P.idx ? (uint64_t)__ldg(P.seg_end + f) : P.count; };
  auto seg_start = [&](int f) -> uint64_t { return f ? seg_end(f - 1) : 0ull; };
  // first class overlapping [beg, end)
  int f0 = 0;
  if (P.idx) {
    int lo = 0, hi = C;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (seg_end(mid) <= beg) lo = mid + 1; else hi = mid;
    }
    f0 = lo;
  }
  // tile iterator over [beg, end) by class segments (uniform in every thread)
  auto next_tile = [&](int& f, uint64_t& pos, Seg& t) -> bool {
    while (f < C && pos < end) {
      const uint64_t s1 = umin64(seg_end(f), end);
      if (pos < s1) {
        t.f = f;
        t.p0 = pos;
        t.rows = (uint32_t)umin64(KT, s1 - pos);
        pos += t.rows;
        return true;
      }
      ++f;
      pos = umax64(pos, seg_start(f));
    }
    return false;
  };

  if (warp == G::MMA_W) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su32(tmem_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) { mbar_init(&a_full[i], SW); mbar_init(&a_empty[i], G::NISSUE); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_sh;

  // N = 64: MMA issue for tile k in buffer b (the MMA warp's lane 0, once the tile's digits are
  // complete)
  auto issue_mma = [&](uint32_t k) {
    const int b = (int)(k & 1);
    mbar_wait(&a_full[b], (k >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const bool fresh = flag[2 + b] != 0;
    const uint32_t base = su32(sm + b * G::BUF);
    if (P.dbg & 1) goto committed;  // dbg 1 (timing diagnostic): no MMAs
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const uint64_t da = desc_sw128(base + (uint32_t)s64_pos(s64_a(m)) * SLICE);
      const uint64_t db = desc_sw128(base + (uint32_t)s64_pos(s64_b(m)) * SLICE);
      const uint32_t d = tmem + (uint32_t)(m * CN);
#pragma unroll
      for (int j = 0; j < KT / 32; ++j) {
        const uint32_t acc = (fresh && j == 0) ? 0u : 1u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
            :: "r"(d), "l"(da + 2u * j), "l"(db + 2u * j), "r"(IDESC_I8), "r"(acc));
      }
    }
  committed:
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(su32(&a_empty[b])) : "memory");
  };
  // Pairs: issuer warp `is` (converged; one elected lane issues, as in hygt_gemm.cu's elect_one,
  // so the descriptors stay in uniform registers) issues the digit pairs of levels is and 6 - is
  // of tile k: A = stack p, B = digit q of block J.
  auto issue_pr = [&](uint32_t k, int is) {
    const int b = (int)(k & 1);
    mbar_wait(&a_full[b], (k >> 1) & 1);
    __syncwarp();  // lanes leave the wait loop independently
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t leader;
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(leader));
    if (leader) {
      const uint32_t fresh = flag[2 + b] != 0 ? 1u : 0u;
      // descriptor low words (start address >> 4 | LBO); the high word (SBO = 1024 B, version,
      // SWIZZLE_128B) is the constant DESC_HI, joined inside the asm: ptxas 12.9 dropped the high
      // word of 64-bit descriptor arithmetic hoisted into uniform registers here
      const uint32_t lo0 = (uint32_t)desc_sw128(su32(sm + b * G::BUF));
      constexpr uint32_t PST = G::PSTRIDE >> 4, SL = SLICE >> 4;  // descriptor address units
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int L = t ? NDIG - 1 - is : is;
        if (t && L == is) break;
        const uint32_t d = tmem + (uint32_t)(L * CN);
#pragma unroll 1
        for (int pp = 0; pp <= L; ++pp) {
          const uint32_t la = lo0 + (uint32_t)pp * PST, lb = lo0 + (uint32_t)(L - pp) * PST + SL;
          const uint32_t acc = (fresh && pp == 0) ? 0u : 1u;
#pragma unroll
          for (int j = 0; j < KT / 32; ++j)
            asm volatile(
                "{\n\t.reg .pred p;\n\t.reg .b64 da, db;\n\t"
                "mov.b64 da, {%1, %5};\n\tmov.b64 db, {%2, %5};\n\t"
                "setp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], da, db, %3, p;\n\t}\n"
                :: "r"(d), "r"(la + 2u * j), "r"(lb + 2u * j), "r"(IDESC_I8), "r"(j ? 1u : acc), "r"(DESC_HI));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                   :: "r"(su32(&a_empty[b])) : "memory");
    }
    __syncwarp();
  };
  if (!PR && warp == SW) {
    // ---------------------------------------------------------------- MMA issuer ----
    if (lane == 0 && beg < end) {
      int f = f0;
      uint64_t pos = beg < seg_start(f0) ? seg_start(f0) : beg;
      Seg t;
      for (uint32_t k = 0; next_tile(f, pos, t); ++k) issue_mma(k);
    }
  } else {
    // ---------------------------------------------------------------- split warps ----
    const int w = warp;
    const int h = PR ? w >> 3 : 0;           // block of this warp: 0 = I, 1 = J
    const int g = w & 7;                     // 16-row group
    const int col0 = (h ? role.J : role.I) * CN;  // first column of the block in a row
    uint32_t waited[2] = {0u, 0u};  // a_empty completions consumed per buffer
    uint32_t used[2] = {0u, 0u};    // tiles written per buffer
    auto drain = [&](int b) {       // every tile written into buffer b has been multiplied
      while (waited[b] < used[b]) {
        mbar_wait(&a_empty[b], waited[b] & 1);
        ++waited[b];
      }
    };
    int run_class = -1, run_tiles = 0;
    // flush the run's TMEM levels into sum[run_class]: warp w reads lanes 32 (w % 4) + lane,
    // columns FCOLS (w / 4) .. + FCOLS - 1 of every level block.
    //   N = 64: lanes 0-63 hold level L at block L, lanes 64-127 level L at block L - 1, both for
    //           output (i, j) with i = lane mod 64;
    //   pairs:  block L holds level L; lanes 0-63 output block (I, J), lanes 64-127 block (J, J).
    auto flush = [&]() {
      drain(0);
      drain(1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int qd = w & 3, cc = w >> 2;
      const int half = qd >> 1, i = (qd & 1) * 32 + lane;
      const bool write = !PR || (half ? role.diag : role.off);
      if (write) {
        const int ib = PR ? (half ? role.J : role.I) : 0, jb = PR ? role.J : 0;
        const int gi = ib * CN + i;
        double* out = P.sum + ((size_t)run_class * n + gi) * n + jb * CN + cc * G::FCOLS;
        const int ei = erun[(PR && half ? CN : 0) + i];
        const int* ej = erun + (PR ? CN : 0) + cc * G::FCOLS;
#pragma unroll 1
        for (int j0 = 0; j0 < G::FCOLS; j0 += 8) {  // 8 columns at a time (registers)
          double s8[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) s8[j] = 0.0;
#pragma unroll 1
          for (int blk = 0; blk < (PR ? NDIG : 8); ++blk) {
            // pairs: block = level; N = 64: the (block, lane half) slot's level, diagonal pairs halved
            const int L = PR ? blk : (half ? c_s64_level[1][blk] : c_s64_level[0][blk]);
            const double diag = (!PR && !half && c_s64_diag[blk]) ? 0.5 : 1.0;
            uint32_t v[8];
            const uint32_t ta = tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(blk * CN + cc * G::FCOLS + j0);
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                         : "r"(ta));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            const double wl = ldexp(diag, -8 * L);
#pragma unroll
            for (int j = 0; j < 8; ++j) s8[j] = fma((double)(int)v[j], wl, s8[j]);
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (s8[j] == 0.0) continue;
            const double v = ldexp(s8[j], ei + ej[j0 + j] - 12);
            atomicAdd(out + j0 + j, v);
            // mirror: pairs, the off-diagonal block's transpose; N = 64, U^T
            if (!PR || !half) atomicAdd(P.sum + ((size_t)run_class * n + jb * CN + cc * G::FCOLS + j0 + j) * n + gi, v);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      split_sync<SW>();  // TMEM read and erun used before the next run overwrites them
    };

    // Software pipeline: the row ids of tile k + 2 (lane j < 16 holds the id of the warp's row j)
    // and the samples of tile k + 1 are loaded while tile k is quantized, so the dependent
    // id -> address -> sample loads never stall the in-order issue of the current tile.
    int f = f0;
    uint64_t pos = beg < end && beg < seg_start(f0) ? seg_start(f0) : beg;
    Seg tq[3];
    bool hq[3];
    hq[0] = beg < end && next_tile(f, pos, tq[0]);
    hq[1] = hq[0] && next_tile(f, pos, tq[1]);
    hq[2] = hq[1] && next_tile(f, pos, tq[2]);
    // Loads are unconditional (rows past the tile's end read its last row and are masked where
    // the samples are used): a predicated load-or-zero compiles to moves that wait on the loads.
    auto load_ids = [&](const Seg& t, bool have) -> uint32_t {
      if (!have) return 0u;
      const uint32_t rr = min((uint32_t)(g * 16 + (lane & 15)), t.rows - 1u);
      return P.idx ? __ldg(P.idx + t.p0 + rr) : (uint32_t)(t.p0 + rr);
    };
    const char* xb = reinterpret_cast<const char*>(P.x + col0 + lane);
    const uint32_t rowb = (uint32_t)n * 4u;
    auto load_x = [&](uint32_t ids, float (&v)[16][2]) {
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const uint32_t row = __shfl_sync(0xffffffffu, ids, r);
        const float* src = reinterpret_cast<const float*>(xb + (uint64_t)row * rowb);  // IMAD.WIDE.U32
        if constexpr (PR) {  // the other roles' CTAs read these rows too: keep them in L2
          v[r][0] = __ldg(src);
          v[r][1] = __ldg(src + 32);
        } else {
          v[r][0] = __ldcs(src);
          v[r][1] = __ldcs(src + 32);
        }
      }
    };
    // N = 64: the rows go through shared memory instead. Samples held in registers a tile ahead
    // were moved by ptxas right behind their loads (loop-carried register homes), so every tile
    // waited out the DRAM latency there (24 % of the stall samples). The warp copies its 16 rows
    // of tile k + 1 with cp.async (lanes 0-15 one row, lanes 16-31 the next, 16 B each) while it
    // converts tile k, and reads tile k back with conflict-free LDS (lane = column).
    auto stage_rows = [&](uint32_t ids, uint32_t b) {
      const uint32_t dst0 = su32(sm + G::XRAW_OFF) + b * G::XRAW_TILE + (uint32_t)(g * 16 + (lane >> 4)) * (CN * 4u) +
                            (uint32_t)(lane & 15) * 16u;
      const char* src0 = reinterpret_cast<const char*>(P.x) + (lane & 15) * 16;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t row = __shfl_sync(0xffffffffu, ids, 2 * i + (lane >> 4));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                     :: "r"(dst0 + (uint32_t)i * (2u * CN * 4u)), "l"(src0 + (uint64_t)row * (CN * 4u)) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    float va[16][2], vb[16][2];
    uint32_t ida = load_ids(tq[0], hq[0]);
    if constexpr (PR) load_x(ida, va);
    else stage_rows(ida, 0u);
    uint32_t idn = load_ids(tq[1], hq[1]);  // ids of the next tile
    int last_f = -1;
    bool fresh_next = true;
    auto do_tile = [&](const Seg& t, uint32_t k, float (&v)[16][2], float (&vn)[16][2]) {
      // tile k + 1's samples, in flight from here. Unconditional (without a next tile idn = 0 and
      // row 0 is read and never used): under `if (hq[1])` ptxas loaded into temporaries and moved
      // them into vn inside the branch, and those moves waited for the loads (12 % of the kernel's
      // stall samples).
      if constexpr (PR) {
        load_x(idn, vn);
      } else {
        __syncwarp();  // the warp's reads of tile k - 1 (same buffer) are done
        stage_rows(idn, (k + 1u) & 1u);
      }
      idn = load_ids(tq[2], hq[2]);                 // tile k + 2's ids
      if (tid == 0 && role_id == 0 && t.f != last_f) {  // rows of this class in the CTA's range, once
        const uint64_t s1 = umin64(seg_end(t.f), end);
        atomicAdd(P.cnt + t.f, (unsigned long long)(s1 - t.p0));
      }
      last_f = t.f;
      if constexpr (!PR) {  // tile k's rows have landed (all groups but the one just committed)
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncwarp();
        const float* xr = reinterpret_cast<const float*>(sm + G::XRAW_OFF + (k & 1u) * G::XRAW_TILE) + g * 16 * CN + lane;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          v[r][0] = xr[r * CN];
          v[r][1] = xr[r * CN + 32];
        }
      }
      // rows past the tile's end (warp-uniform): zero
      const int nvalid = (int)t.rows - g * 16;
      if (nvalid < 16) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
          if (r >= nvalid) v[r][0] = v[r][1] = 0.f;
      }
      float m0 = 0.f, m1 = 0.f;
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        m0 = fmaxf(m0, fabsf(v[r][0]));
        m1 = fmaxf(m1, fabsf(v[r][1]));
      }
      // the exponent field of the maxima (0 for zero / subnormal), [block][column][group]
      cex[(h * CN + lane) * 8 + g] = (unsigned char)(__float_as_uint(m0) >> 23);
      cex[(h * CN + lane + 32) * 8 + g] = (unsigned char)(__float_as_uint(m1) >> 23);
      if (tid == 0) flag[k & 1] = 0;  // (slot k & 1: the previous tile's readers use the other one)
      split_sync<SW>();
      // smallest E with |x| < 2^E for every sample of the column in this tile
      int et[2];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const uint2 e8 = *reinterpret_cast<const uint2*>(cex + (h * CN + lane + 32 * hh) * 8);
        uint32_t m = __vmaxu4(e8.x, e8.y);
        m = __vmaxu4(m, m >> 16);
        m = max(m & 0xFFu, (m >> 8) & 0xFFu);
        et[hh] = (m ? (int)m : 1) - 126;
      }
      // a new run at a class change, when a column outgrows the run's scale, or for int32 headroom
      const bool change = t.f != run_class || run_tiles >= MAX_RUN_TILES;
      if (!change && g == 0 && (et[0] > erun[h * CN + lane] || et[1] > erun[h * CN + lane + 32])) flag[k & 1] = 1;
      split_sync<SW>();
      if (change || flag[k & 1]) {
        if (run_class >= 0) flush();
        if (g == 0) {  // HEADROOM bits above the tile's maxima: later tiles rarely force a re-base
          const bool keep = !change;  // re-base: the run's scale only grows
          int* e = erun + h * CN;
          e[lane] = keep ? max(e[lane], et[0] + HEADROOM) : et[0] + HEADROOM;
          e[lane + 32] = keep ? max(e[lane + 32], et[1] + HEADROOM) : et[1] + HEADROOM;
        }
        run_class = t.f;
        run_tiles = 0;
        fresh_next = true;
        split_sync<SW>();
      }
      ++run_tiles;
      // digits into buffer b (free once its previous tile was multiplied)
      const int b = (int)(k & 1);
      drain(b);
      if (tid == 0) flag[2 + b] = fresh_next ? 1 : 0;
      fresh_next = false;
      unsigned char* buf = sm + b * G::BUF + (PR ? h * SLICE : 0);
#pragma unroll
      for (int hh = 0; hh < ((P.dbg & 2) ? 0 : 2); ++hh) {  // dbg 2 (timing diagnostic): no digits
        const int col = lane + 32 * hh;
        // 2^(54 - E) as two exact factors (E in [-125, 131])
        const int a = 54 - erun[h * CN + col], a1 = a >> 1;
        const float f1 = pow2f(a1), f2 = pow2f(a - a1);
        // z[r]: the 7 digit bytes of row r (byte 0 = d_6, the least significant); RC rows at a
        // time (RC = 8 in the block-pair layout keeps 17 warps within 96 registers)
        constexpr int RC = PR ? 8 : 16;
#pragma unroll
        for (int r0 = 0; r0 < 16; r0 += RC) {
          uint32_t zl[RC], zh[RC];
#pragma unroll
          for (int r = 0; r < RC; ++r) digit_bytes(v[r0 + r][hh], f1, f2, zl[r], zh[r]);
          // digit p = byte 6 - p: gather it from 4 rows per 32-bit word (PRMT)
#pragma unroll
          for (int p = 0; p < NDIG; ++p) {
            const int bsel = 6 - p, kk = bsel & 3;
            const uint32_t s01 = (uint32_t)(kk | ((4 + kk) << 4));
            uint32_t q[RC / 4];
#pragma unroll
            for (int gg = 0; gg < RC / 4; ++gg) {
              const uint32_t a0 = bsel < 4 ? zl[4 * gg] : zh[4 * gg], a1w = bsel < 4 ? zl[4 * gg + 1] : zh[4 * gg + 1];
              const uint32_t a2 = bsel < 4 ? zl[4 * gg + 2] : zh[4 * gg + 2], a3 = bsel < 4 ? zl[4 * gg + 3] : zh[4 * gg + 3];
              q[gg] = __byte_perm(__byte_perm(a0, a1w, s01), __byte_perm(a2, a3, s01), 0x5410);
            }
            unsigned char* dst = buf + (uint32_t)(PR ? p : s64_pos(p)) * G::PSTRIDE + swz(col, g) + (uint32_t)r0;
            if constexpr (RC == 16) *reinterpret_cast<uint4*>(dst) = make_uint4(q[0], q[1], q[2], q[3]);
            else *reinterpret_cast<uint2*>(dst) = make_uint2(q[0], q[1]);
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      ++used[b];
      if (lane == 0) mbar_arrive(&a_full[b]);
      if (PR && w < G::NISSUE) issue_pr(k, w);
    };
    auto advance = [&]() {
      tq[0] = tq[1];
      hq[0] = hq[1];
      tq[1] = tq[2];
      hq[1] = hq[2];
      hq[2] = hq[1] && next_tile(f, pos, tq[2]);
    };
    // unrolled by two so that each call site works on fixed registers (no buffer selects)
    for (uint32_t k = 0; hq[0]; k += 2) {
      do_tile(tq[0], k, va, vb);
      advance();
      if (!hq[0]) break;
      do_tile(tq[0], k + 1, vb, va);
      advance();
    }
    if (run_class >= 0) flush();
    if constexpr (!PR) asm volatile("cp.async.wait_all;" ::: "memory");  // the look-ahead copy past the last tile
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == G::MMA_W) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem));
}

}  // namespace

bool corr_tc_supported(int log2n) { return log2n >= 6 && log2n <= 8; }

int corr_tc_run(const CorrTcParams& P, int sms, cudaStream_t st) {
  CorrTcParams Q = P;
  const int roles = roles_of(P.n);
  // row ranges: one CTA per SM and role; the roles of a range walk the same rows together
  const uint64_t ranges = std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)std::max(1, sms / roles),
                                                                     (P.count + KT - 1) / KT));
  Q.cta_span = (P.count + ranges - 1) / ranges;
  const unsigned ctas = (unsigned)(ranges * (uint64_t)roles);
  if (P.n == 64) {
    hygt_smem_attr(reinterpret_cast<const void*>(corr_tc_kernel<false>), Geo<false>::SMEM);
    corr_tc_kernel<false><<<ctas, Geo<false>::THREADS, Geo<false>::SMEM, st>>>(Q);
  } else {
    hygt_smem_attr(reinterpret_cast<const void*>(corr_tc_kernel<true>), Geo<true>::SMEM);
    corr_tc_kernel<true><<<ctas, Geo<true>::THREADS, Geo<true>::SMEM, st>>>(Q);
  }
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HYGT_OK : hygt_set_error(HYGT_ERR_CUDA, cudaGetErrorString(e));
}

}  // namespace hygt_gpu
