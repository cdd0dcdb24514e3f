// hygt_corr_tc.cu -- per-class second moments sum_c += r r^T (SURVEY.md §8 f3,
// CorrelationAccumulator::add, statistics.hpp:63-99) on the 5th-generation tensor cores, N = 64.
//
// Exactness. The reference accumulates r_i r_j in fp64, and fp32 samples make every product exact
// there; the parity bar is 1e-12 of the largest sum. Floating-point tensor-core inputs cannot
// carry that, integers can: within a run of tiles of one class, column i of every row is taken to
// fixed point relative to a per-column power of two 2^E_i > max |r_i| (X = r 2^(54 - E_i),
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
// Layout (one CTA per SM, tiles of 128 bucketed rows of one class):
//   warps 0-7  split: lane l holds columns l and l + 32 of 16 rows; per-column tile maxima
//              (shared-memory reduction), the run's exponents, the digits; digit p of column i
//              is row i of slice p, K = the tile's 128 rows, SWIZZLE_128B K-major (one 16 B chunk
//              per warp and column); slices 0..6 plus a zero slice 7, double-buffered. They also
//              flush: warp w reads TMEM lane quadrant w % 4, columns 32 (w / 4) .. + 31.
//   warp 8     MMA: one thread issues M = 128 (slices p, p + 1 stacked) x N = 64 (slice q) x
//              K = 32 int8 MMAs, 16 stacks x 4 K steps per tile: rows 0-63 of a stack's result
//              are (p, q) at level p + q, rows 64-127 are (p + 1, q) at level p + q + 1, both
//              written to column block p + q (lanes 64-127 hold level L at block L - 1).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../../include/hygt_gpu.h"
#include "hygt_corr_tc.h"

int hygt_set_error(int status, const char* msg);  // hygt_capi.cu
void hygt_smem_attr(const void* fn, size_t bytes);

namespace hygt_gpu {
namespace {

constexpr int CN = 64;             // samples per row
constexpr int KT = 128;            // rows per tile (MMA K)
constexpr int NDIG = 7;            // digits per sample
constexpr int SLOTS = 8;           // digit slices per buffer (slot 7 stays zero)
constexpr int SPLIT_W = 8;
constexpr int MMA_W = SPLIT_W;
constexpr int THREADS = (SPLIT_W + 1) * 32;
constexpr uint32_t SLICE = CN * 128;          // 64 rows x 128 B (K = 128 int8)
constexpr uint32_t BUF = SLOTS * SLICE;       // 64 KB
constexpr uint32_t CMAX_OFF = 2 * BUF;        // [8][64] float column maxima
constexpr uint32_t EXP_OFF = CMAX_OFF + SPLIT_W * CN * 4;  // [64] int run exponents
constexpr uint32_t MISC_OFF = EXP_OFF + CN * 4;            // flags
constexpr uint32_t BAR_OFF = MISC_OFF + 64;
constexpr uint32_t SMEM = BAR_OFF + 64;
constexpr int MAX_RUN_TILES = 128;
constexpr int HEADROOM = 2;  // bits of a run's exponents above the first tile's column maxima  // int32 headroom: |D_L| <= 7 * 128 * 128^2 per tile < 2^31 / 146

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
__device__ __forceinline__ void split_sync() { asm volatile("bar.sync 1, %0;" :: "n"(SPLIT_W * 32) : "memory"); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// D s32, A and B signed 8-bit, both K-major, N = 64, M = 128
constexpr uint32_t IDESC_I8 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(CN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
__device__ __forceinline__ uint32_t swz(int r, int q) { return (uint32_t)r * 128u + (uint32_t)((q ^ (r & 7)) << 4); }

// smallest E with |m| < 2^E (m > 0, finite); 0 -> a very small exponent
__device__ __forceinline__ int exp_above(float m) {
  if (!(m > 0.f)) return -160;
  const int e = (int)(__float_as_uint(m) >> 23);  // biased; 0 for subnormals
  return e == 0 ? -126 : e - 126;
}
// X = round(x 2^(54 - E)) as int64, |x| < 2^E, integer arithmetic on the fp32 fields
__device__ __forceinline__ long long fixed_of(float x, int E) {
  const uint32_t u = __float_as_uint(x);
  const int ex = (int)((u >> 23) & 0xFFu);
  const long long mant = (long long)((u & 0x7FFFFFu) | (ex ? 0x800000u : 0u));
  const int s = (ex ? ex : 1) - 96 - E;  // x = mant 2^(ex - 150): X = mant 2^(ex - 150 + 54 - E)
  long long m;
  if (s >= 0) m = mant << s;                          // s <= 30
  else if (s > -40) m = (mant + (1ll << (-s - 1))) >> (-s);
  else m = 0;
  return (u >> 31) ? -m : m;
}

// The balanced base-256 digits of X = round(x 2^(54 - E)) are the bytes of (X + C) ^ C with
// C = 0x80 in each of the 7 bytes: X + C = sum (d_p + 128) 256^(6-p), each d_p + 128 in
// [0, 255], and XOR 0x80 maps that byte to d_p as a signed 8-bit value. Returns the low and the
// high (3 bytes) words.
__device__ __forceinline__ void digit_bytes(float x, int E, uint32_t& zl, uint32_t& zh) {
  const uint32_t u = __float_as_uint(x);
  const int ex = (int)((u >> 23) & 0xFFu);
  const uint32_t mant = (u & 0x7FFFFFu) | (ex ? 0x800000u : 0u);
  const int s = (ex ? ex : 1) - 96 - E;  // |x| < 2^E: s <= 30
  // signed mantissa, then a 64-bit shift of the signed value (funnel shift over its sign word)
  int32_t m = (int32_t)mant;
  if (s < 0) m = s > -32 ? (int32_t)((mant + (1u << (-s - 1))) >> (-s)) : 0;  // rare: tiny samples
  const int32_t ms = (u >> 31) ? -m : m;
  const uint32_t sh = s > 0 ? (uint32_t)s : 0u;
  const uint32_t lo = (uint32_t)ms << sh;
  const uint32_t hi = __funnelshift_l((uint32_t)ms, (uint32_t)(ms >> 31), sh);
  const uint64_t y = (((uint64_t)hi << 32) | lo) + 0x0080808080808080ull;
  zl = (uint32_t)y ^ 0x80808080u;
  zh = (uint32_t)(y >> 32) ^ 0x00808080u;
}

struct Seg {  // the CTA's next tile: class f, positions [p0, p0 + rows)
  int f;
  uint64_t p0;
  uint32_t rows;
};

__global__ void __launch_bounds__(THREADS, 1) corr_tc_kernel(const CorrTcParams P) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* cmax = reinterpret_cast<float*>(sm + CMAX_OFF);
  int* erun = reinterpret_cast<int*>(sm + EXP_OFF);
  volatile int* flag = reinterpret_cast<volatile int*>(sm + MISC_OFF);  // [k & 1] flush vote, [2+b] fresh[b]
  uint64_t* a_full = reinterpret_cast<uint64_t*>(sm + BAR_OFF);   // [2] split warps -> MMA
  uint64_t* a_empty = a_full + 2;                                   // [2] MMA commit -> split
  uint32_t* tmem_sh = reinterpret_cast<uint32_t*>(a_empty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const uint64_t beg = (uint64_t)blockIdx.x * P.cta_span;
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

  if (warp == MMA_W) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su32(tmem_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (uint32_t i = tid; i < 2 * SLICE / 16; i += THREADS) {  // the zero slice 7 of both buffers
    const uint32_t b = i / (SLICE / 16), o = i % (SLICE / 16);
    reinterpret_cast<uint4*>(sm + b * BUF + 7 * SLICE)[o] = make_uint4(0u, 0u, 0u, 0u);
  }
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) { mbar_init(&a_full[i], SPLIT_W); mbar_init(&a_empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_sh;

  // MMA issue for tile k in buffer b (warp 0, lane 0, once the tile's digits are complete)
  auto issue_mma = [&](uint32_t k) {
    const int b = (int)(k & 1);
    mbar_wait(&a_full[b], (k >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const bool fresh = flag[2 + b] != 0;
    const uint32_t base = su32(sm + b * BUF);
    uint32_t touched = 0;
#pragma unroll 1
    for (int q = 0; q < NDIG; ++q)
#pragma unroll 1
      for (int p0 = 0; p0 + q <= NDIG - 1; p0 += 2) {
        const int blk = p0 + q;
        const uint64_t da = desc_sw128(base + (uint32_t)p0 * SLICE), db = desc_sw128(base + (uint32_t)q * SLICE);
        const uint32_t d = tmem + (uint32_t)(blk * CN);
#pragma unroll
        for (int j = 0; j < KT / 32; ++j) {
          const uint32_t acc = (fresh && !(touched >> blk & 1u) && j == 0) ? 0u : 1u;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
              :: "r"(d), "l"(da + 2u * j), "l"(db + 2u * j), "r"(IDESC_I8), "r"(acc));
        }
        touched |= 1u << blk;
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(su32(&a_empty[b])) : "memory");
  };
  if (warp == MMA_W) {
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
    // columns 32 (w / 4) .. + 31 of every block; lanes 0-63 hold level L at block L, lanes 64-127
    // level L at block L - 1
    auto flush = [&]() {
      drain(0);
      drain(1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int qd = w & 3, ch = w >> 2;
      const int half = qd >> 1, i = (qd & 1) * 32 + lane;
      double* out = P.sum + ((size_t)run_class * CN + i) * CN + ch * 32;
      const int ei = erun[i];
#pragma unroll 1
      for (int j0 = 0; j0 < 32; j0 += 8) {  // 8 columns at a time (registers)
        double s8[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) s8[j] = 0.0;
#pragma unroll 1
        for (int blk = 0; blk < NDIG; ++blk) {
          const int L = blk + half;
          if (L > NDIG - 1) break;
          uint32_t v[8];
          const uint32_t ta = tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(blk * CN + ch * 32 + j0);
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                       : "r"(ta));
          asm volatile("tcgen05.wait::ld.sync.aligned;");
          const double wl = ldexp(1.0, -8 * L);
#pragma unroll
          for (int j = 0; j < 8; ++j) s8[j] = fma((double)(int)v[j], wl, s8[j]);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (s8[j] != 0.0) atomicAdd(out + j0 + j, ldexp(s8[j], ei + erun[ch * 32 + j0 + j] - 12));
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      split_sync();  // TMEM read and erun used before the next run overwrites them
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
      const uint32_t rr = min((uint32_t)(w * 16 + (lane & 15)), t.rows - 1u);
      return P.idx ? __ldg(P.idx + t.p0 + rr) : (uint32_t)(t.p0 + rr);
    };
    auto load_x = [&](uint32_t ids, float (&v)[16][2]) {
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const uint32_t row = __shfl_sync(0xffffffffu, ids, r);
        const float* src = P.x + (uint64_t)row * CN;
        v[r][0] = __ldcs(src + lane);
        v[r][1] = __ldcs(src + lane + 32);
      }
    };
    float va[16][2], vb[16][2];
    uint32_t ida = load_ids(tq[0], hq[0]);
    load_x(ida, va);
    uint32_t idn = load_ids(tq[1], hq[1]);  // ids of the next tile
    int last_f = -1;
    bool fresh_next = true;
    auto do_tile = [&](const Seg& t, uint32_t k, float (&v)[16][2], float (&vn)[16][2]) {
      if (hq[1]) load_x(idn, vn);                   // tile k + 1's samples, in flight from here
      idn = load_ids(tq[2], hq[2]);                 // tile k + 2's ids
      if (tid == 0 && t.f != last_f) {  // rows of this class in the CTA's range, once per class
        const uint64_t s1 = umin64(seg_end(t.f), end);
        atomicAdd(P.cnt + t.f, (unsigned long long)(s1 - t.p0));
      }
      last_f = t.f;
      // rows past the tile's end (warp-uniform): zero
      const int nvalid = (int)t.rows - w * 16;
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (r >= nvalid) v[r][0] = v[r][1] = 0.f;
      float m0 = 0.f, m1 = 0.f;
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        m0 = fmaxf(m0, fabsf(v[r][0]));
        m1 = fmaxf(m1, fabsf(v[r][1]));
      }
      cmax[w * CN + lane] = m0;
      cmax[w * CN + lane + 32] = m1;
      if (tid == 0) flag[k & 1] = 0;  // (slot k & 1: the previous tile's readers use the other one)
      split_sync();
      int et[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float m = 0.f;
        for (int ww = 0; ww < SPLIT_W; ++ww) m = fmaxf(m, cmax[ww * CN + lane + 32 * h]);
        et[h] = exp_above(m);
      }
      // a new run at a class change, when a column outgrows the run's scale, or for int32 headroom
      const bool change = t.f != run_class || run_tiles >= MAX_RUN_TILES;
      if (!change && w == 0 && (et[0] > erun[lane] || et[1] > erun[lane + 32])) flag[k & 1] = 1;
      split_sync();
      if (change || flag[k & 1]) {
        if (run_class >= 0) flush();
        if (w == 0) {  // HEADROOM bits above the tile's maxima: later tiles rarely force a re-base
          const bool keep = !change;  // re-base: the run's scale only grows
          erun[lane] = keep ? max(erun[lane], et[0] + HEADROOM) : et[0] + HEADROOM;
          erun[lane + 32] = keep ? max(erun[lane + 32], et[1] + HEADROOM) : et[1] + HEADROOM;
        }
        run_class = t.f;
        run_tiles = 0;
        fresh_next = true;
        split_sync();
      }
      ++run_tiles;
      // digits into buffer b (free once its previous tile was multiplied)
      const int b = (int)(k & 1);
      drain(b);
      if (tid == 0) flag[2 + b] = fresh_next ? 1 : 0;
      fresh_next = false;
      unsigned char* buf = sm + b * BUF;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = lane + 32 * h;
        const int E = erun[col];
        // z[r]: the 7 digit bytes of row r (byte 0 = d_6, the least significant)
        uint32_t zl[16], zh[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) digit_bytes(v[r][h], E, zl[r], zh[r]);
        // digit p = byte 6 - p: gather it from 4 rows per 32-bit word (PRMT), 16 rows per chunk
#pragma unroll
        for (int p = 0; p < NDIG; ++p) {
          const int bsel = 6 - p, k = bsel & 3;
          const uint32_t s01 = (uint32_t)(k | ((4 + k) << 4));
          uint32_t q[4];
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const uint32_t a0 = bsel < 4 ? zl[4 * g] : zh[4 * g], a1 = bsel < 4 ? zl[4 * g + 1] : zh[4 * g + 1];
            const uint32_t a2 = bsel < 4 ? zl[4 * g + 2] : zh[4 * g + 2], a3 = bsel < 4 ? zl[4 * g + 3] : zh[4 * g + 3];
            q[g] = __byte_perm(__byte_perm(a0, a1, s01), __byte_perm(a2, a3, s01), 0x5410);
          }
          *reinterpret_cast<uint4*>(buf + (uint32_t)p * SLICE + swz(col, w)) = make_uint4(q[0], q[1], q[2], q[3]);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      ++used[b];
      if (lane == 0) mbar_arrive(&a_full[b]);

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
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == MMA_W) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem));
}

}  // namespace

bool corr_tc_supported(int log2n) { return log2n == 6; }

int corr_tc_run(const CorrTcParams& P, int sms, cudaStream_t st) {
  hygt_smem_attr(reinterpret_cast<const void*>(corr_tc_kernel), SMEM);
  CorrTcParams Q = P;
  const uint64_t ctas = std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)sms, (P.count + KT - 1) / KT));
  Q.cta_span = (P.count + ctas - 1) / ctas;
  corr_tc_kernel<<<(unsigned)ctas, THREADS, SMEM, st>>>(Q);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HYGT_OK : hygt_set_error(HYGT_ERR_CUDA, cudaGetErrorString(e));
}

}  // namespace hygt_gpu
