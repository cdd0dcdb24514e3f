// hygt_klt.cu -- dense per-class KLT comparison path (BASELINE config 4):
//   forward  y = K_c x   (klt_forward, statistics.hpp:222-224 -> multiply, matrix.hpp:70-80)
//   inverse  x = K_c^T y (transposed, matrix.hpp:82-88)
//
// B200 design: rows are bucketed by class (the same bucketing as the HyGT path), then each
// class is a GEMM  OUT[m][n] = sum_k IN[m][k] * B[n][k]  with B = K_c (forward) or K_c^T
// (inverse), M = rows of the class, N = K = n. It runs on the 5th-generation tensor cores:
// tcgen05.mma kind::tf32, M=128 x N=n per instruction, accumulators in TMEM, issued by one
// thread. fp32 accuracy comes from the 3xTF32 split (x = hi + lo, both rounded to tf32;
// D = A_hi B_hi + A_hi B_lo + A_lo B_hi, fp32 accumulation), which meets the 1e-6 relative-L2
// bar that plain TF32 (~1e-3) does not. Operand tiles use the canonical K-major no-swizzle
// layout (8-row x 16-byte core matrices): a warp's 32 rows store one 512-byte run per chunk,
// so the shared-memory fill is bank-conflict free. The epilogue drains TMEM with
// tcgen05.ld.32x32b (one row per thread) and stores the row back to its original position.
// n in {16, 32, 64} uses the tensor cores; other n use the fp32 SIMT kernel.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hygt_gpu.h"

int hygt_set_error(int status, const char* msg);  // hygt_capi.cu
void hygt_smem_attr(const void* fn, size_t bytes);  // hygt_capi.cu: per (device, kernel), only grows
namespace hygt_gpu {
size_t bucket_ws_bytes(int classes, uint64_t chunk_rows, uint64_t count);
int bucket_rows(int classes, uint64_t chunk_rows, const uint16_t* d_cls, uint64_t count,
                void* d_ws, size_t ws_bytes, bool run, cudaStream_t st, const uint32_t** idx,
                const uint32_t** seg_end, uint32_t* nseg);
}  // namespace hygt_gpu

struct hygt_klt_plan {
  int n = 0, classes = 0;
  float* d_k = nullptr;   // [C][n][n]   rows = basis vectors (fp32)
  float* d_kt = nullptr;  // [C][n][n]   transposed
  float* d_b[2] = {nullptr, nullptr};  // tensor-core B operands per direction: [C][hi|lo][layout]
  float* d_bsw[2] = {nullptr, nullptr};  // the same in the SWIZZLE_128B layout (n = 64)
  bool tc = false;
  int num_sms = 148;
};

namespace {
int kfail(int st, const std::string& m) { return hygt_set_error(st, m.c_str()); }

// ------------------------------------------------------------------ fp32 SIMT fallback ----
constexpr int KT = 256;

__global__ void __launch_bounds__(KT) klt_simt_kernel(const float* __restrict__ in, float* out,
                                                      const uint16_t* __restrict__ cls,
                                                      uint64_t count, int n, int classes,
                                                      const float* __restrict__ mt) {
  extern __shared__ float xs[];
  const int rows_per_cta = KT / n;
  const int rl = threadIdx.x / n, i = threadIdx.x % n;
  for (uint64_t r0 = (uint64_t)blockIdx.x * rows_per_cta; r0 < count;
       r0 += (uint64_t)gridDim.x * rows_per_cta) {
    __syncthreads();
    for (int k = threadIdx.x; k < rows_per_cta * n; k += KT) {
      const uint64_t r = r0 + k / n;
      xs[k] = r < count ? in[r * n + (k % n)] : 0.f;
    }
    __syncthreads();
    const uint64_t r = r0 + rl;
    if (rl < rows_per_cta && r < count) {
      int c = cls ? cls[r] : 0;
      if (c >= classes) c = 0;
      const float* m = mt + (size_t)c * n * n;
      const float* xv = xs + rl * n;
      float acc = 0.f;
      for (int j = 0; j < n; ++j) acc = fmaf(__ldg(m + (size_t)j * n + i), xv[j], acc);
      out[r * n + i] = acc;
    }
  }
}

// ------------------------------------------------------------------ tcgen05 kernel --------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// Canonical K-major, no-swizzle operand layout (cute UMMA Layout_K_INTER): element (r, k) of an
// R x K tile at byte (k/4)*(R*16) + (r/8)*128 + (r%8)*16 + (k%4)*4 -> SBO = 128 B between
// 8-row groups, LBO = R*16 B between the two 4-wide K core matrices of one K=8 instruction.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  // base offset 0, lbo mode 0, layout type 0 (SWIZZLE_NONE)
  return d;
}
// Instruction descriptor: D f32, A/B tf32, both K-major, N = n, M = 128.
__host__ __device__ constexpr uint32_t idesc_tf32(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

struct KltTcParams {
  const float* in;
  float* out;
  const uint32_t* idx;      // bucketed position -> row (nullptr: identity, one class)
  const uint32_t* seg_end;  // [C+1] run ends (one chunk)
  int classes;
  uint64_t count;
  const float* b;           // [C][2][n*n] B operands (hi, lo) already in the canonical layout
};

template <int NN>
__global__ void __launch_bounds__(128, 1) klt_tc_kernel(const KltTcParams P) {
  constexpr int M = 128;
  constexpr int KCH = NN / 4;                     // 16-byte K chunks per row
  constexpr uint32_t TMEM_COLS = NN < 32 ? 32 : NN;
  constexpr uint32_t A_BYTES = M * NN * 4, B_BYTES = NN * NN * 4;
  extern __shared__ __align__(1024) unsigned char sm[];
  float* a_hi = reinterpret_cast<float*>(sm);
  float* a_lo = reinterpret_cast<float*>(sm + A_BYTES);
  float* b_hi = reinterpret_cast<float*>(sm + 2 * A_BYTES);
  float* b_lo = reinterpret_cast<float*>(sm + 2 * A_BYTES + B_BYTES);
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5;

  if (warp == 0) {  // TMEM allocation (one warp), then give up the permit for co-resident CTAs
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(&tmem_base_sh)), "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_sh;
  uint32_t phase = 0;

  const int C = P.idx ? P.classes : 1;
  // Work items: 128-row tiles of each class run, distributed over the grid class by class.
  for (int c = 0; c < C; ++c) {
    const uint64_t s0 = P.idx ? (c == 0 ? 0 : P.seg_end[c - 1]) : 0;
    const uint64_t s1 = P.idx ? P.seg_end[c] : P.count;
    if (s1 <= s0) continue;
    const uint64_t tiles = (s1 - s0 + M - 1) / M;
    if (tiles <= blockIdx.x) continue;
    // stage this class's B operand (hi and lo, canonical layout, prepared on the host)
    __syncthreads();
    {
      const float4* src = reinterpret_cast<const float4*>(P.b + (size_t)c * 2 * NN * NN);
      float4* dst = reinterpret_cast<float4*>(b_hi);
      for (int i = tid; i < 2 * NN * NN / 4; i += 128) dst[i] = __ldg(src + i);
    }
    for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
      const uint64_t p = s0 + t * M + tid;
      const bool valid = p < s1;
      const uint64_t row = valid ? (P.idx ? (uint64_t)__ldg(P.idx + p) : p) : 0;
      // A tile: thread tid owns row tid of the tile; split into tf32 hi + lo
      const float4* src = reinterpret_cast<const float4*>(P.in + row * NN);
#pragma unroll
      for (int q = 0; q < KCH; ++q) {
        float4 v = valid ? __ldg(src + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 h = make_float4(to_tf32(v.x), to_tf32(v.y), to_tf32(v.z), to_tf32(v.w));
        float4 l = make_float4(to_tf32(v.x - h.x), to_tf32(v.y - h.y), to_tf32(v.z - h.z), to_tf32(v.w - h.w));
        const int off = q * (M * 4) + (tid >> 3) * 32 + (tid & 7) * 4;  // floats
        *reinterpret_cast<float4*>(a_hi + off) = h;
        *reinterpret_cast<float4*>(a_lo + off) = l;
      }
      asm volatile("fence.proxy.async.shared::cta;");  // generic-proxy stores -> tensor core reads
      __syncthreads();
      if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t idesc = idesc_tf32(NN);
        const uint32_t ahi = smem_u32(a_hi), alo = smem_u32(a_lo);
        const uint32_t bhi = smem_u32(b_hi), blo = smem_u32(b_lo);
        int first = 1;
#pragma unroll
        for (int ks = 0; ks < NN / 8; ++ks) {
          const uint32_t aoff = (uint32_t)(2 * ks) * (M * 16), boff = (uint32_t)(2 * ks) * (NN * 16);
          const uint64_t da_hi = umma_desc(ahi + aoff, M * 16, 128), da_lo = umma_desc(alo + aoff, M * 16, 128);
          const uint64_t db_hi = umma_desc(bhi + boff, NN * 16, 128), db_lo = umma_desc(blo + boff, NN * 16, 128);
          const uint64_t da[3] = {da_lo, da_hi, da_hi}, db[3] = {db_hi, db_lo, db_hi};  // small terms first
#pragma unroll
          for (int term = 0; term < 3; ++term) {
            const uint32_t acc = first ? 0u : 1u;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                :: "r"(tmem), "l"(da[term]), "l"(db[term]), "r"(idesc), "r"(acc));
            first = 0;
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     :: "r"(smem_u32(&mbar)));
      }
      // wait for the MMAs (mbarrier phase flip)
      asm volatile(
          "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra WAIT_%=;\n\t}\n"
          :: "r"(smem_u32(&mbar)), "r"(phase));
      phase ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;");
      // epilogue: row tid of the accumulator = TMEM lane tid (warp w owns lanes 32w..32w+31)
      float* dst = P.out + row * NN;
#pragma unroll
      for (int c0 = 0; c0 < NN; c0 += 16) {
        uint32_t r[16];
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
              "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        if (valid) {
#pragma unroll
          for (int j = 0; j < 16; j += 4)
            __stcs(reinterpret_cast<float4*>(dst + c0 + j),
                   make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                               __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3])));
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();  // A tiles and TMEM free for the next tile
      asm volatile("tcgen05.fence::after_thread_sync;");
    }
  }
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(TMEM_COLS));
}

// Pipelined variant for N = 64 (config 4): 8 warps, two A stages and two TMEM accumulators, so
// the global gathers + tf32 split of tile i+1 overlap the tensor-core MMAs of tile i, and the
// epilogue of tile i overlaps the MMAs of tile i+1. Two threads per tile row (each half of the K
// chunks when loading, half of the accumulator columns when draining).
constexpr int KLT_PIPE_THREADS = 256;

template <int NN>
__global__ void __launch_bounds__(KLT_PIPE_THREADS, 1) klt_tc_pipe_kernel(const KltTcParams P) {
  constexpr int M = 128;
  constexpr int KCH = NN / 4;
  constexpr uint32_t A_BYTES = M * NN * 4, B_BYTES = NN * NN * 4;
  static_assert(NN == 64, "pipelined KLT kernel: N = 64");
  extern __shared__ __align__(1024) unsigned char sm[];
  auto a_st = [&](int st, int lo) { return reinterpret_cast<float*>(sm + (2 * st + lo) * A_BYTES); };
  float* b_hi = reinterpret_cast<float*>(sm + 4 * A_BYTES);
  float* b_lo = reinterpret_cast<float*>(sm + 4 * A_BYTES + B_BYTES);
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int trow = tid & (M - 1), half = tid / M;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(&tmem_base_sh)), "r"(2u * NN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&mbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&mbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_sh;
  uint32_t phase[2] = {0, 0};

  auto load_tile = [&](uint64_t s0, uint64_t s1, uint64_t t, int st) -> uint64_t {
    const uint64_t p = s0 + t * M + trow;
    const bool valid = p < s1;
    const uint64_t row = valid ? (P.idx ? (uint64_t)__ldg(P.idx + p) : p) : ~0ull;
    const float4* src = reinterpret_cast<const float4*>(P.in + (valid ? row : 0) * NN);
    float4 v[KCH / 2];
#pragma unroll
    for (int qq = 0; qq < KCH / 2; ++qq)
      v[qq] = valid ? __ldcs(src + half * (KCH / 2) + qq) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int qq = 0; qq < KCH / 2; ++qq) {
      const int q = half * (KCH / 2) + qq;
      const float4 h = make_float4(to_tf32(v[qq].x), to_tf32(v[qq].y), to_tf32(v[qq].z), to_tf32(v[qq].w));
      const float4 l = make_float4(to_tf32(v[qq].x - h.x), to_tf32(v[qq].y - h.y), to_tf32(v[qq].z - h.z),
                                   to_tf32(v[qq].w - h.w));
      const int off = q * (M * 4) + (trow >> 3) * 32 + (trow & 7) * 4;  // canonical K-major
      *reinterpret_cast<float4*>(a_st(st, 0) + off) = h;
      *reinterpret_cast<float4*>(a_st(st, 1) + off) = l;
    }
    asm volatile("fence.proxy.async.shared::cta;");
    return row;
  };
  auto issue = [&](int st) {  // one thread: 3xTF32 MMAs of a 128 x NN tile into accumulator st
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t idesc = idesc_tf32(NN);
    const uint32_t ahi = smem_u32(a_st(st, 0)), alo = smem_u32(a_st(st, 1));
    const uint32_t bhi = smem_u32(b_hi), blo = smem_u32(b_lo);
    const uint32_t d = tmem + (uint32_t)(st * NN);
    int first = 1;
#pragma unroll
    for (int ks = 0; ks < NN / 8; ++ks) {
      const uint32_t aoff = (uint32_t)(2 * ks) * (M * 16), boff = (uint32_t)(2 * ks) * (NN * 16);
      const uint64_t da_hi = umma_desc(ahi + aoff, M * 16, 128), da_lo = umma_desc(alo + aoff, M * 16, 128);
      const uint64_t db_hi = umma_desc(bhi + boff, NN * 16, 128), db_lo = umma_desc(blo + boff, NN * 16, 128);
      const uint64_t da[3] = {da_lo, da_hi, da_hi}, db[3] = {db_hi, db_lo, db_hi};  // small terms first
#pragma unroll
      for (int term = 0; term < 3; ++term) {
        const uint32_t acc = first ? 0u : 1u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
            :: "r"(d), "l"(da[term]), "l"(db[term]), "r"(idesc), "r"(acc));
        first = 0;
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(smem_u32(&mbar[st])));
  };
  auto wait_mma = [&](int st) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra WAIT_%=;\n\t}\n"
        :: "r"(smem_u32(&mbar[st])), "r"(phase[st]));
    phase[st] ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;");
  };
  auto drain = [&](int st, uint64_t row) {  // accumulator st -> rows (half of the columns each)
    float* dst = P.out + row * NN;
#pragma unroll
    for (int c1 = 0; c1 < NN / 2; c1 += 16) {
      const int c0 = half * (NN / 2) + c1;
      uint32_t r[16];
      const uint32_t taddr = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(st * NN + c0);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
            "=r"(r[14]), "=r"(r[15])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      if (row != ~0ull) {
#pragma unroll
        for (int j = 0; j < 16; j += 4)
          __stcs(reinterpret_cast<float4*>(dst + c0 + j),
                 make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                             __uint_as_float(r[j + 3])));
      }
    }
  };

  const int C = P.idx ? P.classes : 1;
  for (int c = 0; c < C; ++c) {
    const uint64_t s0 = P.idx ? (c == 0 ? 0 : P.seg_end[c - 1]) : 0;
    const uint64_t s1 = P.idx ? P.seg_end[c] : P.count;
    if (s1 <= s0) continue;
    const uint64_t tiles = (s1 - s0 + M - 1) / M;
    if (tiles <= blockIdx.x) continue;
    __syncthreads();  // the previous class's MMAs and drains are complete
    {
      const float4* src = reinterpret_cast<const float4*>(P.b + (size_t)c * 2 * NN * NN);
      float4* dst = reinterpret_cast<float4*>(b_hi);
      for (int i = tid; i < 2 * NN * NN / 4; i += KLT_PIPE_THREADS) dst[i] = __ldg(src + i);
    }
    asm volatile("fence.proxy.async.shared::cta;");
    uint64_t t = blockIdx.x;
    int st = 0;
    uint64_t row = load_tile(s0, s1, t, st);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid == 0) issue(st);
    for (;;) {
      const uint64_t tn = t + gridDim.x;
      const bool more = tn < tiles;
      uint64_t row_n = ~0ull;
      if (more) row_n = load_tile(s0, s1, tn, st ^ 1);  // overlaps MMA(t)
      wait_mma(st);
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();  // A(tn) written; stage st and accumulator st^1 free
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (more && tid == 0) issue(st ^ 1);  // overlaps the drain of t
      drain(st, row);
      asm volatile("tcgen05.fence::before_thread_sync;");
      if (!more) break;
      t = tn;
      row = row_n;
      st ^= 1;
    }
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(2u * NN));
}

// SWIZZLE_128B K-major variant for N = 64 (config 4). The operand layout is the one UMMA reads
// with layout type SWIZZLE_128B: K in 128 B atoms (32 tf32); within an atom, row r sits at
// r * 128 B and its 16 B chunk c at chunk c ^ (r & 7); 8-row groups 1024 B apart (SBO). With it,
// a warp can write two whole 256 B rows per STS.128 instruction without bank conflicts, so the
// rows are gathered from HBM coalesced (2 rows per LDG.128 instruction) instead of one 16 B
// piece per row. The accumulator tile leaves the same way: TMEM -> registers -> swizzled
// staging in the spent A stage -> coalesced STG.128. Two A stages and two TMEM accumulators:
// the gather + tf32 split of tile i+1 overlaps the MMAs of tile i.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                 // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;       // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                 // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}

template <int NN>
__global__ void __launch_bounds__(KLT_PIPE_THREADS, 1) klt_sw_kernel(const KltTcParams P) {
  constexpr int M = 128;
  constexpr uint32_t A_BYTES = M * NN * 4, B_BYTES = NN * NN * 4;
  constexpr int RPW = M / (KLT_PIPE_THREADS / 32);  // rows gathered per warp
  static_assert(NN == 64, "swizzled KLT kernel: N = 64 (two 128 B K atoms)");
  extern __shared__ __align__(1024) unsigned char sm[];
  auto a_st = [&](int st, int lo) { return sm + (2 * st + lo) * A_BYTES; };
  unsigned char* b_hi = sm + 4 * A_BYTES;
  unsigned char* b_lo = sm + 4 * A_BYTES + B_BYTES;
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int half = tid / M;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(&tmem_base_sh)), "r"(2u * NN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&mbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&mbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_sh;
  uint32_t phase[2] = {0, 0};
  // swizzled byte offset of (row r, 16 B chunk q of the full 256 B row) inside an operand tile
  auto swz = [&](int rows, int r, int q) -> uint32_t {
    return (uint32_t)(q >> 3) * (rows * 128u) + (uint32_t)r * 128u + (uint32_t)(((q & 7) ^ (r & 7)) << 4);
  };
  auto row_of = [&](uint64_t s0, uint64_t s1, uint64_t t, int r) -> uint64_t {
    const uint64_t p = s0 + t * M + r;
    return p < s1 ? (P.idx ? (uint64_t)__ldg(P.idx + p) : p) : ~0ull;
  };

  // row ids this lane gathers for a tile (rows warp*RPW + 2i + lane/16), loaded a tile ahead
  auto gather_rows = [&](uint64_t s0, uint64_t s1, uint64_t t, uint64_t (&rows)[RPW / 2]) {
#pragma unroll
    for (int i = 0; i < RPW / 2; ++i) rows[i] = row_of(s0, s1, t, warp * RPW + 2 * i + (lane >> 4));
  };
  auto fetch = [&](const uint64_t (&rows)[RPW / 2], float4 (&v)[RPW / 2]) {
    const int q = lane & 15;
#pragma unroll
    for (int i = 0; i < RPW / 2; ++i)  // chunk lane%16 of rows warp*RPW + 2i + lane/16
      v[i] = rows[i] != ~0ull ? __ldcs(reinterpret_cast<const float4*>(P.in + rows[i] * NN) + q)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  auto stash = [&](const float4 (&v)[RPW / 2], int st) {  // tf32 split into the swizzled A stage
    const int q = lane & 15;
#pragma unroll
    for (int i = 0; i < RPW / 2; ++i) {
      const int r = warp * RPW + 2 * i + (lane >> 4);
      const float4 h = make_float4(to_tf32(v[i].x), to_tf32(v[i].y), to_tf32(v[i].z), to_tf32(v[i].w));
      const float4 l = make_float4(to_tf32(v[i].x - h.x), to_tf32(v[i].y - h.y), to_tf32(v[i].z - h.z),
                                   to_tf32(v[i].w - h.w));
      const uint32_t off = swz(M, r, q);
      *reinterpret_cast<float4*>(a_st(st, 0) + off) = h;
      *reinterpret_cast<float4*>(a_st(st, 1) + off) = l;
    }
    asm volatile("fence.proxy.async.shared::cta;");
  };
  auto issue = [&](int st) {  // one thread: 3xTF32 MMAs of a 128 x NN tile into accumulator st
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t idesc = idesc_tf32(NN);
    const uint32_t ahi = smem_u32(a_st(st, 0)), alo = smem_u32(a_st(st, 1));
    const uint32_t bhi = smem_u32(b_hi), blo = smem_u32(b_lo);
    const uint32_t d = tmem + (uint32_t)(st * NN);
    int first = 1;
#pragma unroll
    for (int ks = 0; ks < NN / 8; ++ks) {  // K = 8 tf32 = 32 B per instruction
      const uint32_t aoff = (uint32_t)(ks >> 2) * (M * 128) + (uint32_t)(ks & 3) * 32;
      const uint32_t boff = (uint32_t)(ks >> 2) * (NN * 128) + (uint32_t)(ks & 3) * 32;
      const uint64_t da[3] = {umma_desc_sw128(alo + aoff), umma_desc_sw128(ahi + aoff), umma_desc_sw128(ahi + aoff)};
      const uint64_t db[3] = {umma_desc_sw128(bhi + boff), umma_desc_sw128(blo + boff), umma_desc_sw128(bhi + boff)};
#pragma unroll
      for (int term = 0; term < 3; ++term) {  // small terms first
        const uint32_t acc = first ? 0u : 1u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
            :: "r"(d), "l"(da[term]), "l"(db[term]), "r"(idesc), "r"(acc));
        first = 0;
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(smem_u32(&mbar[st])));
  };
  auto wait_mma = [&](int st) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra WAIT_%=;\n\t}\n"
        :: "r"(smem_u32(&mbar[st])), "r"(phase[st]));
    phase[st] ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;");
  };
  // accumulator st -> swizzled staging (the spent A-hi stage, row r at r*256 B) -> coalesced rows
  auto drain = [&](uint64_t s0, uint64_t s1, uint64_t t, int st) {
    unsigned char* stg = a_st(st, 0);
    const int r = (warp & 3) * 32 + lane;  // TMEM lane = tile row
#pragma unroll
    for (int c1 = 0; c1 < NN / 2; c1 += 16) {
      const int c0 = half * (NN / 2) + c1;
      uint32_t v[16];
      const uint32_t taddr = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(st * NN + c0);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
            "=r"(v[14]), "=r"(v[15])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        const int q = (c0 + j) >> 2;
        *reinterpret_cast<uint4*>(stg + (uint32_t)r * 256u + (uint32_t)(((q & 8) | ((q & 7) ^ (r & 7))) << 4)) =
            make_uint4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    const int q = lane & 15;
#pragma unroll
    for (int i = 0; i < RPW / 2; ++i) {
      const int rr = warp * RPW + 2 * i + (lane >> 4);
      const uint64_t row = row_of(s0, s1, t, rr);
      const float4 o = *reinterpret_cast<const float4*>(stg + (uint32_t)rr * 256u +
                                                        (uint32_t)(((q & 8) | ((q & 7) ^ (rr & 7))) << 4));
      if (row != ~0ull) __stcs(reinterpret_cast<float4*>(P.out + row * NN) + q, o);
    }
  };

  const int C = P.idx ? P.classes : 1;
  for (int c = 0; c < C; ++c) {
    const uint64_t s0 = P.idx ? (c == 0 ? 0 : P.seg_end[c - 1]) : 0;
    const uint64_t s1 = P.idx ? P.seg_end[c] : P.count;
    if (s1 <= s0) continue;
    const uint64_t tiles = (s1 - s0 + M - 1) / M;
    if (tiles <= blockIdx.x) continue;
    __syncthreads();  // the previous class's MMAs and drains are complete
    {  // this class's B operand (hi then lo), prepared on the host in the swizzled layout
      const float4* src = reinterpret_cast<const float4*>(P.b + (size_t)c * 2 * NN * NN);
      float4* dst = reinterpret_cast<float4*>(b_hi);
      for (int i = tid; i < 2 * NN * NN / 4; i += KLT_PIPE_THREADS) dst[i] = __ldg(src + i);
    }
    // Software pipeline: the rows of tile t+1 are in registers while tile t is in the tensor
    // cores; their ids were fetched one tile earlier still.
    uint64_t t = blockIdx.x;
    int st = 0;
    uint64_t rows[RPW / 2];
    float4 v[RPW / 2];
    gather_rows(s0, s1, t, rows);
    fetch(rows, v);
    stash(v, st);
    const bool two = t + gridDim.x < tiles;
    if (two) {
      gather_rows(s0, s1, t + gridDim.x, rows);
      fetch(rows, v);
      gather_rows(s0, s1, t + 2 * (uint64_t)gridDim.x, rows);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid == 0) issue(st);
    for (;;) {
      const uint64_t tn = t + gridDim.x;
      const bool more = tn < tiles;
      if (more) stash(v, st ^ 1);  // rows of tile tn (loaded during the previous iteration)
      wait_mma(st);
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();  // A(tn) written; accumulator st^1 free
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (more && tid == 0) issue(st ^ 1);  // overlaps the drain of t
      if (tn + gridDim.x < tiles) {           // rows of the tile after tn: in flight over the drain
        fetch(rows, v);
        gather_rows(s0, s1, tn + 2 * (uint64_t)gridDim.x, rows);
      }
      drain(s0, s1, t, st);
      __syncthreads();  // staging reads done before stage st is refilled
      if (!more) break;
      t = tn;
      st ^= 1;
    }
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(2u * NN));
}

// Host: B operand of one class in the canonical layout, split into tf32 hi/lo.
float host_tf32(float x) {  // round to nearest (ties away), 10 explicit mantissa bits
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & 0xffffe000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

void build_b(const float* m /*[n][n] row-major: B[nrow][k]*/, int n, float* out /*hi then lo*/) {
  for (int r = 0; r < n; ++r)
    for (int k = 0; k < n; ++k) {
      const float v = m[(size_t)r * n + k];
      const float h = host_tf32(v), l = host_tf32(v - h);
      const size_t off = (size_t)(k / 4) * (n * 4) + (r / 8) * 32 + (r % 8) * 4 + (k % 4);
      out[off] = h;
      out[(size_t)n * n + off] = l;
    }
}

// Host: B operand of one class in the SWIZZLE_128B K-major layout (64 x 64), hi then lo.
void build_b_sw128(const float* m /*[n][n]: B[nrow][k]*/, int n, float* out) {
  for (int r = 0; r < n; ++r)
    for (int k = 0; k < n; ++k) {
      const float v = m[(size_t)r * n + k];
      const float h = host_tf32(v), l = host_tf32(v - h);
      const int q = k / 4, atom = q >> 3;
      const size_t byte = (size_t)atom * (n * 128) + (size_t)r * 128 + (size_t)(((q & 7) ^ (r & 7)) << 4) + (k % 4) * 4;
      out[byte / 4] = h;
      out[(size_t)n * n + byte / 4] = l;
    }
}

template <int NN>
int launch_tc(const hygt_klt_plan* p, int dir, const float* in, float* out, const uint32_t* idx,
              const uint32_t* seg_end, uint64_t count, cudaStream_t st) {
  const size_t smem = (size_t)2 * 128 * NN * 4 + (size_t)2 * NN * NN * 4;
  hygt_smem_attr(reinterpret_cast<const void*>(klt_tc_kernel<NN>), smem);
  KltTcParams P{in, out, idx, seg_end, p->classes, count, p->d_b[dir]};
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, klt_tc_kernel<NN>, 128, smem);
  if (occ < 1) occ = 1;
  const uint64_t tiles = (count + 127) / 128;
  const unsigned grid = (unsigned)std::min<uint64_t>((uint64_t)p->num_sms * occ, tiles);
  klt_tc_kernel<NN><<<grid, 128, smem, st>>>(P);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HYGT_OK : kfail(HYGT_ERR_CUDA, cudaGetErrorString(e));
}

template <int NN>
int launch_pipe(const hygt_klt_plan* p, int dir, const float* in, float* out, const uint32_t* idx,
                const uint32_t* seg_end, uint64_t count, cudaStream_t st) {
  if (getenv("HYGT_KLT_PIPE") && atoi(getenv("HYGT_KLT_PIPE")) == 0)
    return launch_tc<NN>(p, dir, in, out, idx, seg_end, count, st);
  const size_t smem = (size_t)4 * 128 * NN * 4 + (size_t)2 * NN * NN * 4;
  hygt_smem_attr(reinterpret_cast<const void*>(klt_tc_pipe_kernel<NN>), smem);
  const uint64_t tiles = (count + 127) / 128;
  const unsigned grid = (unsigned)std::min<uint64_t>((uint64_t)p->num_sms, tiles);
  if (p->d_bsw[dir] && !(getenv("HYGT_KLT_SW") && atoi(getenv("HYGT_KLT_SW")) == 0)) {
    hygt_smem_attr(reinterpret_cast<const void*>(klt_sw_kernel<NN>), smem);
    KltTcParams Q{in, out, idx, seg_end, p->classes, count, p->d_bsw[dir]};
    klt_sw_kernel<NN><<<grid, KLT_PIPE_THREADS, smem, st>>>(Q);
  } else {
    KltTcParams P{in, out, idx, seg_end, p->classes, count, p->d_b[dir]};
    klt_tc_pipe_kernel<NN><<<grid, KLT_PIPE_THREADS, smem, st>>>(P);
  }
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HYGT_OK : kfail(HYGT_ERR_CUDA, cudaGetErrorString(e));
}

int run_klt(const hygt_klt_plan* p, bool fwd, const float* in, float* out, const uint16_t* cls,
            uint64_t count, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (!p) return kfail(HYGT_ERR_ARGUMENT, "klt: null plan");
  if (!count) return HYGT_OK;
  if (in == out) return kfail(HYGT_ERR_ARGUMENT, "klt: in-place not supported");
  if (p->tc) {
    const uint32_t* idx = nullptr;
    const uint32_t* seg = nullptr;
    uint32_t nseg = 0;
    if (cls && p->classes > 1) {
      if (!ws || ws_bytes < hygt_gpu::bucket_ws_bytes(p->classes, 0, count))
        return kfail(HYGT_ERR_ARGUMENT, "klt: workspace too small");
      if (int s = hygt_gpu::bucket_rows(p->classes, 0, cls, count, ws, ws_bytes, true, st, &idx, &seg, &nseg))
        return s;
    }
    const int dir = fwd ? 0 : 1;
    switch (p->n) {
      case 16: return launch_tc<16>(p, dir, in, out, idx, seg, count, st);
      case 32: return launch_tc<32>(p, dir, in, out, idx, seg, count, st);
      case 64: return launch_pipe<64>(p, dir, in, out, idx, seg, count, st);
      default: break;
    }
  }
  const int rows_per_cta = KT / p->n;
  const uint64_t ctas = std::min<uint64_t>((count + rows_per_cta - 1) / rows_per_cta, (uint64_t)p->num_sms * 8);
  // forward y = K x  -> MT = K^T ; inverse x = K^T y -> MT = K
  klt_simt_kernel<<<(unsigned)ctas, KT, KT * sizeof(float), st>>>(in, out, cls, count, p->n,
                                                                  p->classes, fwd ? p->d_kt : p->d_k);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return kfail(HYGT_ERR_CUDA, cudaGetErrorString(e));
  return HYGT_OK;
}
}  // namespace

extern "C" int hygt_klt_plan_create(int n, int class_count, const double* k, uint32_t flags,
                                    hygt_klt_plan** out) {
  if (!out || !k) return kfail(HYGT_ERR_ARGUMENT, "hygt_klt_plan_create: null argument");
  *out = nullptr;
  if (n < 2 || n > KT || (n & (n - 1))) return kfail(HYGT_ERR_ARGUMENT, "hygt_klt_plan_create: n must be a power of two in [2, 256]");
  if (class_count < 1) return kfail(HYGT_ERR_ARGUMENT, "hygt_klt_plan_create: class_count");
  const size_t nn = (size_t)n * n * class_count;
  std::vector<float> kf(nn), ktf(nn);
  for (int c = 0; c < class_count; ++c)
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        const float v = (float)k[((size_t)c * n + i) * n + j];
        kf[((size_t)c * n + i) * n + j] = v;
        ktf[((size_t)c * n + j) * n + i] = v;
      }
  hygt_klt_plan* p = new hygt_klt_plan();
  p->n = n;
  p->classes = class_count;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, dev);
  p->tc = (n == 16 || n == 32 || n == 64) && !(flags & 1u);  // flag bit 0: force SIMT
  bool okk = cudaMalloc(&p->d_k, nn * sizeof(float)) == cudaSuccess &&
             cudaMalloc(&p->d_kt, nn * sizeof(float)) == cudaSuccess &&
             cudaMemcpy(p->d_k, kf.data(), nn * sizeof(float), cudaMemcpyHostToDevice) == cudaSuccess &&
             cudaMemcpy(p->d_kt, ktf.data(), nn * sizeof(float), cudaMemcpyHostToDevice) == cudaSuccess;
  if (okk && p->tc) {
    // forward: OUT = IN * K^T -> B[nrow][k] = K[nrow][k]; inverse: B = K^T
    for (int d = 0; d < 2 && okk; ++d) {
      std::vector<float> b((size_t)class_count * 2 * n * n);
      for (int c = 0; c < class_count; ++c)
        build_b((d == 0 ? kf.data() : ktf.data()) + (size_t)c * n * n, n, b.data() + (size_t)c * 2 * n * n);
      okk = cudaMalloc(&p->d_b[d], b.size() * sizeof(float)) == cudaSuccess &&
            cudaMemcpy(p->d_b[d], b.data(), b.size() * sizeof(float), cudaMemcpyHostToDevice) == cudaSuccess;
      if (okk && n == 64) {
        for (int c = 0; c < class_count; ++c)
          build_b_sw128((d == 0 ? kf.data() : ktf.data()) + (size_t)c * n * n, n, b.data() + (size_t)c * 2 * n * n);
        okk = cudaMalloc(&p->d_bsw[d], b.size() * sizeof(float)) == cudaSuccess &&
              cudaMemcpy(p->d_bsw[d], b.data(), b.size() * sizeof(float), cudaMemcpyHostToDevice) == cudaSuccess;
      }
    }
  }
  if (!okk) {
    hygt_klt_plan_destroy(p);
    return kfail(HYGT_ERR_CUDA, "hygt_klt_plan_create: device allocation failed");
  }
  *out = p;
  return HYGT_OK;
}

extern "C" int hygt_klt_plan_destroy(hygt_klt_plan* p) {
  if (!p) return HYGT_OK;
  cudaFree(p->d_k);
  cudaFree(p->d_kt);
  cudaFree(p->d_b[0]);
  cudaFree(p->d_b[1]);
  cudaFree(p->d_bsw[0]);
  cudaFree(p->d_bsw[1]);
  delete p;
  return HYGT_OK;
}

extern "C" size_t hygt_klt_workspace_bytes(const hygt_klt_plan* plan, uint64_t count) {
  if (!plan || !plan->tc || plan->classes <= 1) return 256;
  return hygt_gpu::bucket_ws_bytes(plan->classes, 0, count);
}

extern "C" int hygt_klt_forward_f32(const hygt_klt_plan* plan, const float* d_x, float* d_y,
                                    const uint16_t* d_cls, uint64_t count, void* d_ws,
                                    size_t ws_bytes, void* stream) {
  return run_klt(plan, true, d_x, d_y, d_cls, count, d_ws, ws_bytes,
                 reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int hygt_klt_inverse_f32(const hygt_klt_plan* plan, const float* d_y, float* d_x,
                                    const uint16_t* d_cls, uint64_t count, void* d_ws,
                                    size_t ws_bytes, void* stream) {
  return run_klt(plan, false, d_y, d_x, d_cls, count, d_ws, ws_bytes,
                 reinterpret_cast<cudaStream_t>(stream));
}
