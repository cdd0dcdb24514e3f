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
// n in {16, 32} uses this kernel; n in {64, 128, 256} the per-class grouped GEMM of
// hygt_gemm.cu (fp16 3-term split with per-row scaling, CTA pairs, warp-specialised pipeline)
// that also serves the composed-operator HyGT path; other n the fp32 SIMT kernel.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hygt_gpu.h"
#include "hygt_gemm.h"
#include "hygt_nvtx.h"

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
  bool tc = false;                     // N = 16 / 32: klt_tc_kernel (3xTF32)
  bool gemm = false;                   // N = 64 / 128 / 256: hygt_gemm.cu (fp16 3-term, CTA pairs)
  hygt_gpu::GemmOperands gops[2];
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

int run_klt(const hygt_klt_plan* p, bool fwd, const float* in, float* out, const uint16_t* cls,
            uint64_t count, void* ws, size_t ws_bytes, cudaStream_t st, bool reuse = false) {
  if (!p) return kfail(HYGT_ERR_ARGUMENT, "klt: null plan");
  if (!count) return HYGT_OK;
  if (p->gemm) {  // per-class grouped GEMM on the tensor cores (in place allowed)
    if (((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) != 0)
      return kfail(HYGT_ERR_ARGUMENT, "klt: x and y must be aligned to 16 bytes");
    if (count > 0xFFFFFFFFull) return kfail(HYGT_ERR_ARGUMENT, "klt: at most 2^32-1 rows per call");
    const uint32_t* idx = nullptr;
    const uint32_t* seg = nullptr;
    uint32_t nseg = 0;
    if (cls && p->classes > 1) {
      if (!ws || ws_bytes < hygt_gpu::bucket_ws_bytes(p->classes, 0, count))
        return kfail(HYGT_ERR_ARGUMENT, "klt: workspace too small");
      if (int s = hygt_gpu::bucket_rows(p->classes, 0, cls, count, ws, ws_bytes, !reuse, st, &idx, &seg, &nseg))
        return s;
    }
    return hygt_gpu::gemm_run(p->gops[fwd ? 0 : 1], in, out, idx, seg, count, nullptr, st);
  }
  if (in == out) return kfail(HYGT_ERR_ARGUMENT, "klt: in-place not supported");
  if (p->tc) {
    const uint32_t* idx = nullptr;
    const uint32_t* seg = nullptr;
    uint32_t nseg = 0;
    if (cls && p->classes > 1) {
      if (!ws || ws_bytes < hygt_gpu::bucket_ws_bytes(p->classes, 0, count))
        return kfail(HYGT_ERR_ARGUMENT, "klt: workspace too small");
      if (int s = hygt_gpu::bucket_rows(p->classes, 0, cls, count, ws, ws_bytes, !reuse, st, &idx, &seg, &nseg))
        return s;
    }
    const int dir = fwd ? 0 : 1;
    switch (p->n) {
      case 16: return launch_tc<16>(p, dir, in, out, idx, seg, count, st);
      case 32: return launch_tc<32>(p, dir, in, out, idx, seg, count, st);
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
  HYGT_NVTX("hygt_klt_plan_create");
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
  p->tc = (n == 16 || n == 32) && !(flags & 1u);  // flag bit 0: force SIMT
  if (!(flags & 1u) && hygt_gpu::gemm_supported(n, class_count)) {
    // forward y = K x: B[nrow][k] = K[nrow][k]; inverse x = K^T y: B = K^T (fp64 from the caller)
    std::vector<double> kt(nn);
    for (int c = 0; c < class_count; ++c)
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) kt[((size_t)c * n + j) * n + i] = k[((size_t)c * n + i) * n + j];
    hygt_klt_plan* q = new hygt_klt_plan();
    q->n = n;
    q->classes = class_count;
    q->num_sms = 148;
    int st = hygt_gpu::gemm_build(n, class_count, k, q->gops[0]);
    if (!st) st = hygt_gpu::gemm_build(n, class_count, kt.data(), q->gops[1]);
    if (st) {
      hygt_klt_plan_destroy(q);
      return st;
    }
    q->gemm = true;
    *out = q;
    return HYGT_OK;
  }
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
  hygt_gpu::gemm_release(p->gops[0]);
  hygt_gpu::gemm_release(p->gops[1]);
  delete p;
  return HYGT_OK;
}

extern "C" size_t hygt_klt_workspace_bytes(const hygt_klt_plan* plan, uint64_t count) {
  if (!plan || !(plan->tc || plan->gemm) || plan->classes <= 1) return 256;
  return hygt_gpu::bucket_ws_bytes(plan->classes, 0, count);
}

extern "C" int hygt_klt_forward_f32(const hygt_klt_plan* plan, const float* d_x, float* d_y,
                                    const uint16_t* d_cls, uint64_t count, void* d_ws,
                                    size_t ws_bytes, void* stream) {
  HYGT_NVTX("hygt_klt_forward_f32");
  return run_klt(plan, true, d_x, d_y, d_cls, count, d_ws, ws_bytes,
                 reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int hygt_klt_inverse_f32(const hygt_klt_plan* plan, const float* d_y, float* d_x,
                                    const uint16_t* d_cls, uint64_t count, void* d_ws,
                                    size_t ws_bytes, void* stream) {
  HYGT_NVTX("hygt_klt_inverse_f32");
  return run_klt(plan, false, d_y, d_x, d_cls, count, d_ws, ws_bytes,
                 reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int hygt_klt_bucket(const hygt_klt_plan* plan, const uint16_t* d_cls, uint64_t count,
                               void* d_ws, size_t ws_bytes, void* stream) {
  HYGT_NVTX("hygt_klt_bucket");
  if (!plan) return kfail(HYGT_ERR_ARGUMENT, "klt: null plan");
  if (!count || !d_cls || plan->classes <= 1 || !(plan->gemm || plan->tc)) return HYGT_OK;
  if (!d_ws || ws_bytes < hygt_gpu::bucket_ws_bytes(plan->classes, 0, count))
    return kfail(HYGT_ERR_ARGUMENT, "klt: workspace too small");
  const uint32_t* idx = nullptr;
  const uint32_t* seg = nullptr;
  uint32_t nseg = 0;
  return hygt_gpu::bucket_rows(plan->classes, 0, d_cls, count, d_ws, ws_bytes, true,
                               reinterpret_cast<cudaStream_t>(stream), &idx, &seg, &nseg);
}

extern "C" int hygt_klt_forward_f32_ex(const hygt_klt_plan* plan, const float* d_x, float* d_y,
                                       const uint16_t* d_cls, uint64_t count, void* d_ws,
                                       size_t ws_bytes, uint32_t flags, void* stream) {
  HYGT_NVTX("hygt_klt_forward_f32");
  return run_klt(plan, true, d_x, d_y, d_cls, count, d_ws, ws_bytes,
                 reinterpret_cast<cudaStream_t>(stream), (flags & HYGT_REUSE_BUCKETS) != 0);
}

extern "C" int hygt_klt_inverse_f32_ex(const hygt_klt_plan* plan, const float* d_y, float* d_x,
                                       const uint16_t* d_cls, uint64_t count, void* d_ws,
                                       size_t ws_bytes, uint32_t flags, void* stream) {
  HYGT_NVTX("hygt_klt_inverse_f32");
  return run_klt(plan, false, d_y, d_x, d_cls, count, d_ws, ws_bytes,
                 reinterpret_cast<cudaStream_t>(stream), (flags & HYGT_REUSE_BUCKETS) != 0);
}
