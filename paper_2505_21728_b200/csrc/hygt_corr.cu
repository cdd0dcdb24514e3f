// hygt_corr.cu -- per-class second-moment accumulation: sum_c += r r^T over the
// rows of class c, count_c += rows (CorrelationAccumulator::add, statistics.hpp:63-99; finalize
// divides by the count). It is the statistic `hygt train` builds before optimizing a class
// (tools/hygt_main.cpp:85-87), and shards merge by addition (statistics.hpp:110-120) -- one
// NCCL all-reduce of the sums and counts (paper_2505_21728_b200/dist.py).
//
// Exactness: the samples are fp32 (RBLK storage), so every product r_i r_j is exact in fp64 and
// the kernel accumulates with DFMA in fp64 -- the result differs from the reference only by the
// order of the fp64 additions.
// Layout: rows are globally class-bucketed (hygt_bucket's histogram / scan / scatter); each CTA
// walks a contiguous range of bucketed positions. A CTA owns one 64 x 64 (or N x N for N < 64)
// output tile of the upper block triangle; its 256 threads hold 4 x 4 fp64 accumulators each.
// 32-row chunks of the class run are staged through shared memory with coalesced 128-bit loads.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>

#include "../../include/hygt_gpu.h"
#include "hygt_corr_tc.h"
#include "hygt_knobs.h"
#include "hygt_nvtx.h"

int hygt_set_error(int status, const char* msg);  // hygt_capi.cu
namespace hygt_gpu {
size_t bucket_ws_bytes(int classes, uint64_t chunk_rows, uint64_t count);
int bucket_rows(int classes, uint64_t chunk_rows, const uint16_t* d_cls, uint64_t count,
                void* d_ws, size_t ws_bytes, bool run, cudaStream_t st, const uint32_t** idx,
                const uint32_t** seg_end, uint32_t* nseg);
}  // namespace hygt_gpu

namespace {

constexpr int CORR_THREADS = 256;
constexpr int CORR_RT = 32;  // rows per shared-memory chunk

struct CorrParams {
  const float* x;
  const uint32_t* idx;      // bucketed position -> row (nullptr: identity, one class)
  const uint32_t* seg_end;  // [C+1] run ends
  int classes;
  uint64_t count;
  double* sum;              // [C][N][N]
  unsigned long long* cnt;  // [C]
  uint64_t cta_span;
};

// Per chunk, the tile's two row slices are staged once as fp64 (each sample converted once, not
// once per thread that reads it); the j slice is stored element-interleaved (k = b E + w at
// w TD + b) so a warp's 16 column threads read 16 consecutive doubles. Diagonal tiles compute
// only the 4 x 4 blocks on or above the diagonal (the rest is their mirror).
template <int N>
__global__ void __launch_bounds__(CORR_THREADS) corr_kernel(const CorrParams P) {
  constexpr int OT = N < 64 ? N : 64;           // output tile side
  constexpr int TD = OT < 16 ? OT : 16;         // threads per tile side
  constexpr int E = OT / TD;                    // accumulators per thread per side
  constexpr int TILES = N / OT;
  __shared__ __align__(16) double si[CORR_RT][OT];  // rows' samples i0 .. of the tile, natural order
  __shared__ __align__(16) double sj[CORR_RT][OT];  // samples j0 .., element-interleaved
  // upper block-triangle tile (ti <= tj) of this CTA
  int ti = 0, tj = (int)blockIdx.y;
  while (tj >= TILES - ti) { tj -= TILES - ti; ++ti; }
  tj += ti;
  const int tid = threadIdx.x;
  const int a = tid / TD, b = tid % TD;
  const bool active = tid < TD * TD && (ti != tj || a <= b);
  const int i0 = ti * OT + a * E, j0 = tj * OT + b * E;

  const uint64_t beg = (uint64_t)blockIdx.x * P.cta_span;
  if (beg >= P.count) return;
  const uint64_t end = beg + P.cta_span < P.count ? beg + P.cta_span : P.count;
  const int C = P.idx ? P.classes : 1;
  int f = 0;
  if (P.idx) {
    int lo = 0, hi = C + 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((uint64_t)__ldg(P.seg_end + mid) <= beg) lo = mid + 1; else hi = mid;
    }
    f = lo;
  }
  for (uint64_t pos = beg; pos < end; ++f) {
    const uint64_t se = P.idx ? (uint64_t)__ldg(P.seg_end + f) : P.count;
    const uint64_t stop = se < end ? se : end;
    if (stop <= pos) continue;
    if (f >= C) break;  // invalid ids (bin C) are flagged by the bucketing and not counted
    double acc[E][E];
#pragma unroll
    for (int u = 0; u < E; ++u)
#pragma unroll
      for (int w = 0; w < E; ++w) acc[u][w] = 0.0;
    for (uint64_t r0 = pos; r0 < stop; r0 += CORR_RT) {
      const int nr = (int)(stop - r0 < (uint64_t)CORR_RT ? stop - r0 : (uint64_t)CORR_RT);
      __syncthreads();
      // coalesced 16 B pieces of the two slices, converted to fp64 once
      constexpr int Q = OT / 4;
      for (int q = tid; q < nr * Q * 2; q += CORR_THREADS) {
        const int half = q / (nr * Q), qq = q % (nr * Q);
        const int r = qq / Q, k4 = qq % Q;
        if (half == 1 && ti == tj) continue;  // diagonal tile: one slice serves both sides
        const uint64_t row = P.idx ? (uint64_t)__ldg(P.idx + r0 + r) : r0 + r;
        const float4 v = __ldcs(reinterpret_cast<const float4*>(P.x + row * N + (half ? tj : ti) * OT) + k4);
        const float e4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int k = 4 * k4 + t;
          if (!half) si[r][k] = (double)e4[t];
          if (half || ti == tj) sj[r][(k % E) * TD + k / E] = (double)e4[t];
        }
      }
      __syncthreads();
      if (active)
        for (int r = 0; r < nr; ++r) {
          double xi[E], xj[E];
#pragma unroll
          for (int u = 0; u < E; ++u) {
            xi[u] = si[r][a * E + u];
            xj[u] = sj[r][u * TD + b];
          }
#pragma unroll
          for (int u = 0; u < E; ++u)
#pragma unroll
            for (int w = 0; w < E; ++w) acc[u][w] = fma(xi[u], xj[w], acc[u][w]);  // exact products
        }
    }
    if (active) {
      double* s = P.sum + (size_t)f * N * N;
      const bool mirror = ti != tj || a < b;  // diagonal blocks of diagonal tiles hold both halves
#pragma unroll
      for (int u = 0; u < E; ++u)
#pragma unroll
        for (int w = 0; w < E; ++w) {
          atomicAdd(s + (size_t)(i0 + u) * N + (j0 + w), acc[u][w]);
          if (mirror) atomicAdd(s + (size_t)(j0 + w) * N + (i0 + u), acc[u][w]);
        }
    }
    if (blockIdx.y == 0 && tid == 0) atomicAdd(P.cnt + f, (unsigned long long)(stop - pos));
    pos = stop;
  }
}

using CorrFn = void (*)(CorrParams);
CorrFn select_corr(int log2n) {
  switch (log2n) {
    case 2: return corr_kernel<4>;
    case 3: return corr_kernel<8>;
    case 4: return corr_kernel<16>;
    case 5: return corr_kernel<32>;
    case 6: return corr_kernel<64>;
    case 7: return corr_kernel<128>;
    case 8: return corr_kernel<256>;
    default: return nullptr;
  }
}

}  // namespace

extern "C" size_t hygt_correlation_workspace_bytes(int classes, uint64_t count) {
  return hygt_gpu::bucket_ws_bytes(classes < 1 ? 1 : classes, 0, count);
}

extern "C" int hygt_correlation_f64(int log2_n, int classes, const float* d_x, const uint16_t* d_cls,
                                    uint64_t count, double* d_sum, unsigned long long* d_count,
                                    void* d_ws, size_t ws_bytes, void* stream) {
  HYGT_NVTX("hygt_correlation_f64");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CorrFn fn = select_corr(log2_n);
  if (!fn) return hygt_set_error(HYGT_ERR_ARGUMENT, "hygt_correlation_f64: log2_n must be in [2, 8]");
  if (classes < 1) return hygt_set_error(HYGT_ERR_ARGUMENT, "hygt_correlation_f64: class_count");
  if (!d_sum || !d_count) return hygt_set_error(HYGT_ERR_ARGUMENT, "hygt_correlation_f64: null output");
  if (count == 0) return HYGT_OK;
  if (!d_x || (reinterpret_cast<uintptr_t>(d_x) & 15))
    return hygt_set_error(HYGT_ERR_ARGUMENT, "hygt_correlation_f64: x must be 16-byte aligned");
  CorrParams P{};
  P.x = d_x;
  P.classes = classes;
  P.count = count;
  P.sum = d_sum;
  P.cnt = d_count;
  if (d_cls) {  // also for one class: the bucketing validates the ids (ResidualDataset)
    if (!d_ws || ws_bytes < hygt_gpu::bucket_ws_bytes(classes, 0, count))
      return hygt_set_error(HYGT_ERR_ARGUMENT, "hygt_correlation_f64: workspace too small");
    uint32_t nseg = 0;
    if (int s = hygt_gpu::bucket_rows(classes, 0, d_cls, count, d_ws, ws_bytes, true, st, &P.idx, &P.seg_end, &nseg))
      return s;
    if (classes == 1) P.idx = P.seg_end = nullptr;  // ids only validated; rows in place
  }
  const int n = 1 << log2_n, ot = n < 64 ? n : 64, tiles = n / ot;
  const int tiles_ut = tiles * (tiles + 1) / 2;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (hygt_gpu::corr_tc_supported(log2_n) && hygt_gpu::knob("HYGT_CORR_TC", 1) != 0) {  // (d_x is 16-byte aligned, checked above)
    // N >= 64: exact integer-digit products on the tensor cores (hygt_corr_tc.cu)
    hygt_gpu::CorrTcParams Q{};
    Q.x = d_x;
    Q.n = 1 << log2_n;
    Q.dbg = hygt_gpu::knob("HYGT_CORR_DBG", 0);
    Q.idx = P.idx;
    Q.seg_end = P.seg_end;
    Q.classes = classes;
    Q.count = count;
    Q.sum = d_sum;
    Q.cnt = d_count;
    return hygt_gpu::corr_tc_run(Q, sms, st);
  }
  const uint64_t want = std::max<uint64_t>(1, (uint64_t)sms * 8 / tiles_ut);
  const uint64_t ctas = std::min<uint64_t>(want, (count + CORR_RT - 1) / CORR_RT);
  P.cta_span = (count + ctas - 1) / ctas;
  fn<<<dim3((unsigned)ctas, (unsigned)tiles_ut), CORR_THREADS, 0, st>>>(P);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HYGT_OK : hygt_set_error(HYGT_ERR_CUDA, cudaGetErrorString(e));
}
