// hygt_segment.cuh -- the "segment" HyGT kernel for long rows (N >= 64: the per-class tables
// are 6-33 KB, too large to hold every class in shared memory).
//
// Rows are globally bucketed by class first (hygt_bucket: histogram + scan + scatter of row
// indices, the batched form of run_apply's cache[b.class_id] dispatch, hygt_main.cpp:143-149).
// Each persistent CTA takes a contiguous range of bucketed positions and walks the class
// segments inside it: for each segment it stages that class's coefficient / scale / gather
// tables into shared memory once, then every warp processes VPT rows per lane group with all
// coefficient loads shared by the group's rows and broadcast across the warp. The fused energy
// epilogue (statistics.hpp:69-77 diagonal) accumulates y^2 per lane in fp32 for at most 128 rows,
// then reduces across the warp's lane groups in fp64 and adds into the [C][N] fp64 sums.
#pragma once

#include "hygt_tile.cuh"

namespace hygt_gpu {

struct SegParams {
  const float* x;
  float* y;
  const uint32_t* idx;      // bucketed position -> row
  const uint32_t* seg_end;  // [C+1] end position of each class run (bin C = invalid ids)
  int classes;
  int rounds;
  uint64_t count;
  const float4* coef;       // [C][units][TPV] float4
  uint32_t units;
  const uint4* gidx;        // [C][R+1][words][TPV] uint4 (byte offsets into the scratch)
  uint64_t gmask;
  uint64_t cta_span;        // positions per CTA
  double* energy;
};

template <int LOG2N, int L, int VPT>
__device__ __forceinline__ void seg_load(const SegParams& P, const uint32_t (&row)[VPT],
                                         float2 (&dst)[VPT][TileGeom<LOG2N, L>::NP], int t) {
  using G = TileGeom<LOG2N, L>;
#pragma unroll
  for (int r = 0; r < VPT; ++r) {
    const float4* xr = reinterpret_cast<const float4*>(P.x + (size_t)row[r] * G::N);
#pragma unroll
    for (int u = 0; u < G::E / G::CH; ++u) {
      const float4 a = __ldcs(xr + t + G::TPV * u);
      dst[r][2 * u] = make_float2(a.x, a.y);
      dst[r][2 * u + 1] = make_float2(a.z, a.w);
    }
  }
}

template <int LOG2N, int L, int VPT, bool STD, bool FWD, bool ENERGY, bool PREFETCH, int THREADS>
__global__ void __launch_bounds__(THREADS, (LOG2N >= 8 ? 1 : 2)) hygt_segment_kernel(const SegParams P) {
  using G = TileGeom<LOG2N, L>;
  constexpr Layout LY = G::LY;
  constexpr int N = G::N, TPV = G::TPV, E = G::E, NP = G::NP, V = G::V;
  constexpr int ROWS = V * VPT;
  constexpr int WARPS = THREADS / 32;
  constexpr int S = G::template stride<VPT>();
  // energy by shuffle reduce-scatter (lanes per row >= 4, at least one full group per lane)
  constexpr bool SEG_RS = L >= 2 && E >= (2 << (5 - L));
  extern __shared__ __align__(16) unsigned char seg_smem[];
  const int C = P.classes;
  const uint32_t cw = P.units * TPV;                                   // float4 per class
  const uint32_t gw = P.gmask ? (P.rounds + 1) * ((E + 7) / 8) * TPV : 0;  // uint4 per class
  float4* s_coef = reinterpret_cast<float4*>(seg_smem);
  uint4* s_gidx = reinterpret_cast<uint4*>(s_coef + cw);
  float* s_scratch = reinterpret_cast<float*>(s_gidx + gw);
  // fused energy: per-lane fp64 partial sums in shared memory, [E][32] per warp (keeps the
  // accumulators out of the register file, which the E samples of a long row already fill).
  // Each addition is an fp32 sum of at most 32 squares of one step's rows.
  double* s_acc = reinterpret_cast<double*>(s_scratch + (((P.gmask ? (size_t)WARPS * N * S : 0) + 1) & ~(size_t)1)) +
                  (size_t)(threadIdx.x >> 5) * E * 32 + (threadIdx.x & 31);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> L, t = lane & (TPV - 1);
  float* wscr = s_scratch + (size_t)warp * N * S;
  float* wbase = wscr + g + ((t << LY.chl()) * S);
  const char* rbase = reinterpret_cast<const char*>(wscr + g);
  const uint32_t gstep_words = ((E + 7) / 8) * TPV;

  const uint64_t beg = (uint64_t)blockIdx.x * P.cta_span;
  if (beg >= P.count) return;
  const uint64_t end = beg + P.cta_span < P.count ? beg + P.cta_span : P.count;
  uint32_t f = 0;
  {
    uint32_t lo = 0, hi = (uint32_t)C + 1;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if ((uint64_t)__ldg(P.seg_end + mid) <= beg) lo = mid + 1; else hi = mid;
    }
    f = lo;
  }
  for (uint64_t pos = beg; pos < end; ++f) {
    const uint64_t stop = (uint64_t)__ldg(P.seg_end + f) < end ? (uint64_t)__ldg(P.seg_end + f) : end;
    const int c = (int)f;
    if (stop <= pos) continue;
    if (c >= C) {  // rows with invalid class ids: copy through (error flagged by hygt_bucket)
      for (uint64_t p = pos + tid / TPV; p < stop; p += THREADS / TPV) {
        const uint32_t row = __ldg(P.idx + p);
        const float4* xr = reinterpret_cast<const float4*>(P.x + (size_t)row * N);
        float4* yr = reinterpret_cast<float4*>(P.y + (size_t)row * N);
        for (int q = t; q < N / 4; q += TPV) yr[q] = xr[q];
      }
      pos = stop;
      continue;
    }
    __syncthreads();  // previous segment's tables no longer in use
    for (uint32_t i = tid; i < cw; i += THREADS) s_coef[i] = __ldg(P.coef + (size_t)c * cw + i);
    for (uint32_t i = tid; i < gw; i += THREADS) s_gidx[i] = __ldg(P.gidx + (size_t)c * gw + i);
    __syncthreads();
    if constexpr (ENERGY) {
#pragma unroll 8
      for (int s = 0; s < E; ++s) s_acc[s * 32] = 0.0;
    }
    int acc_rows = 0;
    auto flush = [&]() {
      if constexpr (ENERGY) {
        // fp64 partial sums, reduced across the lane groups in fp64
#pragma unroll 4
        for (int s = 0; s < E; ++s) {
          double d = s_acc[s * 32];
#pragma unroll
          for (int o = TPV; o < 32; o <<= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
          s_acc[s * 32] = 0.0;
          if (g == 0) atomicAdd(P.energy + (size_t)c * N + LY.elem(t, s), d);
        }
      }
    };
    const uint64_t nseg = stop - pos;
    const uint64_t steps = (nseg + ROWS - 1) / ROWS;
    uint32_t row_n[VPT];
    float2 vn[VPT][NP];
    auto rows_of = [&](uint64_t step, uint32_t (&rw)[VPT], bool (&ok)[VPT]) {
#pragma unroll
      for (int r = 0; r < VPT; ++r) {
        const uint64_t p = pos + step * ROWS + r * V + g;
        ok[r] = p < stop;
        rw[r] = __ldg(P.idx + (ok[r] ? p : pos));  // inactive slots re-read a valid row
      }
    };
    uint64_t step = warp;
    bool ok_n[VPT];
    if (PREFETCH && step < steps) {
      rows_of(step, row_n, ok_n);
      seg_load<LOG2N, L, VPT>(P, row_n, vn, t);
    }
    for (; step < steps; step += WARPS) {  // warp-uniform trip count
      uint32_t row[VPT];
      bool ok[VPT];
      float2 v[VPT][NP];
      if constexpr (PREFETCH) {
#pragma unroll
        for (int r = 0; r < VPT; ++r) {
          row[r] = row_n[r];
          ok[r] = ok_n[r];
#pragma unroll
          for (int k = 0; k < NP; ++k) v[r][k] = vn[r][k];
        }
        if (step + WARPS < steps) {
          rows_of(step + WARPS, row_n, ok_n);
          seg_load<LOG2N, L, VPT>(P, row_n, vn, t);
        }
      } else {
        rows_of(step, row, ok);
        seg_load<LOG2N, L, VPT>(P, row, v, t);
      }
      const float4* cp[VPT];
      const uint4* gp[VPT];
#pragma unroll
      for (int r = 0; r < VPT; ++r) {
        cp[r] = s_coef + t;
        gp[r] = s_gidx + t;
      }
      tile_rows<LOG2N, L, STD, FWD, VPT, true>(v, cp, gp, gstep_words, wbase, rbase, P.rounds,
                                               P.gmask);
#pragma unroll
      for (int r = 0; r < VPT; ++r) {
        if (!ok[r]) continue;
        float4* yr = reinterpret_cast<float4*>(P.y + (size_t)row[r] * N);
#pragma unroll
        for (int u = 0; u < E / G::CH; ++u)
          __stcs(yr + t + TPV * u,
                 make_float4(v[r][2 * u].x, v[r][2 * u].y, v[r][2 * u + 1].x, v[r][2 * u + 1].y));
        if constexpr (ENERGY && !SEG_RS) {
#pragma unroll
          for (int k = 0; k < NP; ++k) {
            s_acc[(2 * k) * 32] += (double)(v[r][k].x * v[r][k].x);
            s_acc[(2 * k + 1) * 32] += (double)(v[r][k].y * v[r][k].y);
          }
        }
      }
      if constexpr (ENERGY && SEG_RS) {
        // y^2 of the warp's rows reduce-scattered over the row-group lane bits with shuffles, in
        // groups of GS slots: each lane adds 2 sums per group to its partials (instead of one
        // shared-memory read-modify-write per sample and row)
        constexpr int S = 5 - L, GS = 2 << S;
#pragma unroll
        for (int g0 = 0; g0 < E; g0 += GS) {
          float q[GS];
#pragma unroll
          for (int i = 0; i < GS; ++i) {
            float acc = 0.f;
#pragma unroll
            for (int r = 0; r < VPT; ++r)
              if (ok[r]) {
                const float e = ((g0 + i) & 1) ? v[r][(g0 + i) >> 1].y : v[r][(g0 + i) >> 1].x;
                acc = fmaf(e, e, acc);
              }
            q[i] = acc;
          }
          int m = GS, off = 0;
#pragma unroll
          for (int o = 16; o >= TPV; o >>= 1) {  // lanes with bit o keep the upper half
            m >>= 1;
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int i = 0; i < m; ++i) {
              const float send = up ? q[i] : q[i + m];
              const float keep = up ? q[i + m] : q[i];
              q[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
            off += up ? m : 0;
          }
          s_acc[(g0 + off) * 32] += (double)q[0];
          s_acc[(g0 + off + 1) * 32] += (double)q[1];
        }
      }
      if constexpr (ENERGY) {
        acc_rows += VPT;
        if (acc_rows >= 128) {
          flush();
          acc_rows = 0;
        }
      }
    }
    if constexpr (ENERGY) flush();
    pos = stop;
  }
}

}  // namespace hygt_gpu
