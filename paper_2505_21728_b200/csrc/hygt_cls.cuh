// hygt_cls.cuh -- one launch per class: the class's coefficient stream travels as kernel
// parameters, so every butterfly reads its coefficient as a constant-bank FFMA operand.
//
// Why it exists: over globally class-bucketed rows the thread-per-row kernel (hygt_seg2.cuh)
// spends 12.5 of its ~40 LSU data-pipe wavefronts per N = 64 row on warp-uniform LDS.128
// broadcasts of the class table (profiles/r01). Every lane of a warp needs the same coefficient
// at the same instruction there, which is exactly what the constant bank serves without touching
// the LSU pipe -- but a constant operand needs a compile-time offset, and 35 classes of tables
// (215 KB per direction at N = 64, R = 4) do not fit one 64 KB bank. So the plan keeps one
// parameter block per class and direction (coefficients + gather offsets, 7.7 KB at N = 64,
// R = 4) and launches one grid per class over that class's bucketed range:
//
//   * `FFMA y, c[0x0][k_i], x_partner, y` per element and pass (scale-folded form, the element
//     streams of build_elem_tables), `FMUL` by c[0x0][scale_i] at the end;
//   * rows arrive through a per-warp shared slot area with cp.async (two rows per warp
//     instruction), leave through it as coalesced STG.128;
//   * permutations go through a conflict-free [element][lane] scratch (the slot area again),
//     the gather offsets being parameter words as well.
//
// Launch chain: the class grids are issued back to back on one stream with programmatic
// stream serialisation. Each grid triggers its dependent at entry (the grids are independent:
// different rows), so class c + 1's warps start as soon as class c's warps leave the SMs and the
// per-launch tails overlap; each grid waits on its predecessor's completion before it exits, so
// the last grid's completion (what the stream orders later work on) implies all of them.
//
// Reference semantics: run_passes / forward / inverse (transform.hpp:45-96), coefficient tables
// from build_programs() (hygt_plan.cpp) -- the same fp64 (c, s) per butterfly as every path.
#pragma once

#include <cstdint>

#include "hygt_stage.cuh"

namespace hygt_gpu {

// Parameter block of one class launch. Stays below the 32764-byte kernel parameter limit for
// N = 64 up to R = 8 (coef: (R * log2N + 1) * N / 4 float4, gat: (R + 1) * N u32).
template <int LOG2N, int R>
struct ClsParams {
  static constexpr int N = 1 << LOG2N, NC = N / 4;
  static constexpr int CW = R * LOG2N * NC + NC;
  const float* x;
  float* y;
  const uint32_t* idx;      // bucketed position -> row
  const uint32_t* seg_end;  // [C + 1] end of each class run; bin C = invalid class ids
  uint32_t bin;             // class of this launch
  uint32_t copy_bin;        // != 0: afterwards copy bin `bin + 1` (invalid ids) through
  uint32_t gmask;           // gather steps present (bit k: before round k, k = R: final)
  uint32_t pad_;
  float4 coef[CW];          // element-ordered k_i per step, then the final scales
  uint32_t gat[R + 1][N];   // scratch byte offsets src * 128 per gather step
};

HYGT_HD constexpr uint32_t cls_row_stride(int log2n) { return (4u << log2n) + 16u; }
// per-warp shared memory: VPT * 32 row slots (also the [row][element][lane] permutation
// scratch) and the batch's row ids
HYGT_HD constexpr uint32_t cls_warp_bytes(int log2n, int vpt) {
  return 32u * vpt * cls_row_stride(log2n) + 128u * vpt;
}

namespace cls_detail {

template <int LOG2N, int R, int VPT, int S, bool FWD>
__device__ __forceinline__ void pass_step(float (&v)[VPT][1 << LOG2N], const ClsParams<LOG2N, R>& P) {
  constexpr int N = 1 << LOG2N;
  constexpr int PP = S % LOG2N;
  constexpr int B = 1 << (FWD ? PP : LOG2N - 1 - PP);
  const float* k = reinterpret_cast<const float*>(&P.coef[S * (N / 4)]);
#pragma unroll
  for (int m = 0; m < N; ++m) {
    if (m & B) continue;
#pragma unroll
    for (int r = 0; r < VPT; ++r) {
      const float a = v[r][m], b = v[r][m | B];
      v[r][m] = fmaf(k[m], b, a);          // y_m = x_m + t1 x_n   (scale-folded butterfly)
      v[r][m | B] = fmaf(k[m | B], a, b);  // y_n = x_n - t2 x_m   (k_n = -t2)
    }
  }
}

template <int LOG2N, int R, int VPT, int S, bool FWD>
__device__ __forceinline__ void round_steps(float (&v)[VPT][1 << LOG2N], const ClsParams<LOG2N, R>& P) {
  pass_step<LOG2N, R, VPT, S, FWD>(v, P);
  if constexpr ((S + 1) % LOG2N != 0) round_steps<LOG2N, R, VPT, S + 1, FWD>(v, P);
}

// Permutation k (gather out[i] = in[src_i]) through the [row][element][lane] scratch.
template <int LOG2N, int R, int VPT>
__device__ __forceinline__ void gather(float (&v)[VPT][1 << LOG2N], const ClsParams<LOG2N, R>& P, int k,
                                       uint32_t scr) {
  constexpr int N = 1 << LOG2N;
  __syncwarp();
#pragma unroll
  for (int r = 0; r < VPT; ++r)
#pragma unroll
    for (int i = 0; i < N; ++i) stage_detail::sts32(scr + (uint32_t)(r * N + i) * 128u, v[r][i]);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const uint32_t a = scr + P.gat[k][i];
#pragma unroll
    for (int r = 0; r < VPT; ++r) v[r][i] = stage_detail::lds32(a + (uint32_t)(r * N) * 128u);
  }
}

template <int LOG2N, int R, int VPT, int RR, bool FWD>
__device__ __forceinline__ void rounds(float (&v)[VPT][1 << LOG2N], const ClsParams<LOG2N, R>& P, uint32_t scr) {
  if constexpr (RR < R) {
    round_steps<LOG2N, R, VPT, RR * LOG2N, FWD>(v, P);
    if ((P.gmask >> (RR + 1)) & 1u) gather<LOG2N, R, VPT>(v, P, RR + 1, scr);
    rounds<LOG2N, R, VPT, RR + 1, FWD>(v, P, scr);
  }
}

}  // namespace cls_detail

// One warp per CTA; a thread owns VPT rows of a batch of 32 * VPT bucketed rows of the class,
// and warps take batches round-robin over the grid.
template <int LOG2N, int R, int VPT, bool FWD>
__global__ void __launch_bounds__(32, VPT == 1 ? 1 : 10) hygt_cls_kernel(const __grid_constant__ ClsParams<LOG2N, R> P) {
  using namespace stage_detail;
  constexpr int N = 1 << LOG2N, NC = N / 4, BATCH = 32 * VPT;
  constexpr uint32_t RS = cls_row_stride(LOG2N);
  constexpr int RPI = 32 / NC;  // rows per coalesced warp instruction
  static_assert(NC <= 32 && 32 % NC == 0, "cls: N in {16, ..., 128}");
  static_assert(N * 128 <= 32 * RS, "cls: permutation scratch must fit the slot area");
  extern __shared__ __align__(128) unsigned char smem[];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x;
  const uint32_t slot_s = su32(smem);
  uint32_t* s_row = reinterpret_cast<uint32_t*>(smem + BATCH * RS);
  const uint32_t scr = slot_s + lane * 4u;

  const uint64_t beg = P.bin ? __ldg(P.seg_end + P.bin - 1) : 0u;
  const uint64_t end = __ldg(P.seg_end + P.bin);
  const uint64_t nb = (end - beg + BATCH - 1) / BATCH;
  // row ids of this lane in batch b (~0u past the class run)
  auto row_ids = [&](uint64_t b, uint32_t (&ids)[VPT]) {
#pragma unroll
    for (int r = 0; r < VPT; ++r) {
      const uint64_t p = beg + b * BATCH + lane + 32 * r;
      ids[r] = b < nb && p < end ? __ldg(P.idx + p) : 0xffffffffu;
    }
  };
  uint32_t id_next[VPT];
  row_ids(blockIdx.x, id_next);
  for (uint64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    __syncwarp();
#pragma unroll
    for (int r = 0; r < VPT; ++r) s_row[lane + 32 * r] = id_next[r];
    row_ids(b + gridDim.x, id_next);  // one batch ahead: its rows are prefetched into L2 below
    __syncwarp();
#pragma unroll 4
    for (uint32_t i0 = 0; i0 < BATCH; i0 += RPI) {
      const uint32_t i = i0 + lane / NC, q = lane % NC;
      const uint32_t row = s_row[i];
      if (row != 0xffffffffu)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(slot_s + i * RS + q * 16),
                     "l"(P.x + (size_t)row * N + q * 4)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    float v[VPT][N];
#pragma unroll
    for (int r = 0; r < VPT; ++r)
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        const float4 a = lds128(slot_s + (lane + 32 * r) * RS + q * 16);
        v[r][4 * q] = a.x;
        v[r][4 * q + 1] = a.y;
        v[r][4 * q + 2] = a.z;
        v[r][4 * q + 3] = a.w;
      }
    if (P.gmask & 1u) cls_detail::gather<LOG2N, R, VPT>(v, P, 0, scr);
    cls_detail::round_steps<LOG2N, R, VPT, 0, FWD>(v, P);
#pragma unroll
    for (int r = 0; r < VPT; ++r)  // the next batch's rows: in L2 by the time this batch is done
      if (id_next[r] != 0xffffffffu)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(P.x + (size_t)id_next[r] * N), "n"(N * 4)
                     : "memory");
    if ((P.gmask >> 1) & 1u) cls_detail::gather<LOG2N, R, VPT>(v, P, 1, scr);
    cls_detail::rounds<LOG2N, R, VPT, 1, FWD>(v, P, scr);
    {
      const float* s = reinterpret_cast<const float*>(&P.coef[R * LOG2N * NC]);
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int r = 0; r < VPT; ++r) v[r][i] *= s[i];
    }
    __syncwarp();  // scratch reads of the last permutation are done
#pragma unroll
    for (int r = 0; r < VPT; ++r)
#pragma unroll
      for (int q = 0; q < NC; ++q)
        sts128(slot_s + (lane + 32 * r) * RS + q * 16,
               make_float4(v[r][4 * q], v[r][4 * q + 1], v[r][4 * q + 2], v[r][4 * q + 3]));
    __syncwarp();
#pragma unroll 4
    for (uint32_t i0 = 0; i0 < BATCH; i0 += RPI) {
      const uint32_t i = i0 + lane / NC, q = lane % NC;
      const uint32_t row = s_row[i];
      if (row != 0xffffffffu)
        __stcs(reinterpret_cast<float4*>(P.y + (size_t)row * N) + q, lds128(slot_s + i * RS + q * 16));
    }
  }
  if (P.copy_bin) {  // rows with invalid class ids are copied through (hygt_bucket flags them)
    const uint64_t e2 = __ldg(P.seg_end + P.bin + 1);
    for (uint64_t p = end + (uint64_t)blockIdx.x * (32 / NC) + lane / NC; p < e2; p += (uint64_t)gridDim.x * (32 / NC)) {
      const uint32_t row = __ldg(P.idx + p);
      reinterpret_cast<float4*>(P.y + (size_t)row * N)[lane % NC] =
          reinterpret_cast<const float4*>(P.x + (size_t)row * N)[lane % NC];
    }
  }
  // complete only after the previous class grid has: the stream's next operation then follows
  // every grid of the chain
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

}  // namespace hygt_gpu
