// hygt_seg2.cuh -- thread-per-row HyGT kernel for N = 64 (BASELINE config 3), over globally
// class-bucketed rows.
//
// Why it exists: the segment kernel (hygt_segment.cuh) gives a row two lanes, reads it from HBM
// as 32 B pieces of scattered rows and exchanges one pass per round by shuffles; its LSU data
// pipe runs at ~55 wavefronts per row (profiles/r01: 16 global, 8 shuffle, 17 permutation with
// bank conflicts, 13 coefficient), 2.4x the 22.7 clk/row HBM budget of a 256 B row.
//
// Here, per warp and batch of 64 bucketed rows (all of one class):
//   1. the row ids go to shared memory; the rows are copied in with cp.async, two rows (512
//      contiguous bytes) per warp instruction, into a per-warp slot area whose 272 B row stride
//      makes every later 16 B access bank-conflict-free;
//   2. each thread takes rows l and l + 32 into registers (64 fp32 each) and runs all rounds
//      there: every pass is in-register FFMA2, the coefficient units are warp-uniform LDS.128
//      broadcasts shared by the thread's two rows, permutations go through the slot area reused
//      as a [row][element][lane] scratch (conflict-free);
//   3. the rows go back to the slots and out to HBM two rows per coalesced STG.128.
// Tables: the element-ordered per-class streams of the staged kernel (hygt_stage.cuh), one class
// at a time in shared memory (6.4 KB at N = 64, R = 4).
#pragma once

#include "hygt_stage.cuh"

namespace hygt_gpu {

struct Seg2Params {
  const float* x;
  float* y;
  const uint32_t* idx;      // bucketed position -> row
  const uint32_t* seg_end;  // [C+1] end position of each class run (bin C = invalid ids)
  int classes;
  int rounds;
  uint64_t count;
  const float4* coef;       // [C][cw] element-ordered units (build_elem_tables)
  uint32_t cw;
  const uint16_t* gtab;     // [C][gstride] bytes: [R+1][N] u16 scratch offsets src * 128
  uint32_t gstride;
  uint64_t gmask;
  uint64_t cta_span;        // bucketed positions per CTA
};

HYGT_HD constexpr uint32_t seg2_row_stride(int log2n) { return (4u << log2n) + 16u; }

HYGT_HD constexpr uint32_t seg2_smem_bytes(int log2n, int vpt, int warps, uint32_t cw, uint32_t gstride) {
  return stage_align(cw * 16u, 128) + stage_align(gstride, 128) +
         (uint32_t)warps * (stage_align(32u * vpt * seg2_row_stride(log2n), 128) + 32u * vpt * 4u);
}

// One pass P on VPT rows of NW float2 words with the coefficients streamed a unit (4 floats) or
// two at a time; cb = shared address of this step's N/4 units (standard form: c units, then s').
template <int NW, int P, bool STD, int VPT>
__device__ __forceinline__ void seg2_pass(float2 (&v)[VPT][NW], uint32_t cb) {
  using namespace stage_detail;
  constexpr int NC = NW / 2;
  auto unit = [&](int c, float2& k0, float2& k1, float2& s0, float2& s1) {
    const float4 q = lds128(cb + c * 16);
    k0 = make_float2(q.x, q.y);
    k1 = make_float2(q.z, q.w);
    if constexpr (STD) {
      const float4 t = lds128(cb + (NC + c) * 16);
      s0 = make_float2(t.x, t.y);
      s1 = make_float2(t.z, t.w);
    }
  };
  if constexpr (P <= 1) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      float2 k0, k1, s0, s1;
      unit(c, k0, k1, s0, s1);
#pragma unroll
      for (int r = 0; r < VPT; ++r) {
        const float2 a = v[r][2 * c], b = v[r][2 * c + 1];
        if constexpr (P == 0) {
          if constexpr (!STD) {
            v[r][2 * c] = ffma2(k0, swap2(a), a);
            v[r][2 * c + 1] = ffma2(k1, swap2(b), b);
          } else {
            v[r][2 * c] = ffma2(k0, a, fmul2(s0, swap2(a)));
            v[r][2 * c + 1] = ffma2(k1, b, fmul2(s1, swap2(b)));
          }
        } else {
          if constexpr (!STD) {
            v[r][2 * c] = ffma2(k0, b, a);
            v[r][2 * c + 1] = ffma2(k1, a, b);
          } else {
            v[r][2 * c] = ffma2(k0, a, fmul2(s0, b));
            v[r][2 * c + 1] = ffma2(k1, b, fmul2(s1, a));
          }
        }
      }
    }
  } else {
    constexpr int MU = 1 << (P - 2);  // unit distance of the pair partner
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      if (c & MU) continue;
      float2 ka0, ka1, sa0, sa1, kb0, kb1, sb0, sb1;
      unit(c, ka0, ka1, sa0, sa1);
      unit(c + MU, kb0, kb1, sb0, sb1);
#pragma unroll
      for (int r = 0; r < VPT; ++r)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int wa = 2 * c + h, wb = 2 * (c + MU) + h;
          const float2 a = v[r][wa], b = v[r][wb];
          const float2 ka = h ? ka1 : ka0, kb = h ? kb1 : kb0;
          if constexpr (!STD) {
            v[r][wa] = ffma2(ka, b, a);
            v[r][wb] = ffma2(kb, a, b);
          } else {
            const float2 sa = h ? sa1 : sa0, sb = h ? sb1 : sb0;
            v[r][wa] = ffma2(ka, a, fmul2(sa, b));
            v[r][wb] = ffma2(kb, b, fmul2(sb, a));
          }
        }
    }
  }
}

template <int LOG2N, bool STD, bool FWD, int VPT, int PP>
__device__ __forceinline__ void seg2_round(float2 (&v)[VPT][(1 << LOG2N) / 2], uint32_t cb) {
  if constexpr (PP < LOG2N) {
    constexpr int P = FWD ? PP : LOG2N - 1 - PP;
    constexpr uint32_t STEP = (1u << LOG2N) / 4 * 16 * (STD ? 2 : 1);
    seg2_pass<(1 << LOG2N) / 2, P, STD, VPT>(v, cb + PP * STEP);
    seg2_round<LOG2N, STD, FWD, VPT, PP + 1>(v, cb);
  }
}

template <int LOG2N, int VPT, bool STD, bool FWD, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) hygt_seg2_kernel(const Seg2Params P) {
  using namespace stage_detail;
  constexpr int N = 1 << LOG2N, NW = N / 2, NC = N / 4;
  constexpr int THREADS = WARPS * 32, BATCH = 32 * VPT;
  constexpr uint32_t RS = seg2_row_stride(LOG2N);
  constexpr int RPI = 32 / NC;  // rows per coalesced warp instruction
  static_assert(NC <= 32 && 32 % NC == 0, "seg2: N in {16, ..., 128}");
  static_assert(VPT * N * 128 <= BATCH * RS, "seg2: permutation scratch must fit the slot area");
  extern __shared__ __align__(128) unsigned char smem[];
  const int C = P.classes;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t coef_bytes = stage_align(P.cw * 16u, 128);
  float4* s_coef = reinterpret_cast<float4*>(smem);
  uint32_t* s_gt = reinterpret_cast<uint32_t*>(smem + coef_bytes);
  const uint32_t warp_bytes = stage_align(BATCH * RS, 128) + BATCH * 4u;
  unsigned char* wslot = smem + coef_bytes + stage_align(P.gstride, 128) + warp * warp_bytes;
  uint32_t* s_row = reinterpret_cast<uint32_t*>(wslot + stage_align(BATCH * RS, 128));
  const uint32_t slot_s = su32(wslot);
  const uint32_t scr = slot_s + lane * 4u;
  const uint32_t coef_s = su32(s_coef), gt_s = su32(s_gt);
  __syncthreads();

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
    const uint64_t se = (uint64_t)__ldg(P.seg_end + f);
    const uint64_t stop = se < end ? se : end;
    const int c = (int)f;
    if (stop <= pos) continue;
    if (c >= C) {  // rows with invalid class ids: copied through (error flagged by hygt_bucket)
      for (uint64_t p = pos + tid / NC; p < stop; p += THREADS / NC) {
        const uint32_t row = __ldg(P.idx + p);
        const float4* xr = reinterpret_cast<const float4*>(P.x + (size_t)row * N);
        float4* yr = reinterpret_cast<float4*>(P.y + (size_t)row * N);
        yr[tid % NC] = xr[tid % NC];
      }
      pos = stop;
      continue;
    }
    __syncthreads();  // the previous segment's tables are no longer in use
    for (uint32_t i = tid; i < P.cw; i += THREADS) s_coef[i] = __ldg(P.coef + (size_t)c * P.cw + i);
    if (P.gmask)
      for (uint32_t i = tid; i < P.gstride / 4; i += THREADS)
        s_gt[i] = __ldg(reinterpret_cast<const uint32_t*>(P.gtab) + (size_t)c * (P.gstride / 4) + i);
    __syncthreads();
    // row ids of a batch, loaded one batch ahead so their latency hides behind the arithmetic
    auto load_ids = [&](uint64_t b0, uint32_t (&ids)[VPT]) {
#pragma unroll
      for (int r = 0; r < VPT; ++r) {
        const uint64_t i = b0 + lane + 32u * r;
        ids[r] = i < stop ? __ldg(P.idx + i) : 0xffffffffu;
      }
    };
    uint32_t ids_next[VPT];
    load_ids(pos + (uint64_t)warp * BATCH, ids_next);
    for (uint64_t bb = pos + (uint64_t)warp * BATCH; bb < stop; bb += (uint64_t)WARPS * BATCH) {
      __syncwarp();  // the previous batch's slot reads are done
#pragma unroll
      for (int r = 0; r < VPT; ++r) s_row[lane + 32u * r] = ids_next[r];
      load_ids(bb + (uint64_t)WARPS * BATCH, ids_next);
      __syncwarp();
      // rows -> slots: RPI rows of N / 4 chunks per warp instruction, 16 B cp.async each
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
      float2 v[VPT][NW];
#pragma unroll
      for (int r = 0; r < VPT; ++r)
#pragma unroll
        for (int q = 0; q < NC; ++q) {
          const float4 a = lds128(slot_s + (lane + 32u * r) * RS + q * 16);
          v[r][2 * q] = make_float2(a.x, a.y);
          v[r][2 * q + 1] = make_float2(a.z, a.w);
        }
      const uint32_t gbase = gt_s;
      if (P.gmask & 1ull) stage_gather<LOG2N, VPT, VPT>(v, scr, gbase, 0u, 0u);
      constexpr uint32_t ROUND = (uint32_t)LOG2N * NC * 16u * (STD ? 2u : 1u);
      for (int rr = 0; rr < P.rounds; ++rr) {
        seg2_round<LOG2N, STD, FWD, VPT, 0>(v, coef_s + (uint32_t)rr * ROUND);
        if ((P.gmask >> (rr + 1)) & 1ull)
          stage_gather<LOG2N, VPT, VPT>(v, scr, gbase + (uint32_t)(rr + 1) * N * 2u, 0u, 0u);
      }
      if constexpr (!STD) {  // remaining per-sample scales of the scale-folded form
        const uint32_t so = coef_s + (uint32_t)P.rounds * ROUND;
#pragma unroll
        for (int q = 0; q < NC; ++q) {
          const float4 s4 = lds128(so + q * 16);
#pragma unroll
          for (int r = 0; r < VPT; ++r) {
            v[r][2 * q] = fmul2(v[r][2 * q], make_float2(s4.x, s4.y));
            v[r][2 * q + 1] = fmul2(v[r][2 * q + 1], make_float2(s4.z, s4.w));
          }
        }
      }
      __syncwarp();  // scratch reads of the last permutation are done
#pragma unroll
      for (int r = 0; r < VPT; ++r)
#pragma unroll
        for (int q = 0; q < NC; ++q)
          sts128(slot_s + (lane + 32u * r) * RS + q * 16,
                 make_float4(v[r][2 * q].x, v[r][2 * q].y, v[r][2 * q + 1].x, v[r][2 * q + 1].y));
      __syncwarp();
#pragma unroll 4
      for (uint32_t i0 = 0; i0 < BATCH; i0 += RPI) {
        const uint32_t i = i0 + lane / NC, q = lane % NC;
        const uint32_t row = s_row[i];
        if (row != 0xffffffffu)
          __stcs(reinterpret_cast<float4*>(P.y + (size_t)row * N) + q, lds128(slot_s + i * RS + q * 16));
      }
    }
    pos = stop;
  }
}

}  // namespace hygt_gpu
