// hygt_kernels.cuh -- sm_100a kernels of the batched HyGT hot path.
//
// Reference behaviour (paths under /root/reference/proj/include/hygt):
//   * detail::run_passes (transform.hpp:45-66): R rounds x log2N passes, pass p pairs (m, m+2^p)
//     with m = j + (j & -2^p) (hypercube.hpp:73-74), y_m = c*a + s*b, y_n = c*b - s*a
//     (givens.hpp:39-48); inverse = reverse order with -theta.
//   * forward gathers out[i] = pre[perm[i]] after the passes (transform.hpp:75-80), inverse
//     scatters first (:88-93); BASELINE configs add the same gathers between rounds.
//   * run_apply's per-block class dispatch (tools/hygt_main.cpp:143-149).
//
// B200 design: rows are streamed from HBM with 128-bit cache-streaming loads;
// a group of TPV lanes owns one row in registers (layout.h); in-register passes run as packed
// FFMA2 (fma.rn.f32x2 -- one instruction per butterfly in the scale-folded form); cross-lane
// passes use __shfl_xor_sync; permutations go through a bank-swizzled per-warp shared-memory
// scratch. Rows are visited in class-bucketed order so that the per-class coefficient stream a
// lane reads is (nearly always) warp-uniform, i.e. one broadcast per warp instead of one load per
// row. Coefficients are precomputed on the host in exactly the order each lane consumes them.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "layout.h"

namespace hygt_gpu {

typedef unsigned long long u64;

// ------------------------------------------------------------------ packed fp32x2 helpers ---
__device__ __forceinline__ u64 pk(float2 a) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
  return r;
}
__device__ __forceinline__ float2 upk(u64 a) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(a));
  return r;
}
// d = a * b + c, both halves, round-to-nearest (SASS FFMA2).
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  u64 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pk(a)), "l"(pk(b)), "l"(pk(c)));
  return upk(d);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  u64 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk(a)), "l"(pk(b)));
  return upk(d);
}
__device__ __forceinline__ float2 swap2(float2 a) { return make_float2(a.y, a.x); }
__device__ __forceinline__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }

// Per-lane xor applied to the element index inside the per-warp scratch row so that the 32
// lanes' stores of one slot hit 32 distinct banks ("permutation scratch").
HYGT_HD int scratch_swizzle(int g, int log2n, int l) {
  const int chl = log2n >= 2 ? 2 : log2n;
  const int by_stride = log2n < 5 ? 5 - log2n : 0;  // low group bits spread by the row stride
  int gb = g >> by_stride;
  const int limit = log2n < 5 ? log2n : 5;
  int out = 0;
  for (int b = 0; b < limit && gb; ++b) {
    if (b >= chl && b < chl + l) continue;  // lane bits are already distinct
    out |= (gb & 1) << b;
    gb >>= 1;
  }
  return out;
}

struct ApplyParams {
  const float* x;
  float* y;
  const uint32_t* idx;      // bucketed position -> row; nullptr = identity order
  const uint32_t* seg_end;  // flat [chunks][C+1] run ends; nullptr = every row is class 0
  uint32_t nseg;
  int classes;
  uint64_t count;
  const float2* coef;       // [C][TPV][stream_len] float2, this direction
  uint32_t stream_len;      // float2 words per lane stream (even)
  const uint16_t* gidx;     // [C][R+1][TPV][E] gather sources (element index), this direction
  uint64_t gmask;           // bit k: gather step k present (k = 0 before round slot 0, k = r+1 after)
  int rounds;
  uint64_t warp_span;       // positions per warp (multiple of the rows per warp)
  double* energy;           // [C][N] fp64 accumulators (forward + energy only)
};

// ---------------------------------------------------------------- one hypercube pass ----
template <int LOG2N, int L, bool STD, int P>
__device__ __forceinline__ void hygt_pass(float2 (&v)[(1 << LOG2N) / (1 << L) / 2],
                                          const float2*& cp) {
  constexpr Layout LY{LOG2N, L};
  constexpr int E = LY.e();
  constexpr int NP = E / 2;
  if constexpr (LY.cross(P)) {
    // Cross-lane pass: every own sample pairs with the same slot of lane t ^ mask.
    constexpr int LM = LY.lane_mask(P);
    auto partner = [&](int k) {
      return make_float2(__shfl_xor_sync(0xffffffffu, v[k].x, LM),
                         __shfl_xor_sync(0xffffffffu, v[k].y, LM));
    };
    if constexpr (!STD) {
      // scale-folded: own' = own + kappa * partner (kappa = t1 on the m side, -t2 on the n side)
      if constexpr (NP % 2 == 0) {
        const float4* c4 = reinterpret_cast<const float4*>(cp);
#pragma unroll
        for (int k = 0; k < NP; k += 2) {
          const float4 q = __ldg(c4 + k / 2);
          const float2 w0 = partner(k), w1 = partner(k + 1);
          v[k] = ffma2(make_float2(q.x, q.y), w0, v[k]);
          v[k + 1] = ffma2(make_float2(q.z, q.w), w1, v[k + 1]);
        }
      } else {
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          const float2 w0 = partner(k);
          v[k] = ffma2(__ldg(cp + k), w0, v[k]);
        }
      }
      cp += NP;
    } else {
      // standard: own' = c * own + (+-s) * partner, words (c pair, signed s pair) per sample pair
      const float4* c4 = reinterpret_cast<const float4*>(cp);
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const float4 q = __ldg(c4 + k);
        const float2 w0 = partner(k);
        v[k] = ffma2(make_float2(q.x, q.y), v[k], fmul2(make_float2(q.z, q.w), w0));
      }
      cp += 2 * NP;
    }
  } else if constexpr (P == 0) {
    // In-register pass on bit 0: the pair (m, m+1) is one 64-bit register pair.
    if constexpr (NP % 2 == 0) {
      const float4* c4 = reinterpret_cast<const float4*>(cp);
#pragma unroll
      for (int k = 0; k < NP; k += 2) {
        const float4 q = __ldg(c4 + k / 2);
        if constexpr (!STD) {
          // (y_m, y_n) = (a + t1 b, b - t2 a) = (t1, -t2) * (b, a) + (a, b)
          v[k] = ffma2(make_float2(q.x, q.y), swap2(v[k]), v[k]);
          v[k + 1] = ffma2(make_float2(q.z, q.w), swap2(v[k + 1]), v[k + 1]);
        } else {
          // (y_m, y_n) = c (a, b) + (s, -s) * (b, a)
          v[k] = ffma2(make_float2(q.x, q.x), v[k], fmul2(make_float2(q.y, -q.y), swap2(v[k])));
          v[k + 1] = ffma2(make_float2(q.z, q.z), v[k + 1],
                           fmul2(make_float2(q.w, -q.w), swap2(v[k + 1])));
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const float2 q = __ldg(cp + k);
        if constexpr (!STD)
          v[k] = ffma2(q, swap2(v[k]), v[k]);
        else
          v[k] = ffma2(make_float2(q.x, q.x), v[k], fmul2(make_float2(q.y, -q.y), swap2(v[k])));
      }
    }
    cp += NP;
  } else {
    // In-register pass on a higher bit: register pairs (m, m+1) and (m+k, m+k+1) hold two
    // butterflies j, j+1 whose coefficients are adjacent (one float4 per two butterflies).
    constexpr int SO = LY.slot_stride(P) / 2;  // partner distance in register pairs
    const float4* c4 = reinterpret_cast<const float4*>(cp);
    int k = 0;
#pragma unroll
    for (int a = 0; a < NP; ++a) {
      if ((a & SO) == 0) {
        const float4 q = __ldg(c4 + k);
        const float2 xa = v[a], xb = v[a + SO];
        if constexpr (!STD) {
          v[a] = ffma2(make_float2(q.x, q.y), xb, xa);       // a + t1 b
          v[a + SO] = ffma2(make_float2(q.z, q.w), xa, xb);  // b - t2 a
        } else {
          const float2 c = make_float2(q.x, q.y), s = make_float2(q.z, q.w);
          v[a] = ffma2(c, xa, fmul2(s, xb));
          v[a + SO] = ffma2(c, xb, fmul2(neg2(s), xa));
        }
        ++k;
      }
    }
    cp += NP;
  }
}

template <int LOG2N, int L, bool STD, bool FWD, int PP>
__device__ __forceinline__ void hygt_round(float2 (&v)[(1 << LOG2N) / (1 << L) / 2],
                                           const float2*& cp) {
  if constexpr (PP < LOG2N) {
    constexpr int P = FWD ? PP : LOG2N - 1 - PP;
    hygt_pass<LOG2N, L, STD, P>(v, cp);
    hygt_round<LOG2N, L, STD, FWD, PP + 1>(v, cp);
  }
}

// Gather v[s] <- pre[G[elem(t, s)]] through the warp's scratch rows.
template <int LOG2N, int L>
__device__ __forceinline__ void hygt_gather(float2 (&v)[(1 << LOG2N) / (1 << L) / 2],
                                            float* row, int t, int sw, const uint16_t* gp) {
  constexpr Layout LY{LOG2N, L};
  constexpr int E = LY.e();
  __syncwarp();
#pragma unroll
  for (int s = 0; s < E; s += 2) {
    row[LY.elem(t, s) ^ sw] = v[s / 2].x;
    row[LY.elem(t, s + 1) ^ sw] = v[s / 2].y;
  }
  __syncwarp();
  if constexpr (E % 8 == 0) {
    const uint4* g4 = reinterpret_cast<const uint4*>(gp);
#pragma unroll
    for (int s = 0; s < E; s += 8) {
      const uint4 q = __ldg(g4 + s / 8);
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        v[s / 2 + h].x = row[(w[h] & 0xffffu) ^ sw];
        v[s / 2 + h].y = row[(w[h] >> 16) ^ sw];
      }
    }
  } else {
#pragma unroll
    for (int s = 0; s < E; s += 2) {
      v[s / 2].x = row[__ldg(gp + s) ^ sw];
      v[s / 2].y = row[__ldg(gp + s + 1) ^ sw];
    }
  }
}

// ------------------------------------------------------------------- the apply kernel ---
// One warp walks a contiguous range of bucketed positions, 32/TPV rows per step.
template <int LOG2N, int L, bool STD, bool FWD, bool ENERGY>
__global__ void __launch_bounds__(256) hygt_apply_kernel(const ApplyParams P) {
  constexpr Layout LY{LOG2N, L};
  constexpr int N = LY.n(), TPV = LY.tpv(), E = LY.e(), CH = LY.ch(), V = 32 / TPV, NP = E / 2;
  extern __shared__ float hygt_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> L, t = lane & (TPV - 1);
  float* row_scratch = hygt_smem + (size_t)warp * (V * N) + g * N;
  const int sw = scratch_swizzle(g, LOG2N, L);
  const int C = P.classes;

  const uint64_t gw = (uint64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  const uint64_t wbeg = gw * P.warp_span;
  if (wbeg >= P.count) return;  // warp-uniform
  const uint64_t wend = (wbeg + P.warp_span < P.count) ? wbeg + P.warp_span : P.count;

  uint32_t f = 0;  // flat segment index: class = f % (C+1), bin C = invalid class id
  if (P.seg_end) {
    uint32_t lo = 0, hi = P.nseg;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if ((uint64_t)__ldg(P.seg_end + mid) <= wbeg) lo = mid + 1; else hi = mid;
    }
    f = lo;
  }

  float acc[ENERGY ? E : 1];
  int acc_class = -1, acc_rows = 0;
  if constexpr (ENERGY) {
#pragma unroll
    for (int s = 0; s < E; ++s) acc[s] = 0.f;
  }
  auto flush = [&]() {
    if constexpr (ENERGY) {
      if (acc_class >= 0 && acc_rows > 0) {
        double* e = P.energy + (size_t)acc_class * N;
#pragma unroll
        for (int s = 0; s < E; ++s) {
          atomicAdd(e + LY.elem(t, s), (double)acc[s]);
          acc[s] = 0.f;
        }
      }
      acc_rows = 0;
    }
  };

  for (uint64_t pos0 = wbeg; pos0 < wend; pos0 += V) {
    const uint64_t s = pos0 + g;
    const bool active = s < wend;
    int c = 0;
    if (P.seg_end) {
      while (f < P.nseg && (uint64_t)__ldg(P.seg_end + f) <= s) ++f;
      c = (int)(f % (uint32_t)(C + 1));
    }
    const bool passthrough = active && c >= C;  // invalid class id: copy, error already flagged
    if (c >= C) c = 0;
    const uint64_t row = active ? (P.idx ? (uint64_t)__ldg(P.idx + s) : s) : 0;
    const float* xr = P.x + row * N;

    float2 v[NP];
    if (active) {
#pragma unroll
      for (int u = 0; u < E / CH; ++u) {
        const int q = t + TPV * u;
        if constexpr (CH == 4) {
          const float4 a = __ldcs(reinterpret_cast<const float4*>(xr) + q);
          v[2 * u] = make_float2(a.x, a.y);
          v[2 * u + 1] = make_float2(a.z, a.w);
        } else {
          v[u] = __ldcs(reinterpret_cast<const float2*>(xr) + q);
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < NP; ++k) v[k] = make_float2(0.f, 0.f);
    }

    const float2* cp = P.coef + ((size_t)c * TPV + t) * P.stream_len;
    const uint16_t* gbase = P.gidx + (size_t)c * (P.rounds + 1) * TPV * E + (size_t)t * E;
    if (P.gmask & 1ull) hygt_gather<LOG2N, L>(v, row_scratch, t, sw, gbase);
    for (int r = 0; r < P.rounds; ++r) {
      hygt_round<LOG2N, L, STD, FWD, 0>(v, cp);
      if ((P.gmask >> (r + 1)) & 1ull)
        hygt_gather<LOG2N, L>(v, row_scratch, t, sw, gbase + (size_t)(r + 1) * TPV * E);
    }
    if constexpr (!STD) {
      // scale-folded form: undo the folded per-sample scales once at the end
#pragma unroll
      for (int k = 0; k < NP; ++k) v[k] = fmul2(v[k], __ldg(cp + k));
    }

    if (active) {
      float* yr = P.y + row * N;
      if (passthrough) {
#pragma unroll
        for (int u = 0; u < E / CH; ++u) {
          const int q = t + TPV * u;
          if constexpr (CH == 4)
            reinterpret_cast<float4*>(yr)[q] = reinterpret_cast<const float4*>(xr)[q];
          else
            reinterpret_cast<float2*>(yr)[q] = reinterpret_cast<const float2*>(xr)[q];
        }
      } else {
#pragma unroll
        for (int u = 0; u < E / CH; ++u) {
          const int q = t + TPV * u;
          if constexpr (CH == 4)
            __stcs(reinterpret_cast<float4*>(yr) + q,
                   make_float4(v[2 * u].x, v[2 * u].y, v[2 * u + 1].x, v[2 * u + 1].y));
          else
            __stcs(reinterpret_cast<float2*>(yr) + q, v[u]);
        }
        if constexpr (ENERGY) {
          if (c != acc_class || acc_rows >= 16) {  // fp32 partials of at most 16 rows
            flush();
            acc_class = c;
          }
#pragma unroll
          for (int k = 0; k < NP; ++k) {
            acc[2 * k] = fmaf(v[k].x, v[k].x, acc[2 * k]);
            acc[2 * k + 1] = fmaf(v[k].y, v[k].y, acc[2 * k + 1]);
          }
          ++acc_rows;
        }
      }
    }
  }
  flush();
}

}  // namespace hygt_gpu
