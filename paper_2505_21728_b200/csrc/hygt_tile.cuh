// hygt_tile.cuh -- the "tile" HyGT kernel for short rows (N <= 32, all class tables fit in shared
// memory): the production path of BASELINE configs 1 and 2.
//
// Per CTA (persistent, grid-stride over tiles of T rows):
//   1. the direction's coefficient / scale / gather tables of ALL classes are staged once into
//      shared memory (lane-interleaved so the TPV lanes of a row read one contiguous 16*TPV-byte
//      run: one shared-memory wavefront per warp load when the warp is class-uniform);
//   2. each tile's class ids are counting-sorted in shared memory (warp-aggregated atomics) --
//      the batched equivalent of run_apply's cache[b.class_id] dispatch (hygt_main.cpp:143-149)
//      without any index array in HBM;
//   3. warps walk the sorted positions, VPT rows per lane-group, gathering rows from HBM with
//      128-bit loads (a row is TPV consecutive lanes: coalesced), running all rounds in registers
//      (packed FFMA2 butterflies, __shfl_xor_sync for the lane bits, bank-swizzled scratch for
//      the permutations) and streaming the rows back.
// The VPT rows of a lane group share every coefficient load when they have the same class
// (always, except at class-run boundaries where a per-row fallback runs).
#pragma once

#include "hygt_kernels.cuh"

namespace hygt_gpu {

struct TileParams {
  const float* x;
  float* y;
  const uint16_t* cls;      // nullptr: single class
  uint64_t count;
  int classes;
  int rounds;
  const float4* coef;       // [C][units][TPV] float4, units = stream_len / 2
  uint32_t units;           // float4 units per lane stream
  const uint4* gidx;        // [C][R+1][E/8][TPV] uint4 (8 u16 gather sources per uint4)
  uint64_t gmask;
  uint32_t tile_rows;       // T
  double* energy;           // [C][N] (forward + energy)
  uint32_t* err;            // class id out of range flag
  int load_policy;          // 0 ld.global.cs, 1 ld.global.nc, 2 nc + L2::128B prefetch, 3 nc + evict_last
};

__device__ __forceinline__ float4 ld_row(const float4* p, int policy) {
  float4 r;
  switch (policy) {
    case 0: return __ldcs(p);
    case 1: return __ldg(p);
    case 2:
      asm volatile("ld.global.nc.L1::no_allocate.L2::128B.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
      return r;
    default:
      asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
      return r;
  }
}

template <int LOG2N, int L>
struct TileGeom {
  static constexpr Layout LY{LOG2N, L};
  static constexpr int N = LY.n(), TPV = LY.tpv(), E = LY.e(), CH = LY.ch(), NP = E / 2;
  static constexpr int V = 32 / TPV;  // rows per warp per VPT slot
  // Scratch row stride (floats) for VPT rows per lane group: ROWS = V * VPT row slots, padded so
  // that S * 4 == V (mod 32) -- the 32 lanes' stores of one register slot then land in 32
  // distinct banks (lane bits of the element index times S*4 fill the banks V apart).
  template <int VPT>
  HYGT_HD static constexpr int stride() {
    constexpr int rows = V * VPT;
    constexpr int want = (V / 4) % 8;
    return rows + ((want - rows % 8) % 8 + 8) % 8 + (TPV == 1 ? 0 : 0);
  }
};

// One pass on VPT rows. SHARED: all VPT rows share the coefficient stream cp[0].
template <int LOG2N, int L, bool STD, int P, int VPT, bool SHARED>
__device__ __forceinline__ void tile_pass(float2 (&v)[VPT][TileGeom<LOG2N, L>::NP],
                                          const float4* (&cp)[VPT]) {
  using G = TileGeom<LOG2N, L>;
  constexpr Layout LY = G::LY;
  constexpr int NP = G::NP, TPV = G::TPV;
  auto ld = [&](int r, int u) -> float4 { return cp[SHARED ? 0 : r][u * TPV]; };
  if constexpr (LY.cross(P)) {
    constexpr int LM = LY.lane_mask(P);
    if constexpr (!STD) {
#pragma unroll
      for (int k = 0; k < NP; k += 2) {
        float4 q = ld(0, k / 2);
#pragma unroll
        for (int r = 0; r < VPT; ++r) {
          if (!SHARED && r) q = ld(r, k / 2);
          const float2 w0 = make_float2(__shfl_xor_sync(0xffffffffu, v[r][k].x, LM),
                                        __shfl_xor_sync(0xffffffffu, v[r][k].y, LM));
          const float2 w1 = make_float2(__shfl_xor_sync(0xffffffffu, v[r][k + 1].x, LM),
                                        __shfl_xor_sync(0xffffffffu, v[r][k + 1].y, LM));
          v[r][k] = ffma2(make_float2(q.x, q.y), w0, v[r][k]);
          v[r][k + 1] = ffma2(make_float2(q.z, q.w), w1, v[r][k + 1]);
        }
      }
#pragma unroll
      for (int r = 0; r < VPT; ++r) cp[r] += (NP / 2) * TPV;
    } else {
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        float4 q = ld(0, k);
#pragma unroll
        for (int r = 0; r < VPT; ++r) {
          if (!SHARED && r) q = ld(r, k);
          const float2 w0 = make_float2(__shfl_xor_sync(0xffffffffu, v[r][k].x, LM),
                                        __shfl_xor_sync(0xffffffffu, v[r][k].y, LM));
          v[r][k] = ffma2(make_float2(q.x, q.y), v[r][k], fmul2(make_float2(q.z, q.w), w0));
        }
      }
#pragma unroll
      for (int r = 0; r < VPT; ++r) cp[r] += NP * TPV;
    }
  } else if constexpr (P == 0) {
#pragma unroll
    for (int k = 0; k < NP; k += 2) {
      float4 q = ld(0, k / 2);
#pragma unroll
      for (int r = 0; r < VPT; ++r) {
        if (!SHARED && r) q = ld(r, k / 2);
        if constexpr (!STD) {
          v[r][k] = ffma2(make_float2(q.x, q.y), swap2(v[r][k]), v[r][k]);
          v[r][k + 1] = ffma2(make_float2(q.z, q.w), swap2(v[r][k + 1]), v[r][k + 1]);
        } else {
          v[r][k] = ffma2(make_float2(q.x, q.x), v[r][k], fmul2(make_float2(q.y, -q.y), swap2(v[r][k])));
          v[r][k + 1] = ffma2(make_float2(q.z, q.z), v[r][k + 1],
                              fmul2(make_float2(q.w, -q.w), swap2(v[r][k + 1])));
        }
      }
    }
#pragma unroll
    for (int r = 0; r < VPT; ++r) cp[r] += (NP / 2) * TPV;
  } else {
    constexpr int SO = LY.slot_stride(P) / 2;
    int u = 0;
#pragma unroll
    for (int a = 0; a < NP; ++a) {
      if ((a & SO) == 0) {
        float4 q = ld(0, u);
#pragma unroll
        for (int r = 0; r < VPT; ++r) {
          if (!SHARED && r) q = ld(r, u);
          const float2 xa = v[r][a], xb = v[r][a + SO];
          if constexpr (!STD) {
            v[r][a] = ffma2(make_float2(q.x, q.y), xb, xa);
            v[r][a + SO] = ffma2(make_float2(q.z, q.w), xa, xb);
          } else {
            const float2 c = make_float2(q.x, q.y), s = make_float2(q.z, q.w);
            v[r][a] = ffma2(c, xa, fmul2(s, xb));
            v[r][a + SO] = ffma2(c, xb, fmul2(neg2(s), xa));
          }
        }
        ++u;
      }
    }
#pragma unroll
    for (int r = 0; r < VPT; ++r) cp[r] += (NP / 2) * TPV;
  }
}

template <int LOG2N, int L, bool STD, bool FWD, int VPT, bool SHARED, int PP>
__device__ __forceinline__ void tile_round(float2 (&v)[VPT][TileGeom<LOG2N, L>::NP],
                                          const float4* (&cp)[VPT]) {
  if constexpr (PP < LOG2N) {
    constexpr int P = FWD ? PP : LOG2N - 1 - PP;
    tile_pass<LOG2N, L, STD, P, VPT, SHARED>(v, cp);
    tile_round<LOG2N, L, STD, FWD, VPT, SHARED, PP + 1>(v, cp);
  }
}

// Gather v[r][s] <- pre[G[elem(t, s)]] through the warp's scratch. Element i of the row in slot
// (r, g) lives at scratch[i * S + r * V + g] (S = stride<VPT>(): the 32 lanes' stores of one
// register slot land in 32 distinct banks). `wbase` is this lane's store base
// (scratch + g + (t << chl) * S, so every store is [reg + imm]); `rbase` = scratch + g. The
// gather words hold the source elements pre-multiplied by 4*S (byte offsets, host-computed),
// so every load is one IADD + LDS [reg + imm].
template <int LOG2N, int L, int VPT>
__device__ __forceinline__ void tile_gather(float2 (&v)[VPT][TileGeom<LOG2N, L>::NP],
                                            float* wbase, const char* rbase,
                                            const uint4* (&gp)[VPT]) {
  using G = TileGeom<LOG2N, L>;
  constexpr Layout LY = G::LY;
  constexpr int E = G::E, TPV = G::TPV, V = G::V;
  constexpr int S = G::template stride<VPT>();
  __syncwarp();
#pragma unroll
  for (int r = 0; r < VPT; ++r)
#pragma unroll
    for (int s = 0; s < E; s += 2) {
      // elem(t, s) = (t << chl) + elem(0, s): the lane part is folded into wbase
      wbase[(LY.elem(0, s)) * S + r * V] = v[r][s / 2].x;
      wbase[(LY.elem(0, s + 1)) * S + r * V] = v[r][s / 2].y;
    }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < VPT; ++r) {
    const char* rb = rbase + r * V * 4;
    auto at = [&](uint32_t off) { return *reinterpret_cast<const float*>(rb + off); };
    if constexpr (E % 8 == 0) {
#pragma unroll
      for (int s = 0; s < E; s += 8) {
        const uint4 q = gp[r][(s / 8) * TPV];
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          v[r][s / 2 + h].x = at(w[h] & 0xffffu);
          v[r][s / 2 + h].y = at(w[h] >> 16);
        }
      }
    } else {
      const uint4 q = gp[r][0];
      v[r][0].x = at(q.x & 0xffffu);
      v[r][0].y = at(q.x >> 16);
      v[r][1].x = at(q.y & 0xffffu);
      v[r][1].y = at(q.y >> 16);
    }
  }
}

template <int LOG2N, int L, bool STD, bool FWD, int VPT, bool SHARED>
__device__ __forceinline__ void tile_rows(float2 (&v)[VPT][TileGeom<LOG2N, L>::NP],
                                          const float4* (&cp)[VPT], const uint4* (&g0)[VPT],
                                          uint32_t gstep_words, float* wbase, const char* rbase,
                                          const int rounds, const uint64_t gmask) {
  const uint4* gp[VPT];
#pragma unroll
  for (int r = 0; r < VPT; ++r) gp[r] = g0[r];
  if (gmask & 1ull) tile_gather<LOG2N, L, VPT>(v, wbase, rbase, gp);
  for (int rr = 0; rr < rounds; ++rr) {
    tile_round<LOG2N, L, STD, FWD, VPT, SHARED, 0>(v, cp);
    if ((gmask >> (rr + 1)) & 1ull) {
#pragma unroll
      for (int r = 0; r < VPT; ++r) gp[r] = g0[r] + (size_t)(rr + 1) * gstep_words;
      tile_gather<LOG2N, L, VPT>(v, wbase, rbase, gp);
    }
  }
  if constexpr (!STD) {
    using G = TileGeom<LOG2N, L>;
#pragma unroll
    for (int k = 0; k < G::NP; k += 2) {
      float4 q = cp[0][(k / 2) * G::TPV];
#pragma unroll
      for (int r = 0; r < VPT; ++r) {
        if (!SHARED && r) q = cp[r][(k / 2) * G::TPV];
        v[r][k] = fmul2(v[r][k], make_float2(q.x, q.y));
        v[r][k + 1] = fmul2(v[r][k + 1], make_float2(q.z, q.w));
      }
    }
  }
}

// Shared-memory footprint of one CTA (bytes), given the table sizes.
HYGT_HD constexpr size_t tile_smem_bytes(size_t coef_bytes, size_t gidx_bytes, int classes,
                                         int tile_rows, int warps, int scratch_floats_per_warp) {
  return ((coef_bytes + 15) & ~size_t(15)) + ((gidx_bytes + 15) & ~size_t(15)) +
         ((size_t)(classes + 2 + 3) / 4 * 4) * 4 +         // run offsets
         ((size_t)(tile_rows + 3) / 4 * 4) * 4 +            // sorted entries (class << 16 | row)
         (size_t)warps * scratch_floats_per_warp * 4;
}

template <int LOG2N, int L, int VPT, bool STD, bool FWD, bool ENERGY, int THREADS>
__global__ void __launch_bounds__(THREADS, THREADS >= 512 ? 2 : 3) hygt_tile_kernel(const TileParams P) {
  using G = TileGeom<LOG2N, L>;
  constexpr Layout LY = G::LY;
  constexpr int N = G::N, TPV = G::TPV, E = G::E, CH = G::CH, NP = G::NP, V = G::V;
  constexpr int ROWS = V * VPT;  // rows per warp step
  constexpr int WARPS = THREADS / 32;
  constexpr int S = G::template stride<VPT>();
  constexpr int SCR = N * S;  // scratch floats per warp
  extern __shared__ __align__(16) unsigned char tile_smem[];
  const int C = P.classes;
  const int T = (int)P.tile_rows;
  const size_t coef_words = (size_t)C * P.units * TPV;  // float4
  const size_t gidx_words = P.gmask ? (size_t)C * (P.rounds + 1) * ((E + 7) / 8) * TPV : 0;
  float4* s_coef = reinterpret_cast<float4*>(tile_smem);
  uint4* s_gidx = reinterpret_cast<uint4*>(s_coef + coef_words);
  uint32_t* s_off = reinterpret_cast<uint32_t*>(s_gidx + gidx_words);  // [C+2]
  uint32_t* s_ent = s_off + ((C + 2 + 3) & ~3);                         // [T] (class << 16 | row)
  float* s_scratch = reinterpret_cast<float*>(s_ent + ((T + 3) & ~3));

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> L, t = lane & (TPV - 1);
  float* wscr = s_scratch + (size_t)warp * SCR;
  float* wbase = wscr + g + ((t << LY.chl()) * S);
  const char* rbase = reinterpret_cast<const char*>(wscr + g);
  const bool sorted = P.cls && C > 1;

  for (size_t i = tid; i < coef_words; i += THREADS) s_coef[i] = __ldg(P.coef + i);
  for (size_t i = tid; i < gidx_words; i += THREADS) s_gidx[i] = __ldg(P.gidx + i);
  const uint32_t gstep_words = ((E + 7) / 8) * TPV;
  const uint64_t tiles = (P.count + T - 1) / T;

  // class ids of a tile: IDS consecutive rows per thread (T == IDS * THREADS), 128-bit loads,
  // prefetched one tile ahead so the sort never waits on HBM
  constexpr int IDS = THREADS >= 512 ? 8 : 16;
  auto load_ids = [&](uint64_t tl, uint32_t (&q)[IDS / 2]) {
#pragma unroll
    for (int w = 0; w < IDS / 2; ++w) q[w] = 0;
    if (!sorted || tl >= tiles) return;
    const uint64_t r0 = tl * T + (uint64_t)tid * IDS;
    if (r0 + IDS <= P.count && ((reinterpret_cast<uintptr_t>(P.cls + r0) & 15) == 0)) {
#pragma unroll
      for (int w = 0; w < IDS / 8; ++w) {
        const uint4 v = __ldcs(reinterpret_cast<const uint4*>(P.cls + r0) + w);
        q[4 * w] = v.x; q[4 * w + 1] = v.y; q[4 * w + 2] = v.z; q[4 * w + 3] = v.w;
      }
    } else {
      for (int h = 0; h < IDS; ++h)
        if (r0 + h < P.count) q[h >> 1] |= (uint32_t)P.cls[r0 + h] << (16 * (h & 1));
    }
  };
  uint32_t ids[IDS / 2], ids_next[IDS / 2];
  load_ids(blockIdx.x, ids);
  for (uint64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const uint64_t row0 = tile * T;
    const int rows = (int)((P.count - row0) < (uint64_t)T ? (P.count - row0) : (uint64_t)T);
    const float* xt = P.x + row0 * N;
    float* yt = P.y + row0 * N;
    __syncthreads();
    if (sorted) {  // counting sort of the tile by class (bin C = invalid id)
      for (int i = tid; i < C + 2; i += THREADS) s_off[i] = 0;
      __syncthreads();
#pragma unroll
      for (int h = 0; h < IDS; ++h) {
        int c = (ids[h >> 1] >> (16 * (h & 1))) & 0xffff;
        c = c < C ? c : C;
        if (tid * IDS + h < rows) atomicAdd(&s_off[c + 1], 1u);  // lanes serialise in the ATOMS unit
      }
      __syncthreads();
      if (warp == 0) {
        uint32_t carry = 0;
        for (int base = 1; base < C + 2; base += 32) {
          const int i = base + lane;
          uint32_t v0 = i < C + 2 ? s_off[i] : 0;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t n = __shfl_up_sync(0xffffffffu, v0, o);
            if (lane >= o) v0 += n;
          }
          if (i < C + 2) s_off[i] = v0 + carry;
          carry += __shfl_sync(0xffffffffu, v0, 31);
        }
      }
      __syncthreads();
#pragma unroll
      for (int h = 0; h < IDS; ++h) {
        const int i = tid * IDS + h;
        int c = (ids[h >> 1] >> (16 * (h & 1))) & 0xffff;
        if (i < rows) {
          if (c >= C) {
            c = C;
            atomicOr(P.err, 1u);
          }
          // unstable within a class: the order only affects which warp handles a row
          const uint32_t b = atomicAdd(&s_off[c], 1u);
          s_ent[b] = ((uint32_t)c << 16) | (uint32_t)i;
        }
      }
      load_ids(tile + gridDim.x, ids_next);
      __syncthreads();
#pragma unroll
      for (int h = 0; h < IDS / 2; ++h) ids[h] = ids_next[h];
    }

    // entry of sorted position p: (class << 16) | local row; inactive positions map to row 0
    auto entry = [&](int p) -> uint32_t {
      if (p >= rows) return 0u;
      if (sorted) return s_ent[p];
      uint32_t c = P.cls ? (uint32_t)P.cls[row0 + p] : 0u;
      if (c >= (uint32_t)C) {
        atomicOr(P.err, 1u);
        c = (uint32_t)C;
      }
      return (c << 16) | (uint32_t)p;
    };
    auto load = [&](const uint32_t (&en)[VPT], float2 (&dst)[VPT][NP]) {
#pragma unroll
      for (int r = 0; r < VPT; ++r) {
        const float4* xr = reinterpret_cast<const float4*>(xt + (size_t)(en[r] & 0xffffu) * N);
#pragma unroll
        for (int u = 0; u < E / CH; ++u) {
          const float4 a = ld_row(xr + t + TPV * u, P.load_policy);
          dst[r][2 * u] = make_float2(a.x, a.y);
          dst[r][2 * u + 1] = make_float2(a.z, a.w);
        }
      }
    };

    int p0 = warp * ROWS;
    uint32_t en_n[VPT];
    float2 vn[VPT][NP];
#pragma unroll
    for (int r = 0; r < VPT; ++r) en_n[r] = entry(p0 + r * V + g);
    if (p0 < rows) load(en_n, vn);
    for (; p0 < rows; p0 += WARPS * ROWS) {
      uint32_t en[VPT];
      float2 v[VPT][NP];
#pragma unroll
      for (int r = 0; r < VPT; ++r) {
        en[r] = en_n[r];
#pragma unroll
        for (int k = 0; k < NP; ++k) v[r][k] = vn[r][k];
      }
      const int pn = p0 + WARPS * ROWS;  // prefetch the next step's rows
      if (pn < rows) {
#pragma unroll
        for (int r = 0; r < VPT; ++r) en_n[r] = entry(pn + r * V + g);
        load(en_n, vn);
      }
      const float4* cp[VPT];
      const uint4* gp[VPT];
      bool same = true;
#pragma unroll
      for (int r = 0; r < VPT; ++r) {
        uint32_t c = en[r] >> 16;
        c = c < (uint32_t)C ? c : 0u;
        cp[r] = s_coef + (size_t)c * P.units * TPV + t;
        gp[r] = s_gidx + (size_t)c * (P.rounds + 1) * gstep_words + t;
        same &= (en[r] >> 16) == (en[0] >> 16);
      }
      if (__all_sync(0xffffffffu, same))
        tile_rows<LOG2N, L, STD, FWD, VPT, true>(v, cp, gp, gstep_words, wbase, rbase, P.rounds, P.gmask);
      else
        tile_rows<LOG2N, L, STD, FWD, VPT, false>(v, cp, gp, gstep_words, wbase, rbase, P.rounds, P.gmask);

#pragma unroll
      for (int r = 0; r < VPT; ++r) {
        const int p = p0 + r * V + g;
        const uint32_t c = en[r] >> 16;
        const size_t lr = en[r] & 0xffffu;
        float4* yr = reinterpret_cast<float4*>(yt + lr * N);
        if (p < rows && c < (uint32_t)C) {
#pragma unroll
          for (int u = 0; u < E / CH; ++u)
            __stcs(yr + t + TPV * u,
                   make_float4(v[r][2 * u].x, v[r][2 * u].y, v[r][2 * u + 1].x, v[r][2 * u + 1].y));
          if constexpr (ENERGY) {
            double* e = P.energy + (size_t)c * N;
#pragma unroll
            for (int k = 0; k < NP; ++k) {
              atomicAdd(e + LY.elem(t, 2 * k), (double)(v[r][k].x * v[r][k].x));
              atomicAdd(e + LY.elem(t, 2 * k + 1), (double)(v[r][k].y * v[r][k].y));
            }
          }
        } else if (p < rows) {  // invalid class id: pass the row through (error flagged)
          const float4* xr = reinterpret_cast<const float4*>(xt + lr * N);
#pragma unroll
          for (int u = 0; u < E / CH; ++u) yr[t + TPV * u] = xr[t + TPV * u];
        }
      }
    }
  }
}

}  // namespace hygt_gpu
