// hygt_stage.cuh -- the TMA-staged HyGT kernel for short rows (N = 16): production path of
// BASELINE config 2 (C = 35 classes, random class per row).
//
// Why it exists: the tile kernel (hygt_tile.cuh) gathers class-sorted rows straight from HBM;
// every row then costs 4 L1 wavefronts of scattered 32 B global accesses plus the shuffles of a
// two-lanes-per-row layout, and the L1/LSU data pipe (not HBM) bounds it (profiles/r01). Here
// the rows never touch the LSU on their way in or out. Two kernels:
//
//   hygt_stage_sort_kernel (once per batch of class ids, reused by forward and inverse): for
//     every tile of T rows, a counting sort of the rows by class -- the batched equivalent of
//     run_apply's cache[b.class_id] dispatch (hygt_main.cpp:143-149) -- with every class run
//     padded to VPT and the tail padded to a whole batch of 32*VPT positions; writes one block
//     [total, entries] per tile (entry = class << 10 | row, pad 0xffff) to the workspace.
//
//   hygt_stage_kernel (persistent, one CTA per SM, ring of STAGES tiles in shared memory):
//     producer warp (lane 0)                 consumer warps (WARPS)
//     -----------------------------------    --------------------------------------------------
//     TMA x[tile] + entry block -> stage s    wait full[s]; thread = VPT sorted rows of one
//       (cp.async.bulk, complete_tx full[s])  class: all rounds in registers, coefficients from
//     wait computed[s]                        shared memory (one LDS.128 feeds VPT rows),
//     TMA stage s -> y[tile]                  permutations through a conflict-free per-warp
//     wait_group.read, next load              scratch, rows written back into their slots;
//                                             fence.proxy.async, arrive computed[s]
//
// Bank spreading: a 64 B row occupies half a 128 B bank line, so 32 threads reading chunk c of
// 32 random rows would hit only 2 of the 8 16-byte bank groups. Thread l therefore keeps its
// rows with the element labels XOR-ed by X = (l & 3) << 2 (register i holds element i ^ X).
// Hypercube pairs (i, i ^ 2^p) stay register pairs under that relabelling, so the arithmetic is
// unchanged; only the addresses of the coefficient units, gather offsets and row chunks are
// rotated per thread -- and the row chunks then spread over all 8 bank groups. The order of a
// thread's VPT rows is free as well; rows alternate between the two halves of a bank line.
//
// Reference semantics are those of run_passes / forward / inverse (transform.hpp:45-96); tables
// come from build_programs() (hygt_plan.cpp), the same per-butterfly fp64 (c, s) as every other
// path.
#pragma once

#include <cstdint>

#include "hygt_kernels.cuh"

namespace hygt_gpu {

constexpr int STAGES = 3;          // ring of TMA-staged tiles
constexpr int STAGE_SCR_ROWS = 2;  // rows per thread permuted per scratch round trip
constexpr uint32_t STAGE_PAD = 0xffffu;
constexpr int STAGE_MAX_CLASSES = 63;  // entry = class << 10 | row, pad = 0xffff

struct StageParams {
  const float* x;
  float* y;
  uint64_t count;
  int classes;
  int rounds;
  const float4* coef;      // [C][cw] float4, element-ordered units per step (see setup_stage)
  uint32_t cw;             // float4 units per class
  const uint16_t* gtab;    // [C][gstride] bytes: [R+1][N] u16 scratch offsets src * 128
  uint64_t gmask;
  uint32_t tile_rows;      // T (multiple of 8, <= 1016)
  const uint16_t* ent;     // [tiles][block_words] sorted entry blocks, nullptr: identity order
  uint32_t block_words;    // u16 per entry block: 8 (header: total) + positions
  const uint16_t* cls;     // identity order with class ids given (one class): validated here
  uint32_t* err;           // invalid class id flag (identity order)
  unsigned long long* trace;  // debug: per-tile clock64 events of CTA 0 (nullptr = off)
  uint32_t debug_skip;        // debug: consumers skip the arithmetic (timing of the other roles)
};

struct StageSortParams {
  const uint16_t* cls;
  uint64_t count;
  int classes;
  uint32_t tile_rows;
  uint32_t block_words;
  uint16_t* ent;
  uint32_t* err;
};

HYGT_HD constexpr uint32_t stage_align(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }

// u16 words of one tile's entry block: 8-word header (u32 total) + positions padded to batches.
HYGT_HD constexpr uint32_t stage_block_words(uint32_t tile_rows, int vpt, int classes) {
  return 8u + stage_align(tile_rows + (uint32_t)(vpt - 1) * classes + 32u * vpt, 32u * vpt);
}

// Byte stride of one class's gather table [R+1][N] u16, padded so that consecutive classes start
// 32 B apart in the bank space (threads of several classes read their tables in one wavefront).
HYGT_HD constexpr uint32_t stage_gstride(int log2n, int rounds) {
  return ((uint32_t)(rounds + 1) * (2u << log2n) + 31u) / 32u * 32u +
         ((((uint32_t)(rounds + 1) * (2u << log2n) + 31u) / 32u * 32u) % 128u == 0 ? 32u : 0u);
}

// Shared-memory carve-up of hygt_stage_kernel, identical on host and device.
struct StageSmem {
  uint32_t coef, gtab, gstride, stage, stage_bytes, ent_off, scratch, bar, total;
};

HYGT_HD StageSmem stage_smem_layout(int log2n, int vpt, int warps, int classes, uint32_t cw,
                                    int rounds, uint32_t tile_rows, bool gathers) {
  const uint32_t n = 1u << log2n;
  StageSmem s{};
  uint32_t o = 0;
  s.coef = o;
  o += stage_align((uint32_t)classes * cw * 16u, 128);
  s.gtab = o;
  s.gstride = stage_gstride(log2n, rounds);
  o += gathers ? stage_align((uint32_t)classes * s.gstride, 128) : 0u;
  s.ent_off = tile_rows * n * 4u;
  s.stage_bytes = stage_align(s.ent_off + stage_block_words(tile_rows, vpt, classes) * 2u, 128);
  s.stage = o;
  o += STAGES * s.stage_bytes;
  s.scratch = o;
  o += gathers ? (uint32_t)warps * (vpt < STAGE_SCR_ROWS ? vpt : STAGE_SCR_ROWS) * n * 128u : 0u;
  s.bar = stage_align(o, 16);
  s.total = s.bar + (2 * STAGES + 1) * 8;
  return s;
}

namespace stage_detail {

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
#define STAGE_TRACE(k, e)                                                           \
  do {                                                                              \
    if (DEBUG && P.trace && blockIdx.x == 0 && (k) < 64) P.trace[(k) * 16 + (e)] = clock64(); \
  } while (0)

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "STAGE_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra STAGE_WAIT_%=;\n\t}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(su32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
template <int NT>
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ float lds32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts32(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}

}  // namespace stage_detail

template <int NW, int P, bool STD, int VPT>
__device__ __forceinline__ void stage_pass(float2 (&v)[VPT][NW], const uint32_t (&cu)[NW / 2],
                                           uint32_t step_off) {
  constexpr int NC = NW / 2;
  float2 k[NW], s[NW];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const float4 q = stage_detail::lds128(cu[c] + step_off);
    k[2 * c] = make_float2(q.x, q.y);
    k[2 * c + 1] = make_float2(q.z, q.w);
    if constexpr (STD) {
      const float4 t = stage_detail::lds128(cu[c] + step_off + NC * 16);
      s[2 * c] = make_float2(t.x, t.y);
      s[2 * c + 1] = make_float2(t.z, t.w);
    }
  }
#pragma unroll
  for (int r = 0; r < VPT; ++r) {
    if constexpr (P == 0) {
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        if constexpr (!STD) v[r][w] = ffma2(k[w], swap2(v[r][w]), v[r][w]);
        else v[r][w] = ffma2(k[w], v[r][w], fmul2(s[w], swap2(v[r][w])));
      }
    } else {
      constexpr int M = 1 << (P - 1);
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        if (w & M) continue;
        const float2 a = v[r][w], b = v[r][w + M];
        if constexpr (!STD) {
          v[r][w] = ffma2(k[w], b, a);
          v[r][w + M] = ffma2(k[w + M], a, b);
        } else {
          v[r][w] = ffma2(k[w], a, fmul2(s[w], b));
          v[r][w + M] = ffma2(k[w + M], b, fmul2(s[w + M], a));
        }
      }
    }
  }
}

template <int LOG2N, bool STD, bool FWD, int VPT, int PP>
__device__ __forceinline__ void stage_round(float2 (&v)[VPT][(1 << LOG2N) / 2],
                                            const uint32_t (&cu)[(1 << LOG2N) / 4],
                                            uint32_t round_off) {
  if constexpr (PP < LOG2N) {
    constexpr int P = FWD ? PP : LOG2N - 1 - PP;
    constexpr uint32_t STEP = (1u << LOG2N) / 4 * 16 * (STD ? 2 : 1);
    stage_pass<(1 << LOG2N) / 2, P, STD, VPT>(v, cu, round_off + PP * STEP);
    stage_round<LOG2N, STD, FWD, VPT, PP + 1>(v, cu, round_off);
  }
}

// Permutation of VPT rows through the warp's scratch [SR][N][32] floats, SR rows at a time (thread
// l at word l: every access is bank-conflict-free). gt = shared address of this step's [N] u16
// gather table (element order, byte offsets src * 128); register i receives element i ^ X, which
// is old element src[i ^ X], stored in old register src[i ^ X] ^ X.
template <int LOG2N, int VPT, int SR>
__device__ __forceinline__ void stage_gather(float2 (&v)[VPT][(1 << LOG2N) / 2], uint32_t scr,
                                             uint32_t gt, uint32_t x, uint32_t xs) {
  constexpr int N = 1 << LOG2N, NW = N / 2, NC = N / 4;
  if constexpr (SR >= VPT) {  // all rows in one round trip; offsets read per chunk
    __syncwarp();
#pragma unroll
    for (int r = 0; r < VPT; ++r)
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        stage_detail::sts32(scr + (uint32_t)((r * N + 2 * w) * 128), v[r][w].x);
        stage_detail::sts32(scr + (uint32_t)((r * N + 2 * w + 1) * 128), v[r][w].y);
      }
    __syncwarp();
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      uint2 g;
      asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(g.x), "=r"(g.y) : "r"(gt + ((c ^ x) << 3)));
      const uint32_t a0 = scr + ((g.x & 0xffffu) ^ xs), a1 = scr + ((g.x >> 16) ^ xs);
      const uint32_t a2 = scr + ((g.y & 0xffffu) ^ xs), a3 = scr + ((g.y >> 16) ^ xs);
#pragma unroll
      for (int r = 0; r < VPT; ++r) {
        v[r][2 * c].x = stage_detail::lds32(a0 + r * N * 128);
        v[r][2 * c].y = stage_detail::lds32(a1 + r * N * 128);
        v[r][2 * c + 1].x = stage_detail::lds32(a2 + r * N * 128);
        v[r][2 * c + 1].y = stage_detail::lds32(a3 + r * N * 128);
      }
    }
    return;
  }
  uint32_t a[N];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    uint2 g;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(g.x), "=r"(g.y) : "r"(gt + ((c ^ x) << 3)));
    a[4 * c] = scr + ((g.x & 0xffffu) ^ xs);
    a[4 * c + 1] = scr + ((g.x >> 16) ^ xs);
    a[4 * c + 2] = scr + ((g.y & 0xffffu) ^ xs);
    a[4 * c + 3] = scr + ((g.y >> 16) ^ xs);
  }
#pragma unroll
  for (int r0 = 0; r0 < VPT; r0 += SR) {
    __syncwarp();
#pragma unroll
    for (int r = 0; r < SR; ++r)
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        stage_detail::sts32(scr + (uint32_t)((r * N + 2 * w) * 128), v[r0 + r][w].x);
        stage_detail::sts32(scr + (uint32_t)((r * N + 2 * w + 1) * 128), v[r0 + r][w].y);
      }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < SR; ++r)
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        v[r0 + r][w].x = stage_detail::lds32(a[2 * w] + r * N * 128);
        v[r0 + r][w].y = stage_detail::lds32(a[2 * w + 1] + r * N * 128);
      }
  }
}

// ------------------------------------------------------------------------- per-tile sort ----
// One warp per tile (many tiles in flight per SM: this pass is latency-, not bandwidth-bound).
// Ranks come from shared atomics on (class, row parity) counters; inside a class, even and odd
// rows alternate (the shorter parity runs out first) so that each thread of the staged kernel
// gets rows from both halves of a 128 B bank line. Class starts: warp scan of the padded counts.
constexpr int STAGE_SORT_WARPS = 8;

HYGT_HD constexpr uint32_t stage_sort_warp_bytes(int classes, uint32_t block_words) {
  return stage_align((uint32_t)(3 * classes + 1) * 4u, 16) + stage_align((block_words - 8) * 2u, 16);
}

template <int VPT, int H>  // H groups of 4 consecutive ids per lane: T <= 128 H
__global__ void __launch_bounds__(32 * STAGE_SORT_WARPS) hygt_stage_sort_kernel(const StageSortParams P) {
  constexpr int BATCH = 32 * VPT;
  extern __shared__ __align__(16) unsigned char sm[];
  const int C = P.classes;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* mine = sm + warp * stage_sort_warp_bytes(C, P.block_words);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(mine);  // [C][2] counts per (class, row parity)
  uint32_t* start = cnt + 2 * C;                       // [C] padded class starts
  uint16_t* ents = reinterpret_cast<uint16_t*>(mine + stage_align((uint32_t)(3 * C + 1) * 4u, 16));
  const uint32_t T = P.tile_rows;
  const uint64_t tiles = (P.count + T - 1) / T;
  bool bad = false;
  for (uint64_t tile = (uint64_t)blockIdx.x * STAGE_SORT_WARPS + warp; tile < tiles;
       tile += (uint64_t)gridDim.x * STAGE_SORT_WARPS) {
    const uint64_t row0 = tile * T;
    const uint32_t rows = (uint32_t)((P.count - row0) < T ? (P.count - row0) : T);
    for (int c = lane; c < 2 * C; c += 32) cnt[c] = 0;
    uint2 w[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const uint32_t j0 = 128u * h + 4u * lane;
      w[h] = make_uint2(0xffffffffu, 0xffffffffu);
      if (j0 + 4 <= rows && ((reinterpret_cast<uintptr_t>(P.cls + row0 + j0) & 7) == 0)) {
        w[h] = __ldcs(reinterpret_cast<const uint2*>(P.cls + row0 + j0));
      } else if (j0 < rows) {
        uint32_t q[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) q[e] = j0 + e < rows ? (uint32_t)P.cls[row0 + j0 + e] : 0xffffu;
        w[h] = make_uint2(q[0] | (q[1] << 16), q[2] | (q[3] << 16));
      }
    }
    __syncwarp();
    uint32_t pk[4 * H];  // (class << 16) | rank within (class, parity), or 0xffffffff
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t j = 128u * h + 4u * lane + e;
        const uint32_t c = ((e < 2 ? w[h].x : w[h].y) >> (16 * (e & 1))) & 0xffffu;
        const bool in = j < rows, ok = in && c < (uint32_t)C;
        bad |= in && !ok;  // passed through: no entry, the stage slot keeps x
        pk[4 * h + e] = ok ? ((c << 16) | atomicAdd(&cnt[2 * c + (j & 1u)], 1u)) : 0xffffffffu;
      }
    __syncwarp();
    uint32_t carry = 0;
    for (int base = 0; base < C; base += 32) {
      const int c = base + lane;
      const uint32_t n = c < C ? cnt[2 * c] + cnt[2 * c + 1] : 0u;
      const uint32_t padded = (n + VPT - 1) / VPT * VPT;
      uint32_t incl = padded;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (c < C) {
        const uint32_t st = carry + incl - padded;
        start[c] = st | (min(cnt[2 * c], cnt[2 * c + 1]) << 16);  // start, interleaved pairs
        for (uint32_t q = st + n; q < st + padded; ++q) ents[q] = (uint16_t)STAGE_PAD;
      }
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    const uint32_t end = (carry + BATCH - 1) / BATCH * BATCH;
    for (uint32_t q = carry + lane; q < end; q += 32) ents[q] = (uint16_t)STAGE_PAD;
    __syncwarp();
#pragma unroll
    for (int g = 0; g < 4 * H; ++g)
      if (pk[g] != 0xffffffffu) {
        const uint32_t c = pk[g] >> 16, r = pk[g] & 0xffffu;
        const uint32_t j = 128u * (g >> 2) + 4u * lane + (g & 3);
        const uint32_t sm_ = start[c], m = sm_ >> 16;
        ents[(sm_ & 0xffffu) + (r < m ? 2 * r + (j & 1u) : m + r)] = (uint16_t)((c << 10) | j);
      }
    __syncwarp();
    uint16_t* dst = P.ent + tile * P.block_words;
    for (uint32_t i = lane; i < (8u + end) / 8; i += 32) {
      const uint4 v = i == 0 ? make_uint4(carry, 0u, 0u, 0u) : reinterpret_cast<const uint4*>(ents)[i - 1];
      __stcs(reinterpret_cast<uint4*>(dst) + i, v);
    }
    __syncwarp();
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(P.err, 1u);
}

// Build variants (VAR bits): STAGE_VAR_DEBUG honours P.trace / P.debug_skip. The default build
// does not compile it: its never-taken branches alone cost ~1-3% of the kernel's time.
constexpr int STAGE_VAR_DEBUG = 2;
template <int LOG2N, int VPT, bool STD, bool FWD, int WARPS, int VAR = 0>
__global__ void __launch_bounds__((WARPS + 1) * 32, 1) hygt_stage_kernel(const StageParams P) {
  constexpr bool DEBUG = (VAR & STAGE_VAR_DEBUG) != 0;
  using namespace stage_detail;
  constexpr int N = 1 << LOG2N, NW = N / 2, NC = N / 4;
  constexpr int CT = WARPS * 32;  // consumer threads
  constexpr int BATCH = 32 * VPT;
  constexpr int SCR_ROWS = STAGE_SCR_ROWS < VPT ? STAGE_SCR_ROWS : VPT;
  static_assert(NC >= 2 && NC <= 4, "stage kernel: N in {8, 16}");
  static_assert(VPT == 4, "stage kernel: entries are read as one 8-byte word per thread");
  extern __shared__ __align__(128) unsigned char smem[];
  const int C = P.classes;
  const uint32_t T = P.tile_rows;
  const bool gathers = P.gmask != 0;
  const StageSmem L = stage_smem_layout(LOG2N, VPT, WARPS, C, P.cw, P.rounds, T, gathers);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar);
  uint64_t* computed = full + STAGES;
  uint64_t* tables = full + 2 * STAGES;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&computed[i], CT);
    }
    mbar_init(tables, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t tiles = (P.count + T - 1) / T;
  const uint32_t my_tiles =
      blockIdx.x < tiles ? (uint32_t)((tiles - 1 - blockIdx.x) / gridDim.x + 1) : 0u;
  auto tile_id = [&](uint32_t k) -> uint64_t { return (uint64_t)blockIdx.x + (uint64_t)k * gridDim.x; };
  auto tile_rows = [&](uint32_t k) -> uint32_t {
    const uint64_t left = P.count - tile_id(k) * T;
    return left < T ? (uint32_t)left : T;
  };

  // one class with ids given: the tile's ids ride along in the entry region when aligned
  auto ids_tma = [&](uint32_t rows) -> bool {
    return P.cls && !P.ent && (rows % 8u) == 0 && ((reinterpret_cast<uintptr_t>(P.cls) & 15) == 0);
  };

  if (warp == WARPS) {  // ------------------------------------------------ producer warp
    if (lane != 0) return;
    auto load = [&](uint32_t k) {
      const uint32_t s = k % STAGES, rows = tile_rows(k);
      unsigned char* st = smem + L.stage + s * L.stage_bytes;
      const uint32_t eb = P.ent ? P.block_words * 2u : ids_tma(rows) ? rows * 2u : 0u;
      mbar_expect_tx(&full[s], rows * N * 4u + eb);
      if (P.ent) bulk_g2s(st + L.ent_off, P.ent + tile_id(k) * P.block_words, eb, &full[s]);
      else if (eb) bulk_g2s(st + L.ent_off, P.cls + tile_id(k) * T, eb, &full[s]);  // one class: ids
      bulk_g2s(st, P.x + tile_id(k) * T * N, rows * N * 4u, &full[s]);
    };
    auto store = [&](uint32_t k) {
      const uint32_t s = k % STAGES, rows = tile_rows(k);
      mbar_wait(&computed[s], (k / STAGES) & 1u);
      STAGE_TRACE(k, 5);
      bulk_s2g(P.y + tile_id(k) * T * N, smem + L.stage + s * L.stage_bytes, rows * N * 4u);
      bulk_commit();
    };
    {  // the direction's tables, once per CTA
      const uint32_t cb = (uint32_t)C * P.cw * 16u;
      const uint32_t gb = gathers ? (uint32_t)C * L.gstride : 0u;
      mbar_expect_tx(tables, cb + gb);
      bulk_g2s(smem + L.coef, P.coef, cb, tables);
      if (gb) bulk_g2s(smem + L.gtab, P.gtab, gb, tables);
    }
    for (uint32_t k = 0; k < my_tiles; ++k) {
      if (k >= STAGES) {
        store(k - STAGES);
        bulk_wait_read0();  // stage (k % STAGES) is free again
        STAGE_TRACE(k - STAGES, 6);
      }
      load(k);
      STAGE_TRACE(k, 0);
    }
    for (uint32_t k = my_tiles >= STAGES ? my_tiles - STAGES : 0; k < my_tiles; ++k) store(k);
    bulk_wait0();
    return;
  }

  // ------------------------------------------------------------------- consumer warps
  const uint32_t x = lane & (NC - 1);         // chunk rotation of this thread
  const uint32_t xs = x << 9;                 // (x << 2) << 7: register-label XOR in scratch bytes
  const uint32_t tpar = (lane >> 2) & 1;      // preferred row parity of row slot 0
  const uint32_t coef_s = su32(smem + L.coef);
  const uint32_t gtab_s = su32(smem + L.gtab);
  const uint32_t scr = su32(smem + L.scratch) + (uint32_t)warp * SCR_ROWS * N * 128u + lane * 4u;
  mbar_wait(tables, 0);
  for (uint32_t k = 0; k < my_tiles; ++k) {
    const uint32_t s = k % STAGES;
    const unsigned char* st = smem + L.stage + s * L.stage_bytes;
    mbar_wait(&full[s], (k / STAGES) & 1u);
    if (tid == 0) STAGE_TRACE(k, 3);
    const uint32_t rows = tile_rows(k);
    const uint32_t total = P.ent ? *reinterpret_cast<const uint32_t*>(st + L.ent_off) : rows;
    const uint16_t* ent = reinterpret_cast<const uint16_t*>(st + L.ent_off) + 8;
    const uint32_t rows_s = su32(st);

    // ---- transform: VPT consecutive sorted positions per thread ----
    for (uint32_t b = warp; b * BATCH < total && !(DEBUG && P.debug_skip); b += WARPS) {
      uint32_t en[VPT];
      const uint32_t p0 = b * BATCH + lane * VPT;
      if (P.ent) {
        uint2 e2;
        asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(e2.x), "=r"(e2.y) : "r"(su32(ent + p0)));
        en[0] = e2.x & 0xffffu;
        en[1] = e2.x >> 16;
        en[2] = e2.y & 0xffffu;
        en[3] = e2.y >> 16;
      } else {
#pragma unroll
        for (int r = 0; r < VPT; ++r) en[r] = p0 + r < rows ? p0 + r : STAGE_PAD;
        if (P.cls) {  // one class: rows with an id >= 1 pass through unchanged, flagged
          const uint16_t* ids = ids_tma(rows) ? reinterpret_cast<const uint16_t*>(st + L.ent_off) + p0
                                              : P.cls + tile_id(k) * T + p0;
          bool bad = false;
#pragma unroll
          for (int r = 0; r < VPT; ++r)
            if (en[r] != STAGE_PAD && ids[r] != 0) {
              en[r] = STAGE_PAD;
              bad = true;
            }
          if (bad) atomicOr(P.err, 1u);
        }
      }
      const uint32_t cls = en[0] == STAGE_PAD ? 0u : en[0] >> 10;
      // Row order inside the thread is free (the VPT rows share every coefficient): put rows of
      // parity tpar ^ (r & 1) in slot r where possible, so that the 8 threads sharing a chunk
      // rotation read rows from both halves of the 128 B bank lines (row = 64 B).
#pragma unroll
      for (int r = 0; r < VPT - 1; ++r) {
        const uint32_t want = tpar ^ (uint32_t)(r & 1);
        bool done = (en[r] & 1u) == want;
#pragma unroll
        for (int q = r + 1; q < VPT; ++q) {
          const bool take = !done && en[q] != STAGE_PAD && (en[q] & 1u) == want;
          const uint32_t a = en[r], bq = en[q];
          en[r] = take ? bq : a;
          en[q] = take ? a : bq;
          done |= take;
        }
      }
      uint32_t cu[NC];
      const uint32_t cbase = coef_s + cls * P.cw * 16u;
#pragma unroll
      for (int c = 0; c < NC; ++c) cu[c] = cbase + ((c ^ x) << 4);
      float2 v[VPT][NW];
#pragma unroll
      for (int r = 0; r < VPT; ++r) {
        const uint32_t ra = rows_s + (en[r] & 1023u) * (N * 4u);
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
          if (en[r] != STAGE_PAD) q = lds128(ra + ((c ^ x) << 4));
          v[r][2 * c] = make_float2(q.x, q.y);
          v[r][2 * c + 1] = make_float2(q.z, q.w);
        }
      }
      const uint32_t gbase = gtab_s + cls * L.gstride;
      auto permute = [&](int step) {
        stage_gather<LOG2N, VPT, SCR_ROWS>(v, scr, gbase + (uint32_t)step * N * 2u, x, xs);
      };
      if (P.gmask & 1ull) permute(0);
      constexpr uint32_t ROUND = (uint32_t)LOG2N * NC * 16u * (STD ? 2u : 1u);
      for (int rr = 0; rr < P.rounds; ++rr) {
        stage_round<LOG2N, STD, FWD, VPT, 0>(v, cu, (uint32_t)rr * ROUND);
        if ((P.gmask >> (rr + 1)) & 1ull) permute(rr + 1);
      }
      if constexpr (!STD) {  // remaining per-sample scales of the scale-folded form
        const uint32_t so = (uint32_t)P.rounds * ROUND;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const float4 q = lds128(cu[c] + so);
#pragma unroll
          for (int r = 0; r < VPT; ++r) {
            v[r][2 * c] = fmul2(v[r][2 * c], make_float2(q.x, q.y));
            v[r][2 * c + 1] = fmul2(v[r][2 * c + 1], make_float2(q.z, q.w));
          }
        }
      }
#pragma unroll
      for (int r = 0; r < VPT; ++r) {
        if (en[r] == STAGE_PAD) continue;
        const uint32_t ra = rows_s + (en[r] & 1023u) * (N * 4u);
#pragma unroll
        for (int c = 0; c < NC; ++c)
          sts128(ra + ((c ^ x) << 4),
                 make_float4(v[r][2 * c].x, v[r][2 * c].y, v[r][2 * c + 1].x, v[r][2 * c + 1].y));
      }
    }
    if (tid == 0) STAGE_TRACE(k, 4);
    fence_async_smem();
    mbar_arrive(&computed[s]);
  }
}

}  // namespace hygt_gpu
