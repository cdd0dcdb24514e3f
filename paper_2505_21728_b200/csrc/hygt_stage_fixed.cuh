// hygt_stage_fixed.cuh -- the staged kernel (hygt_stage.cuh) for the bit-exact fixed-point
// transform at N = 16: forward_fixed / inverse_fixed (fixedpoint.hpp:154-224) over
// int64 rows, class-sorted per tile by the same sort pass.
//
// Per tile of T rows: the producer warp moves the int64 rows (128 B each) and the tile's sorted
// entry block into a ring of STAGES shared-memory stages with cp.async.bulk and streams the
// results back the same way; each consumer thread takes VPT sorted rows of one class.
//   * values are int32 in registers (|x| <= 2^20 is checked on input; the plan takes this kernel
//     only when fixed_int32_safe() in hygt_capi.cu bounds |value| < 2^30), products
//     and the rounding add in int64: y = (c x_e + s' x_partner + 2^(p-1)) >> p per element with
//     (c, s') = (c, s) on the pair's low element and (c, -s) on its high element
//     (fixedpoint.hpp:170-176), looked up from the TrigTable at plan creation;
//   * thread l relabels elements by X = (l & 7) << 1 (hypercube pairs stay register pairs), so
//     its 16 B row chunks spread over all 8 bank groups of the 128 B rows;
//   * a row that fails (|x| > 2^20) records min(row << 3 | 1) for the host, as the warp-per-row
//     kernel does; rows with an invalid class id were left out by the sort pass (flagged there).
#pragma once

#include "hygt_stage.cuh"

namespace hygt_gpu {

struct StageFxParams {
  const int64_t* x;
  int64_t* y;
  uint64_t count;
  int classes;
  int rounds;
  int precision_bits;
  const int4* tab;         // [C][R*log2N][N/2] int4 (c, s', c, s') of element pairs (2k, 2k+1)
  const uint16_t* gtab;    // [C][gstride] bytes: [R+1][N] u16 scratch offsets src * 128
  uint64_t gmask;
  uint32_t tile_rows;
  const uint16_t* ent;     // sorted entry blocks (stage sort pass), nullptr: identity order
  uint32_t block_words;
  unsigned long long* err;  // min over (row << 3 | status)
};

struct StageFxSmem {
  uint32_t tab, gtab, gstride, stage, stage_bytes, ent_off, scratch, bar, total;
};

HYGT_HD StageFxSmem stage_fx_smem_layout(int log2n, int vpt, int warps, int classes, int rounds,
                                         uint32_t tile_rows, bool gathers) {
  const uint32_t n = 1u << log2n;
  StageFxSmem s{};
  uint32_t o = 0;
  s.tab = o;
  o += stage_align((uint32_t)classes * rounds * log2n * n * 8u, 128);
  s.gtab = o;
  s.gstride = stage_gstride(log2n, rounds);
  o += gathers ? stage_align((uint32_t)classes * s.gstride, 128) : 0u;
  s.ent_off = tile_rows * n * 8u;
  s.stage_bytes = stage_align(s.ent_off + stage_block_words(tile_rows, vpt, classes) * 2u, 128);
  s.stage = o;
  o += STAGES * s.stage_bytes;
  s.scratch = o;
  o += gathers ? (uint32_t)warps * vpt * n * 128u : 0u;
  s.bar = stage_align(o, 16);
  s.total = s.bar + (2 * STAGES + 1) * 8;
  return s;
}

template <int LOG2N, int VPT, bool FWD, int WARPS>
__global__ void __launch_bounds__((WARPS + 1) * 32, 1) hygt_stage_fixed_kernel(const StageFxParams P) {
  using namespace stage_detail;
  constexpr int N = 1 << LOG2N, NC = N / 2;  // 16 B chunks (2 int64) per row
  constexpr int CT = WARPS * 32, BATCH = 32 * VPT;
  static_assert(NC == 8, "staged fixed-point kernel: N = 16");
  extern __shared__ __align__(128) unsigned char smem[];
  const int C = P.classes;
  const uint32_t T = P.tile_rows;
  const bool gathers = P.gmask != 0;
  const StageFxSmem L = stage_fx_smem_layout(LOG2N, VPT, WARPS, C, P.rounds, T, gathers);
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
  const uint32_t steps = (uint32_t)P.rounds * LOG2N;

  if (warp == WARPS) {  // ------------------------------------------------ producer warp
    if (lane != 0) return;
    auto load = [&](uint32_t k) {
      const uint32_t s = k % STAGES, rows = tile_rows(k);
      unsigned char* st = smem + L.stage + s * L.stage_bytes;
      const uint32_t eb = P.ent ? P.block_words * 2u : 0u;
      mbar_expect_tx(&full[s], rows * N * 8u + eb);
      if (eb) bulk_g2s(st + L.ent_off, P.ent + tile_id(k) * P.block_words, eb, &full[s]);
      bulk_g2s(st, P.x + tile_id(k) * T * N, rows * N * 8u, &full[s]);
    };
    auto store = [&](uint32_t k) {
      const uint32_t s = k % STAGES, rows = tile_rows(k);
      mbar_wait(&computed[s], (k / STAGES) & 1u);
      bulk_s2g(P.y + tile_id(k) * T * N, smem + L.stage + s * L.stage_bytes, rows * N * 8u);
      bulk_commit();
    };
    {
      const uint32_t tb = (uint32_t)C * steps * N * 8u, gb = gathers ? (uint32_t)C * L.gstride : 0u;
      mbar_expect_tx(tables, tb + gb);
      bulk_g2s(smem + L.tab, P.tab, tb, tables);
      if (gb) bulk_g2s(smem + L.gtab, P.gtab, gb, tables);
    }
    for (uint32_t k = 0; k < my_tiles; ++k) {
      if (k >= STAGES) {
        store(k - STAGES);
        bulk_wait_read0();
      }
      load(k);
    }
    for (uint32_t k = my_tiles >= STAGES ? my_tiles - STAGES : 0; k < my_tiles; ++k) store(k);
    bulk_wait0();
    return;
  }

  // ------------------------------------------------------------------- consumer warps
  const uint32_t x = lane & 7;       // chunk rotation: register chunk c holds element chunk c ^ x
  const uint32_t xs = x << 8;        // (x << 1) << 7: element-label XOR in scratch bytes
  const uint32_t tab_s = su32(smem + L.tab);
  const uint32_t gtab_s = su32(smem + L.gtab);
  const uint32_t scr = su32(smem + L.scratch) + (uint32_t)warp * VPT * N * 128u + lane * 4u;
  const int prec = P.precision_bits;
  const int64_t rnd = (int64_t)1 << (prec - 1);
  mbar_wait(tables, 0);
  for (uint32_t k = 0; k < my_tiles; ++k) {
    const uint32_t s = k % STAGES;
    const unsigned char* st = smem + L.stage + s * L.stage_bytes;
    mbar_wait(&full[s], (k / STAGES) & 1u);
    const uint32_t rows = tile_rows(k);
    const uint32_t total = P.ent ? *reinterpret_cast<const uint32_t*>(st + L.ent_off) : rows;
    const uint16_t* ent = reinterpret_cast<const uint16_t*>(st + L.ent_off) + 8;
    const uint32_t rows_s = su32(st);
    for (uint32_t b = warp; b * BATCH < total; b += WARPS) {
      uint32_t en[VPT];
      const uint32_t p0 = b * BATCH + lane * VPT;
#pragma unroll
      for (int r = 0; r < VPT; ++r)
        en[r] = P.ent ? (uint32_t)ent[p0 + r] : (p0 + r < rows ? p0 + r : STAGE_PAD);
      const uint32_t cls = en[0] == STAGE_PAD ? 0u : en[0] >> 10;
      int32_t v[VPT][N];
      bool bad[VPT];
#pragma unroll
      for (int r = 0; r < VPT; ++r) {
        bad[r] = false;
        const uint32_t ra = rows_s + (en[r] & 1023u) * (N * 8u);
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          uint4 q = make_uint4(0, 0, 0, 0);
          if (en[r] != STAGE_PAD)
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w)
                         : "r"(ra + ((c ^ x) << 4)));
          const int64_t a = (int64_t)(((uint64_t)q.y << 32) | q.x), bb = (int64_t)(((uint64_t)q.w << 32) | q.z);
          bad[r] |= a > (1 << 20) || a < -(1 << 20) || bb > (1 << 20) || bb < -(1 << 20);  // fixedpoint.hpp:145-150
          v[r][2 * c] = (int32_t)a;
          v[r][2 * c + 1] = (int32_t)bb;
        }
      }
      const uint32_t cbase = tab_s + cls * steps * (N * 8u);
      auto gather = [&](uint32_t gt) {  // permutation through the conflict-free scratch
        __syncwarp();
#pragma unroll
        for (int r = 0; r < VPT; ++r)
#pragma unroll
          for (int i = 0; i < N; ++i) sts32(scr + (uint32_t)((r * N + i) * 128), __int_as_float(v[r][i]));
        __syncwarp();
#pragma unroll
        for (int c = 0; c < N / 4; ++c) {
          // registers 4c + h hold elements (4c + h) ^ X = 4 (c ^ (x >> 1)) + (h ^ 2 (x & 1))
          uint2 g;
          asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(g.x), "=r"(g.y)
                       : "r"(gt + ((uint32_t)(c ^ (x >> 1)) << 3)));
          const bool sw = x & 1u;
          const uint32_t lo = sw ? g.y : g.x, hi = sw ? g.x : g.y;
          const uint32_t o[4] = {lo & 0xffffu, lo >> 16, hi & 0xffffu, hi >> 16};
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const uint32_t a = scr + (o[h] ^ xs);
#pragma unroll
            for (int r = 0; r < VPT; ++r) v[r][4 * c + h] = __float_as_int(lds32(a + r * N * 128));
          }
        }
      };
      const uint32_t gbase = gtab_s + cls * L.gstride;
      if (P.gmask & 1ull) gather(gbase);
      for (int rr = 0; rr < P.rounds; ++rr) {
#pragma unroll
        for (int pp = 0; pp < LOG2N; ++pp) {
          const int d = FWD ? pp : LOG2N - 1 - pp;
          const uint32_t sb = cbase + (uint32_t)(rr * LOG2N + pp) * (N * 8u);
          int32_t o[VPT][N];
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            uint4 q;  // (c, s') of register elements 2c, 2c+1 = table elements 2(c ^ x), +1
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w)
                         : "r"(sb + ((c ^ x) << 4)));
#pragma unroll
            for (int r = 0; r < VPT; ++r) {
              const int i0 = 2 * c, i1 = 2 * c + 1;
              o[r][i0] = (int32_t)(((int64_t)(int32_t)q.x * v[r][i0] + (int64_t)(int32_t)q.y * v[r][i0 ^ (1 << d)] + rnd) >> prec);
              o[r][i1] = (int32_t)(((int64_t)(int32_t)q.z * v[r][i1] + (int64_t)(int32_t)q.w * v[r][i1 ^ (1 << d)] + rnd) >> prec);
            }
          }
#pragma unroll
          for (int r = 0; r < VPT; ++r)
#pragma unroll
            for (int i = 0; i < N; ++i) v[r][i] = o[r][i];
        }
        if ((P.gmask >> (rr + 1)) & 1ull) gather(gbase + (uint32_t)(rr + 1) * N * 2u);
      }
#pragma unroll
      for (int r = 0; r < VPT; ++r) {
        if (en[r] == STAGE_PAD) continue;
        const uint32_t row = en[r] & 1023u;
        const uint32_t ra = rows_s + row * (N * 8u);
        if (bad[r]) {
          atomicMin(P.err, (unsigned long long)(((tile_id(k) * T + row) << 3) | 1ull));
          continue;  // the slot keeps x; the call fails at this row
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const int64_t a = v[r][2 * c], bb = v[r][2 * c + 1];
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(ra + ((c ^ x) << 4)),
                       "r"((uint32_t)a), "r"((uint32_t)((uint64_t)a >> 32)), "r"((uint32_t)bb),
                       "r"((uint32_t)((uint64_t)bb >> 32))
                       : "memory");
        }
      }
    }
    fence_async_smem();
    mbar_arrive(&computed[s]);
  }
}

}  // namespace hygt_gpu
