// layout.h -- register layout shared by the host plan builder and the sm_100a kernels.
//
// A vector of N = 2^LOG2N fp32 samples is owned by a group of TPV = 2^L consecutive lanes.
// Each lane holds E = N / TPV samples in E registers ("slots"). HBM rows are read in 16-byte
// chunks of CH = min(4, N) samples; lane t of the group owns chunks q = t + TPV * u, so one
// warp-wide 128-bit load covers contiguous bytes of each row (coalesced when TPV >= 4, direct
// per-lane 64 B rows when TPV = 1).
//
//   element index i = (t + (u << L)) * CH + e,   slot s = u * CH + e
//
// so bits [0, log2 CH) of i are slot bits, bits [log2 CH, log2 CH + L) are lane bits and the
// remaining high bits are slot bits again. A hypercube pass p (hypercube.hpp:59-77: pairs
// differing in bit p) is therefore either in-register (slot offset slot_stride(p)) or a
// cross-lane exchange with lane t ^ (1 << (p - log2 CH)).
#pragma once

#ifdef __CUDACC__
#define HYGT_HD __host__ __device__ __forceinline__
#else
#define HYGT_HD inline
#endif

namespace hygt_gpu {

HYGT_HD constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v >> 1); }

struct Layout {
  int log2n;  // log2 N
  int l;      // log2 TPV
  HYGT_HD constexpr int n() const { return 1 << log2n; }
  HYGT_HD constexpr int tpv() const { return 1 << l; }
  HYGT_HD constexpr int ch() const { return log2n >= 2 ? 4 : (1 << log2n); }
  HYGT_HD constexpr int chl() const { return log2n >= 2 ? 2 : log2n; }
  HYGT_HD constexpr int e() const { return n() >> l; }
  HYGT_HD constexpr int elem(int t, int s) const {
    return ((t + ((s >> chl()) << l)) << chl()) + (s & (ch() - 1));
  }
  HYGT_HD constexpr bool cross(int p) const { return p >= chl() && p < chl() + l; }
  // Slot distance of the pair partner for an in-register pass p.
  HYGT_HD constexpr int slot_stride(int p) const {
    return p < chl() ? (1 << p) : (ch() << (p - chl() - l));
  }
  // Lane xor mask for a cross-lane pass p.
  HYGT_HD constexpr int lane_mask(int p) const { return 1 << (p - chl()); }
  // float2 coefficient words one lane consumes per pass: E/2 for every pass of the
  // scale-folded form and for in-register passes of the standard form; E for a cross-lane pass
  // of the standard form (c and +-s per own sample).
  HYGT_HD constexpr int words_per_pass(bool standard, int p) const {
    return (standard && cross(p)) ? e() : e() / 2;
  }
};

// Butterfly index j of the pair (m, m + 2^p) in reference order (hypercube.hpp:73-74 inverted:
// j is m with bit p removed).
HYGT_HD constexpr int pair_index(int m, int p) { return ((m >> (p + 1)) << p) | (m & ((1 << p) - 1)); }

}  // namespace hygt_gpu
