// hygt_dispatch_tile.cu -- instantiations of the tile kernel.
#include "hygt_dispatch.h"

namespace hygt_gpu {
namespace {


template <int LOG2N, int L, int VPT, int TT = TILE_THREADS>
TileFn pick_tile(bool standard, bool fwd, bool energy) {
  if (standard) {
    if (!fwd) return hygt_tile_kernel<LOG2N, L, VPT, true, false, false, TT>;
    return energy ? hygt_tile_kernel<LOG2N, L, VPT, true, true, true, TT>
                  : hygt_tile_kernel<LOG2N, L, VPT, true, true, false, TT>;
  }
  if (!fwd) return hygt_tile_kernel<LOG2N, L, VPT, false, false, false, TT>;
  return energy ? hygt_tile_kernel<LOG2N, L, VPT, false, true, true, TT>
                : hygt_tile_kernel<LOG2N, L, VPT, false, true, false, TT>;
}

}  // namespace

// Instantiated (log2 N, log2 TPV, rows per lane group) tile layouts; the first of each N is the
// default. All have E = N / TPV >= 4.
TileFn select_tile(int log2n, int l, int vpt, bool standard, bool fwd, bool energy) {
  switch (log2n * 256 + l * 16 + vpt) {
    case 2 * 256 + 0 * 16 + 2: return pick_tile<2, 0, 2>(standard, fwd, energy);
    case 3 * 256 + 1 * 16 + 2: return pick_tile<3, 1, 2>(standard, fwd, energy);
    case 3 * 256 + 0 * 16 + 2: return pick_tile<3, 0, 2>(standard, fwd, energy);
    
    case 4 * 256 + 2 * 16 + 2: return pick_tile<4, 2, 2>(standard, fwd, energy);
    case 4 * 256 + 1 * 16 + 2: return pick_tile<4, 1, 2>(standard, fwd, energy);
    case 4 * 256 + 0 * 16 + 1: return pick_tile<4, 0, 1>(standard, fwd, energy);
    case 5 * 256 + 2 * 16 + 2: return pick_tile<5, 2, 2>(standard, fwd, energy);
    case 5 * 256 + 3 * 16 + 2: return pick_tile<5, 3, 2>(standard, fwd, energy);
    // 256-thread CTAs (tile of 16 ids per thread), four rows per lane group
    case 4 * 256 + 1 * 16 + 4 + 8: return pick_tile<4, 1, 4, 256>(standard, fwd, energy);
    case 4 * 256 + 2 * 16 + 4 + 8: return pick_tile<4, 2, 4, 256>(standard, fwd, energy);
    case 4 * 256 + 1 * 16 + 2 + 8: return pick_tile<4, 1, 2, 256>(standard, fwd, energy);
    default: return nullptr;
  }
}

}  // namespace hygt_gpu
