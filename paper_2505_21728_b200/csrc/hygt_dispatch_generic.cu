// hygt_dispatch_generic.cu -- instantiations of the bucketed apply kernel.
#include "hygt_dispatch.h"

namespace hygt_gpu {
namespace {

template <int LOG2N, int L>
ApplyFn pick_apply(bool standard, bool fwd, bool energy) {
  if (standard) {
    if (!fwd) return hygt_apply_kernel<LOG2N, L, true, false, false>;
    return energy ? hygt_apply_kernel<LOG2N, L, true, true, true>
                  : hygt_apply_kernel<LOG2N, L, true, true, false>;
  }
  if (!fwd) return hygt_apply_kernel<LOG2N, L, false, false, false>;
  return energy ? hygt_apply_kernel<LOG2N, L, false, true, true>
                : hygt_apply_kernel<LOG2N, L, false, true, false>;
}

}  // namespace

// Instantiated (log2 N, log2 TPV) layouts.
ApplyFn select_apply(int log2n, int l, bool standard, bool fwd, bool energy) {
  switch (log2n * 16 + l) {
    case 1 * 16 + 0: return pick_apply<1, 0>(standard, fwd, energy);
    case 2 * 16 + 0: return pick_apply<2, 0>(standard, fwd, energy);
    case 3 * 16 + 0: return pick_apply<3, 0>(standard, fwd, energy);
    case 4 * 16 + 0: return pick_apply<4, 0>(standard, fwd, energy);
    case 4 * 16 + 2: return pick_apply<4, 2>(standard, fwd, energy);
    case 5 * 16 + 0: return pick_apply<5, 0>(standard, fwd, energy);
    case 6 * 16 + 0: return pick_apply<6, 0>(standard, fwd, energy);
    case 6 * 16 + 1: return pick_apply<6, 1>(standard, fwd, energy);
    case 6 * 16 + 2: return pick_apply<6, 2>(standard, fwd, energy);
    case 7 * 16 + 2: return pick_apply<7, 2>(standard, fwd, energy);
    case 8 * 16 + 1: return pick_apply<8, 1>(standard, fwd, energy);
    case 8 * 16 + 2: return pick_apply<8, 2>(standard, fwd, energy);
    default: return nullptr;
  }
}

}  // namespace hygt_gpu
