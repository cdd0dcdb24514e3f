// hygt_dispatch_segment.cu -- instantiations of the segment kernel.
#include "hygt_dispatch.h"

namespace hygt_gpu {
namespace {
template <int LOG2N, int L, int VPT, bool PF>
SegFn pick_seg(bool standard, bool fwd, bool energy) {
  constexpr int TT = SEG_THREADS;
  if (standard) {
    if (!fwd) return hygt_segment_kernel<LOG2N, L, VPT, true, false, false, PF, TT>;
    return energy ? hygt_segment_kernel<LOG2N, L, VPT, true, true, true, PF, TT>
                  : hygt_segment_kernel<LOG2N, L, VPT, true, true, false, PF, TT>;
  }
  if (!fwd) return hygt_segment_kernel<LOG2N, L, VPT, false, false, false, PF, TT>;
  return energy ? hygt_segment_kernel<LOG2N, L, VPT, false, true, true, PF, TT>
                : hygt_segment_kernel<LOG2N, L, VPT, false, true, false, PF, TT>;
}

}  // namespace

SegFn select_seg(int variant, bool standard, bool fwd, bool energy) {
  switch (variant) {
    case 0: return pick_seg<6, 1, 1, true>(standard, fwd, energy);
    case 1: return pick_seg<6, 1, 2, false>(standard, fwd, energy);
    case 2: return pick_seg<6, 2, 2, true>(standard, fwd, energy);
    case 3: return pick_seg<6, 0, 1, false>(standard, fwd, energy);
    case 4: return pick_seg<7, 2, 1, true>(standard, fwd, energy);
    case 5: return pick_seg<7, 2, 2, false>(standard, fwd, energy);
    case 6: return pick_seg<8, 2, 1, false>(standard, fwd, energy);
    case 7: return pick_seg<8, 2, 1, true>(standard, fwd, energy);
    case 8: return pick_seg<8, 1, 1, false>(standard, fwd, energy);
    case 9: return pick_seg<8, 3, 2, false>(standard, fwd, energy);
    case 10: return pick_seg<8, 2, 2, false>(standard, fwd, energy);
    default: return nullptr;
  }
}

}  // namespace hygt_gpu
