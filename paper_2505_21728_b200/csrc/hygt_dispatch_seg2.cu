// hygt_dispatch_seg2.cu -- instantiations of the thread-per-row bucketed kernel (hygt_seg2.cuh).
#include "hygt_dispatch.h"

namespace hygt_gpu {

Seg2Fn select_seg2(int log2n, bool standard, bool fwd) {
  constexpr int V = SEG2_VPT, W = SEG2_WARPS;
  if (log2n == 6) {
    if (standard) return fwd ? hygt_seg2_kernel<6, V, true, true, W> : hygt_seg2_kernel<6, V, true, false, W>;
    return fwd ? hygt_seg2_kernel<6, V, false, true, W> : hygt_seg2_kernel<6, V, false, false, W>;
  }
  return nullptr;
}

}  // namespace hygt_gpu
