// hygt_dispatch_stage.cu -- instantiations of the TMA-staged kernel (hygt_stage.cuh).
#include "hygt_dispatch.h"

namespace hygt_gpu {

StageFn select_stage(int log2n, bool standard, bool fwd) {
  constexpr int V = STAGE_VPT, W = STAGE_WARPS;
  if (log2n == 4) {
    if (standard) return fwd ? hygt_stage_kernel<4, V, true, true, W> : hygt_stage_kernel<4, V, true, false, W>;
    return fwd ? hygt_stage_kernel<4, V, false, true, W> : hygt_stage_kernel<4, V, false, false, W>;
  }
  return nullptr;
}

StageSortFn select_stage_sort() { return hygt_stage_sort_kernel<STAGE_VPT>; }

}  // namespace hygt_gpu
