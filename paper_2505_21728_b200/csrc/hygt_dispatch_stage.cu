// hygt_dispatch_stage.cu -- instantiations of the TMA-staged kernel (hygt_stage.cuh).
#include "hygt_dispatch.h"

namespace hygt_gpu {

template <int VAR>
static StageFn stage_variant(bool standard, bool fwd) {
  constexpr int V = STAGE_VPT, W = STAGE_WARPS;
  if (standard) return fwd ? hygt_stage_kernel<4, V, true, true, W, VAR> : hygt_stage_kernel<4, V, true, false, W, VAR>;
  return fwd ? hygt_stage_kernel<4, V, false, true, W, VAR> : hygt_stage_kernel<4, V, false, false, W, VAR>;
}

StageFn select_stage(int log2n, bool standard, bool fwd, bool debug) {
  if (log2n != 4) return nullptr;
  return debug ? stage_variant<STAGE_VAR_DEBUG>(standard, fwd) : stage_variant<0>(standard, fwd);
}

StageSortFn select_stage_sort(int vpt, uint32_t tile_rows) {
  // slot groups of 128 ids per warp: only as many as the tile needs (T = 784 -> 7, not 8)
  const bool seven = tile_rows <= 7 * 128;
  if (vpt == 2) return seven ? hygt_stage_sort_kernel<2, 7> : hygt_stage_sort_kernel<2, 8>;
  return seven ? hygt_stage_sort_kernel<STAGE_VPT, 7> : hygt_stage_sort_kernel<STAGE_VPT, 8>;
}

StageFxFn select_stage_fixed(int log2n, bool fwd) {
  if (log2n != 4) return nullptr;
  return fwd ? hygt_stage_fixed_kernel<4, STAGE_FX_VPT, true, STAGE_FX_WARPS>
             : hygt_stage_fixed_kernel<4, STAGE_FX_VPT, false, STAGE_FX_WARPS>;
}

}  // namespace hygt_gpu
