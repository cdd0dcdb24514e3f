// hygt_nvtx.h -- NVTX ranges around the C ABI entry points (header-only NVTX3: no library is
// linked, the ranges cost a branch unless a profiler such as nsys / ncu --nvtx is attached).
#pragma once
#include <nvtx3/nvToolsExt.h>

namespace hygt_gpu {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace hygt_gpu
#define HYGT_NVTX(name) ::hygt_gpu::NvtxRange hygt_nvtx_range_(name)
