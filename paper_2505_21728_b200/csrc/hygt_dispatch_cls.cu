// hygt_dispatch_cls.cu -- instantiations and host-side helpers of the per-class launch kernel
// (hygt_cls.cuh): parameter block layout, occupancy, and the programmatic launch chain.
#include "hygt_dispatch.h"
#include "hygt_cls.cuh"

#include <cstring>

namespace hygt_gpu {

namespace {

template <int LOG2N, int R>
struct ClsOps {
  using Blk = ClsParams<LOG2N, R>;
  static const void* fn(bool fwd, int vpt) {
    if (vpt == 2)
      return fwd ? reinterpret_cast<const void*>(hygt_cls_kernel<LOG2N, R, 2, true>)
                 : reinterpret_cast<const void*>(hygt_cls_kernel<LOG2N, R, 2, false>);
    return fwd ? reinterpret_cast<const void*>(hygt_cls_kernel<LOG2N, R, 1, true>)
               : reinterpret_cast<const void*>(hygt_cls_kernel<LOG2N, R, 1, false>);
  }
  static void fill(void* blk, const float4* coef, uint32_t cw, const uint16_t* gt, uint32_t gmask) {
    Blk* b = static_cast<Blk*>(blk);
    std::memset(b, 0, sizeof(Blk));
    std::memcpy(b->coef, coef, sizeof(float4) * (cw < (uint32_t)Blk::CW ? cw : (uint32_t)Blk::CW));
    for (int k = 0; k <= R; ++k)
      for (int i = 0; i < Blk::N; ++i) b->gat[k][i] = gt ? gt[k * Blk::N + i] : 0u;
    b->gmask = gmask;
  }
  static void bind(void* blk, const float* x, float* y, const uint32_t* idx, const uint32_t* seg_end,
                   uint32_t bin, uint32_t copy_bin) {
    Blk* b = static_cast<Blk*>(blk);
    b->x = x;
    b->y = y;
    b->idx = idx;
    b->seg_end = seg_end;
    b->bin = bin;
    b->copy_bin = copy_bin;
  }
};

template <int LOG2N, class F>
bool dispatch(int rounds, F&& f) {
  switch (rounds) {
    case 1: f(ClsOps<LOG2N, 1>{}); return true;
    case 2: f(ClsOps<LOG2N, 2>{}); return true;
    case 3: f(ClsOps<LOG2N, 3>{}); return true;
    case 4: f(ClsOps<LOG2N, 4>{}); return true;
    default: return false;
  }
}

template <class F>
bool any(int log2n, int rounds, F&& f) {
  if (log2n == 6) return dispatch<6>(rounds, f);
  return false;
}

}  // namespace

size_t cls_param_bytes(int log2n, int rounds) {
  size_t s = 0;
  any(log2n, rounds, [&](auto ops) { s = sizeof(typename decltype(ops)::Blk); });
  return s;
}

uint32_t cls_smem_bytes(int log2n, int vpt) { return cls_warp_bytes(log2n, vpt); }

const void* cls_kernel(int log2n, int rounds, bool fwd, int vpt) {
  const void* f = nullptr;
  any(log2n, rounds, [&](auto ops) { f = decltype(ops)::fn(fwd, vpt); });
  return f;
}

void cls_fill(int log2n, int rounds, void* blk, const float4* coef, uint32_t cw, const uint16_t* gt,
              uint32_t gmask) {
  any(log2n, rounds, [&](auto ops) { decltype(ops)::fill(blk, coef, cw, gt, gmask); });
}

// Launches the class grids of one direction: blks = C parameter blocks of cls_param_bytes each.
cudaError_t cls_launch_chain(int log2n, int rounds, bool fwd, const unsigned char* blks, int classes,
                             const float* x, float* y, const uint32_t* idx, const uint32_t* seg_end,
                             unsigned grid, int vpt, cudaStream_t st) {
  cudaError_t err = cudaSuccess;
  const bool ok = any(log2n, rounds, [&](auto ops) {
    using Ops = decltype(ops);
    typename Ops::Blk blk;
    const void* fn = Ops::fn(fwd, vpt);
    for (int c = 0; c < classes && err == cudaSuccess; ++c) {
      std::memcpy(static_cast<void*>(&blk), blks + (size_t)c * sizeof(blk), sizeof(blk));
      Ops::bind(&blk, x, y, idx, seg_end, (uint32_t)c, c == classes - 1 ? 1u : 0u);
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(32);
      cfg.dynamicSmemBytes = cls_warp_bytes(log2n, vpt);
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = c > 0 ? 1 : 0;  // the first grid follows the bucketing normally
      void* args[1] = {&blk};
      err = cudaLaunchKernelExC(&cfg, fn, args);
    }
  });
  return ok ? err : cudaErrorInvalidValue;
}

}  // namespace hygt_gpu
