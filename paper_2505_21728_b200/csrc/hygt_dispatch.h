// hygt_dispatch.h -- kernel selection tables (instantiated in hygt_dispatch_*.cu so the
// template instantiations compile in parallel).
#pragma once
#include "hygt_kernels.cuh"
#include "hygt_segment.cuh"
#include "hygt_stage.cuh"
#include "hygt_seg2.cuh"
#include "hygt_stage_fixed.cuh"
#include "hygt_tile.cuh"

namespace hygt_gpu {
using ApplyFn = void (*)(ApplyParams);
using TileFn = void (*)(TileParams);
using SegFn = void (*)(SegParams);
using StageFn = void (*)(StageParams);
using StageSortFn = void (*)(StageSortParams);
using Seg2Fn = void (*)(Seg2Params);
using StageFxFn = void (*)(StageFxParams);
constexpr int TILE_THREADS = 512;
constexpr int SEG_THREADS = 256;
constexpr int STAGE_WARPS = 7;  // consumer warps (+ one producer warp)
constexpr int STAGE_VPT = 4;
constexpr int SEG2_WARPS = 8;
constexpr int SEG2_VPT = 2;
ApplyFn select_apply(int log2n, int l, bool standard, bool fwd, bool energy);
TileFn select_tile(int log2n, int l, int vpt, bool standard, bool fwd, bool energy);
SegFn select_seg(int variant, bool standard, bool fwd, bool energy);
StageFn select_stage(int log2n, bool standard, bool fwd, bool debug = false);
StageSortFn select_stage_sort(int vpt, uint32_t tile_rows);
constexpr int STAGE_FX_VPT = 2;
constexpr int STAGE_FX_WARPS = 7;
StageFxFn select_stage_fixed(int log2n, bool fwd);
Seg2Fn select_seg2(int log2n, bool standard, bool fwd);
// per-class launch kernel (hygt_cls.cuh, hygt_dispatch_cls.cu)
size_t cls_param_bytes(int log2n, int rounds);  // 0: unsupported shape
uint32_t cls_smem_bytes(int log2n, int vpt);
const void* cls_kernel(int log2n, int rounds, bool fwd, int vpt);
void cls_fill(int log2n, int rounds, void* blk, const float4* coef, uint32_t cw, const uint16_t* gt,
              uint32_t gmask);
cudaError_t cls_launch_chain(int log2n, int rounds, bool fwd, const unsigned char* blks, int classes,
                             const float* x, float* y, const uint32_t* idx, const uint32_t* seg_end,
                             unsigned grid, int vpt, cudaStream_t st);
}  // namespace hygt_gpu
