// hygt_dispatch.h -- kernel selection tables (instantiated in hygt_dispatch_*.cu so the
// template instantiations compile in parallel).
#pragma once
#include "hygt_kernels.cuh"
#include "hygt_segment.cuh"
#include "hygt_tile.cuh"

namespace hygt_gpu {
using ApplyFn = void (*)(ApplyParams);
using TileFn = void (*)(TileParams);
using SegFn = void (*)(SegParams);
constexpr int TILE_THREADS = 512;
constexpr int SEG_THREADS = 256;
ApplyFn select_apply(int log2n, int l, bool standard, bool fwd, bool energy);
TileFn select_tile(int log2n, int l, int vpt, bool standard, bool fwd, bool energy);
SegFn select_seg(int variant, bool standard, bool fwd, bool energy);
}  // namespace hygt_gpu
