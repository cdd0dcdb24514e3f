// hygt_gemm.h -- per-class dense operators on tcgen05 (hygt_gemm.cu): the composed-operator HyGT
// path (N = 64 / 128 / 256) and the KLT comparison path.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#define HYGT_GEMM_MAX_CLASSES 512

namespace hygt_gpu {

struct GemmParams {
  const float* x;
  float* y;
  const uint32_t* idx;       // bucketed position -> row
  const uint32_t* seg_end;   // [C + 1] bucket ends (bucket C: invalid class ids)
  int classes;
  uint64_t count;
  const unsigned char* bops; // [C][stages][hi | lo][NW x 128 B] fp16, SWIZZLE_128B K-major
  const float* unscale;      // [C] 2^-kB
  double* energy;            // [C][N] fp64 (forward with energy) or nullptr
  unsigned long long* trace; // debug: per-tile clock64 events of CTA 0 ([64][16]) or nullptr
  int dbg;                   // diagnostic switches (test-hook knob HYGT_GEMM_DBG; wrong results when
                             // set): 1 B stages loaded once, 2 no L2 prefetch, 16 no output stores,
                             // 32 accumulators released unread (streamed-B variants for 1); 4 is
                             // exact: N = 256 MMAs issued by a lone lane (the pre-elect.sync form)
};

struct GemmOperands {  // one direction
  int n = 0, classes = 0, num_sms = 148;
  bool pair = true;  // CTA pairs (tcgen05 cta_group::2, M = 256): each SM streams half of B
  int dbg = 0;
  // wide: one unit of all N output columns per tile (N = 256 needs pairs) and one accumulator,
  // the correction terms of all K accumulated before the main term; otherwise units of <= 128
  // columns with separate main / correction accumulators
  bool wide = true;
  // N = 256 with CTA pairs: the class operator resident in TMEM as the MMA's A operand and the
  // data rows as B (hygt_gemm_ts_kernel); otherwise the rows are A and the operator B
  bool ts = true;
  unsigned char* d_ops = nullptr;
  float* d_unscale = nullptr;
};

bool gemm_supported(int n, int classes);
int gemm_smem_bytes(int n);
// ops: host [classes][n][n] fp64, row-major B_c with out = B_c . in per row.
int gemm_build(int n, int classes, const double* ops, GemmOperands& out);
void gemm_release(GemmOperands& g);
// Rows must already be bucketed (idx / seg_end from hygt_bucket over `classes` classes).
int gemm_run(const GemmOperands& g, const float* x, float* y, const uint32_t* idx,
             const uint32_t* seg_end, uint64_t count, double* energy, cudaStream_t st);

}  // namespace hygt_gpu
