// hygt_corr_tc.h -- per-class second moments on the tensor cores (hygt_corr_tc.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace hygt_gpu {

struct CorrTcParams {
  const float* x;
  const uint32_t* idx;      // bucketed position -> row (nullptr: identity, one class)
  const uint32_t* seg_end;  // [C+1] run ends
  int n;                    // samples per row: 64, 128 or 256
  int classes;
  uint64_t count;
  double* sum;              // [C][N][N]
  unsigned long long* cnt;  // [C]
  uint64_t cta_span;        // set by corr_tc_run
  int dbg;                  // development switches (HYGT_CORR_DBG through the test hook)
};

bool corr_tc_supported(int log2n);
int corr_tc_run(const CorrTcParams& P, int sms, cudaStream_t st);

}  // namespace hygt_gpu
