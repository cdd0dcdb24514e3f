// hygt_jit.h -- NVRTC-specialised kernels for N <= 64 (see hygt_jit.cpp).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "hygt_plan.h"

namespace hygt_gpu {

struct JitKernels {
  bool ok = false;
  cudaLibrary_t lib[2] = {nullptr, nullptr};
  cudaKernel_t fn[2] = {nullptr, nullptr};
  int warps = 16;
  uint32_t tile_rows = 4096;
  size_t smem = 0;
};

bool jit_supported(int log2n, int classes, int rounds);
size_t jit_smem_bytes(int log2n, int classes, int warps, int tile_rows);
// Returns 0, or a C-ABI status with `err` set.
int jit_build(int log2n, int rounds, int classes, const double* angles, const uint16_t* perms,
              uint32_t mask, bool standard, JitKernels& out, std::string& err);
void jit_release(JitKernels& k);
// Code generation + NVRTC only (no device needed): total cubin bytes of both directions.
int jit_compile_only(int log2n, int rounds, int classes, const double* angles,
                     const uint16_t* perms, uint32_t mask, bool standard, size_t* cubin_bytes,
                     std::string& err);
int jit_launch(const JitKernels& k, int dir, const float* x, float* y, const uint32_t* idx,
               const uint32_t* seg_end, uint32_t nseg, uint64_t count, int classes, int num_sms,
               cudaStream_t st);

// Per-class kernels for N = 32 / 64 (plan path "clsjit"): one NVRTC module per class holding its
// forward and inverse kernels, launched as one programmatic chain over the class buckets.
struct JitClsKernels {
  bool ok = false;
  std::vector<cudaLibrary_t> lib;
  std::vector<cudaKernel_t> fn[2];
  unsigned grid = 0;
  int threads = 32;
};
bool jit_cls_supported(int log2n, int classes, int rounds);
int jit_cls_build(int log2n, int rounds, int classes, const double* angles, const uint16_t* perms,
                  uint32_t mask, bool standard, JitClsKernels& out, std::string& err);
void jit_cls_release(JitClsKernels& k);
int jit_cls_launch(const JitClsKernels& k, int dir, const float* x, float* y, const uint32_t* idx,
                   const uint32_t* seg_end, int classes, cudaStream_t st);

// The same chain for fixed-point plans (int64 rows, bit-exact with forward_fixed/inverse_fixed):
// per-class kernels with the (c, s) TrigTable pairs as immediates. idx == nullptr: one launch
// of class 0's kernels over rows [0, count) in order.
bool jit_fixed_supported(int log2n, int rounds, int classes);
int jit_fixed_build(int log2n, int rounds, int classes, int angle_bits, int precision_bits,
                    const uint16_t* codes, const int32_t* ct, const int32_t* sn, const uint16_t* perms,
                    uint32_t perm_mask, JitClsKernels& out, std::string& err);
int jit_fixed_launch(const JitClsKernels& k, int dir, const int64_t* x, int64_t* y, const uint32_t* idx,
                     const uint32_t* seg_end, int classes, uint64_t count, unsigned long long* err,
                     cudaStream_t st);

}  // namespace hygt_gpu
