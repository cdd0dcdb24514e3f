// hygt_klt.cu -- dense per-class KLT comparison path (config 4):
//   y = K_c x  (klt_forward, statistics.hpp:222-224 -> multiply, matrix.hpp:70-80)
//   x = K_c^T y (transposed, matrix.hpp:82-88)
// Round-1 implementation: fp32 SIMT dot products with the row staged in shared memory and the
// per-class basis streamed through L1/L2 (fp32 accumulate, so it meets the fp32 parity bar). The
// tcgen05 grouped-GEMM version is the planned replacement ("KLT").
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hygt_gpu.h"

struct hygt_klt_plan {
  int n = 0, classes = 0;
  float* d_k = nullptr;   // [C][n][n]   rows = basis vectors
  float* d_kt = nullptr;  // [C][n][n]   transposed
};

int hygt_set_error(int status, const char* msg);  // hygt_capi.cu

namespace {
int kfail(int st, const std::string& m) { return hygt_set_error(st, m.c_str()); }

constexpr int KT = 256;

// out[r][i] = sum_j M[c][i][j] in[r][j], read through MT[c][j][i] so consecutive threads (i)
// read consecutive addresses.
__global__ void __launch_bounds__(KT) klt_kernel(const float* __restrict__ in, float* out,
                                                 const uint16_t* __restrict__ cls,
                                                 uint64_t count, int n, int classes,
                                                 const float* __restrict__ mt) {
  extern __shared__ float xs[];
  const int rows_per_cta = KT / n;
  const int rl = threadIdx.x / n, i = threadIdx.x % n;
  for (uint64_t r0 = (uint64_t)blockIdx.x * rows_per_cta; r0 < count;
       r0 += (uint64_t)gridDim.x * rows_per_cta) {
    __syncthreads();
    for (int k = threadIdx.x; k < rows_per_cta * n; k += KT) {
      const uint64_t r = r0 + k / n;
      xs[k] = r < count ? in[r * n + (k % n)] : 0.f;
    }
    __syncthreads();
    const uint64_t r = r0 + rl;
    if (rl < rows_per_cta && r < count) {
      int c = cls ? cls[r] : 0;
      if (c >= classes) c = 0;
      const float* m = mt + (size_t)c * n * n;
      const float* xv = xs + rl * n;
      float acc = 0.f;
      for (int j = 0; j < n; ++j) acc = fmaf(__ldg(m + (size_t)j * n + i), xv[j], acc);
      out[r * n + i] = acc;
    }
  }
}

int run_klt(const hygt_klt_plan* p, bool fwd, const float* in, float* out, const uint16_t* cls,
            uint64_t count, cudaStream_t st) {
  if (!p) return kfail(HYGT_ERR_ARGUMENT, "klt: null plan");
  if (!count) return HYGT_OK;
  if (in == out) return kfail(HYGT_ERR_ARGUMENT, "klt: in-place not supported");
  const int rows_per_cta = KT / p->n;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t ctas = std::min<uint64_t>((count + rows_per_cta - 1) / rows_per_cta, (uint64_t)sms * 8);
  // forward y = K x  -> MT = K^T ; inverse x = K^T y -> MT = K
  klt_kernel<<<(unsigned)ctas, KT, KT * sizeof(float), st>>>(in, out, cls, count, p->n,
                                                             p->classes, fwd ? p->d_kt : p->d_k);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return kfail(HYGT_ERR_CUDA, cudaGetErrorString(e));
  return HYGT_OK;
}
}  // namespace

extern "C" int hygt_klt_plan_create(int n, int class_count, const double* k, uint32_t flags,
                                    hygt_klt_plan** out) {
  (void)flags;
  if (!out || !k) return kfail(HYGT_ERR_ARGUMENT, "hygt_klt_plan_create: null argument");
  *out = nullptr;
  if (n < 2 || n > KT || (n & (n - 1))) return kfail(HYGT_ERR_ARGUMENT, "hygt_klt_plan_create: n must be a power of two in [2, 256]");
  if (class_count < 1) return kfail(HYGT_ERR_ARGUMENT, "hygt_klt_plan_create: class_count");
  const size_t nn = (size_t)n * n * class_count;
  std::vector<float> kf(nn), ktf(nn);
  for (int c = 0; c < class_count; ++c)
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        const float v = (float)k[((size_t)c * n + i) * n + j];
        kf[((size_t)c * n + i) * n + j] = v;
        ktf[((size_t)c * n + j) * n + i] = v;
      }
  hygt_klt_plan* p = new hygt_klt_plan();
  p->n = n;
  p->classes = class_count;
  if (cudaMalloc(&p->d_k, nn * sizeof(float)) != cudaSuccess ||
      cudaMalloc(&p->d_kt, nn * sizeof(float)) != cudaSuccess ||
      cudaMemcpy(p->d_k, kf.data(), nn * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->d_kt, ktf.data(), nn * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess) {
    hygt_klt_plan_destroy(p);
    return kfail(HYGT_ERR_CUDA, "hygt_klt_plan_create: device allocation failed");
  }
  *out = p;
  return HYGT_OK;
}

extern "C" int hygt_klt_plan_destroy(hygt_klt_plan* p) {
  if (!p) return HYGT_OK;
  cudaFree(p->d_k);
  cudaFree(p->d_kt);
  delete p;
  return HYGT_OK;
}

extern "C" size_t hygt_klt_workspace_bytes(const hygt_klt_plan* plan, uint64_t count) {
  (void)plan;
  (void)count;
  return 0;
}

extern "C" int hygt_klt_forward_f32(const hygt_klt_plan* plan, const float* d_x, float* d_y,
                                    const uint16_t* d_cls, uint64_t count, void* d_ws,
                                    size_t ws_bytes, void* stream) {
  (void)d_ws;
  (void)ws_bytes;
  return run_klt(plan, true, d_x, d_y, d_cls, count, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int hygt_klt_inverse_f32(const hygt_klt_plan* plan, const float* d_y, float* d_x,
                                    const uint16_t* d_cls, uint64_t count, void* d_ws,
                                    size_t ws_bytes, void* stream) {
  (void)d_ws;
  (void)ws_bytes;
  return run_klt(plan, false, d_y, d_x, d_cls, count, reinterpret_cast<cudaStream_t>(stream));
}
