// microbench_ldcu.cu -- throughput of FFMA with uniform-register coefficients loaded from the
// kernel parameter bank (LDCU.128 -> FFMA R, R, UR, R), the coefficient path of hygt_cls.cuh.
// Variants: REUSE = FFMAs per loaded coefficient (1 = one per FFMA, as the cls kernel at VPT=1).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_ldcu tools/microbench_ldcu.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NK = 1536;
struct Blk { float k[NK]; };

template <int REUSE>
__global__ void __launch_bounds__(32) k_ldcu(const __grid_constant__ Blk p, float* out, int iters) {
  float v[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < NK / REUSE; ++j) {
#pragma unroll
      for (int r = 0; r < REUSE; ++r) {
        const int a = (j * REUSE + r) & 63, b = (a + 17 + j) & 63;
        v[a] = fmaf(p.k[j], v[b], v[a]);
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 64; ++i) s += v[i];
  out[blockIdx.x * 32 + threadIdx.x] = s;
}

// the same with a warp-varying table offset (LDC R, c[0x0][R + imm]: per-thread registers)
template <int REUSE>
__global__ void __launch_bounds__(32) k_ldc(const __grid_constant__ Blk p, float* out, int iters) {
  float v[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i] = threadIdx.x + i;
#ifdef LDC_THREAD
  const int w = (int)(threadIdx.x >> 5) * (NK / 2);  // 0, but not provably warp-uniform: LDC
#else
  const int w = (int)(blockIdx.x & 1) * (NK / 2);  // warp-uniform: LDCU c[0x0][UR + imm]
#endif
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < NK / 2 / REUSE; ++j) {
#pragma unroll
      for (int r = 0; r < REUSE; ++r) {
        const int a = (j * REUSE + r) & 63, b = (a + 17 + j) & 63;
        v[a] = fmaf(p.k[w + j], v[b], v[a]);
      }
    }
#pragma unroll
    for (int j = 0; j < NK / 2 / REUSE; ++j) {
#pragma unroll
      for (int r = 0; r < REUSE; ++r) {
        const int a = (j * REUSE + r) & 63, b = (a + 23 + j) & 63;
        v[a] = fmaf(p.k[w + j], v[b], v[a]);
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 64; ++i) s += v[i];
  out[blockIdx.x * 32 + threadIdx.x] = s;
}

__global__ void __launch_bounds__(32) k_reg(float* out, int iters, float c0) {
  float v[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i] = threadIdx.x + i;
  float k[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) k[i] = c0 + i * 1e-3f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < NK; ++j) {
      const int a = j & 63, b = (a + 17 + j) & 63;
      v[a] = fmaf(k[j & 7], v[b], v[a]);
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 64; ++i) s += v[i];
  out[blockIdx.x * 32 + threadIdx.x] = s;
}

template <class F>
void timeit(const char* name, F launch, double ffma_per_warp) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaEventRecord(a);
  launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("%-28s %8.3f ms  %6.1f lane-FFMA/clk/SM @1.965GHz\n", name, ms,
         ffma_per_warp * 32 / (ms * 1e-3) / sms / 1.965e9);
}

int main() {
  Blk h;
  for (int i = 0; i < NK; ++i) h.k[i] = 1e-4f * (i % 7);
  float* out;
  cudaMalloc(&out, 148 * 64 * 32 * 4);
  const int iters = 64;
  for (int warps : {8, 16, 24}) {
    const int grid = 148 * warps;
    char nm[64];
    snprintf(nm, sizeof nm, "reg   warps/SM=%d", warps);
    timeit(nm, [&] { k_reg<<<grid, 32>>>(out, iters, 0.5f); }, (double)grid * iters * NK);
    snprintf(nm, sizeof nm, "ldcu reuse=1 warps/SM=%d", warps);
    timeit(nm, [&] { k_ldcu<1><<<grid, 32>>>(h, out, iters); }, (double)grid * iters * NK);
    snprintf(nm, sizeof nm, "ldcu reuse=2 warps/SM=%d", warps);
    timeit(nm, [&] { k_ldcu<2><<<grid, 32>>>(h, out, iters); }, (double)grid * iters * NK);
    snprintf(nm, sizeof nm, "ldcu reuse=4 warps/SM=%d", warps);
    timeit(nm, [&] { k_ldcu<4><<<grid, 32>>>(h, out, iters); }, (double)grid * iters * NK);
    snprintf(nm, sizeof nm, "ldc-idx reuse=1 warps/SM=%d", warps);
    timeit(nm, [&] { k_ldc<1><<<grid, 32>>>(h, out, iters); }, (double)grid * iters * NK);
    snprintf(nm, sizeof nm, "ldc-idx reuse=2 warps/SM=%d", warps);
    timeit(nm, [&] { k_ldc<2><<<grid, 32>>>(h, out, iters); }, (double)grid * iters * NK);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
