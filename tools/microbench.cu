// microbench.cu -- throughput probes for the HyGT kernel design decisions on B200:
// FFMA (3-reg), FFMA2 (fma.rn.f32x2), SHFL, uniform-address LDS.128 and per-lane LDS.128.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }

constexpr int ITERS = 4096;

__global__ void k_ffma(float* out, float a, float b) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  float ra = a + threadIdx.x * 1e-9f, rb = b;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[i]) : "f"(ra), "f"(rb));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float* out, float a, float b) {
  u64 x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = pk(threadIdx.x + i, i);
  u64 ra = pk(a + threadIdx.x * 1e-9f, a), rb = pk(b, b);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma2(x[i], ra, rb);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) { float2 f = *reinterpret_cast<float2*>(&x[i]); s += f.x + f.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_shfl(float* out) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __shfl_xor_sync(0xffffffffu, x[i], 1 + (i & 3));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// LDS.128: all lanes of a warp read the same address (uniform) or lane-distinct addresses.
template <bool UNIFORM>
__global__ void k_lds(float* out, int stride) {
  __shared__ float4 tab[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) tab[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  float4 acc = make_float4(0, 0, 0, 0);
  const int lane = threadIdx.x & 31;
  int base = UNIFORM ? 0 : lane;
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float4 v;
      const int idx = (base + (it * 8 + i) * stride) & 2047;
      asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                   : "r"((unsigned)__cvta_generic_to_shared(&tab[idx])));
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

// Stream copy kernel (HBM ceiling with 128-bit cache-streaming loads/stores).
__global__ void k_copy(const float4* __restrict__ a, float4* b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(b + i, __ldcs(a + i));
}

template <class F>
float timeit(F f) {
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  f();
  cudaEventRecord(s);
  for (int r = 0; r < 5; ++r) f();
  cudaEventRecord(e);
  cudaEventSynchronize(e);
  float ms;
  cudaEventElapsedTime(&ms, s, e);
  return ms / 5;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, sizeof(float) * sms * 8 * 1024);
  const int blocks = sms * 8, threads = 256;
  const double lanes = (double)blocks * threads;
  double ms = timeit([&] { k_ffma<<<blocks, threads>>>(out, 0.999f, 0.001f); });
  printf("FFMA   : %.1f Glane-instr/s -> %.1f lane-instr/clk/SM @%d MHz\n", lanes * ITERS * 8 / ms / 1e6,
         lanes * ITERS * 8 / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  ms = timeit([&] { k_ffma2<<<blocks, threads>>>(out, 0.999f, 0.001f); });
  printf("FFMA2  : %.1f Glane-instr/s -> %.1f lane-instr/clk/SM (x2 flop pairs)\n", lanes * ITERS * 8 / ms / 1e6,
         lanes * ITERS * 8 / (ms * 1e-3) / sms / (clk * 1e3));
  ms = timeit([&] { k_shfl<<<blocks, threads>>>(out); });
  printf("SHFL   : %.1f lane-op/clk/SM\n", lanes * ITERS / 4 * 8 / (ms * 1e-3) / sms / (clk * 1e3));
  ms = timeit([&] { k_lds<true><<<blocks, threads>>>(out, 1); });
  printf("LDS128 uniform    : %.2f warp-instr/clk/SM\n", lanes / 32 * ITERS / 4 * 8 / (ms * 1e-3) / sms / (clk * 1e3));
  ms = timeit([&] { k_lds<false><<<blocks, threads>>>(out, 32); });
  printf("LDS128 per-lane   : %.2f warp-instr/clk/SM\n", lanes / 32 * ITERS / 4 * 8 / (ms * 1e-3) / sms / (clk * 1e3));
  size_t n = (size_t)1 << 28;  // 4 GiB per buffer (float4)
  float4 *a, *b;
  cudaMalloc(&a, n * 16);
  cudaMalloc(&b, n * 16);
  cudaMemset(a, 0, n * 16);
  ms = timeit([&] { k_copy<<<sms * 8, 256>>>(a, b, n); });
  printf("copy   : %.0f GB/s (read+write)\n", 2.0 * n * 16 / (ms * 1e-3) / 1e9);
  printf("(clock attr %d MHz; real clock under load may differ)\n", clk / 1000);
  return 0;
}
