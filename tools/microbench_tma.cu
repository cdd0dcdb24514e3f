// microbench_tma.cu -- HBM -> smem -> HBM streaming with cp.async.bulk (one producer thread per
// CTA, ring of STAGES buffers of BYTES each, each buffer moved as PIECES bulk copies).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int STAGES, int PIECES>
__global__ void __launch_bounds__(32, 1) k(const char* x, char* y, uint64_t chunks, uint32_t bytes) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < STAGES; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  const uint64_t my = chunks > blockIdx.x ? (chunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const uint32_t piece = bytes / PIECES;
  auto load = [&](uint64_t kk) {
    const int s = kk % STAGES;
    const uint64_t c = blockIdx.x + kk * gridDim.x;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(bytes) : "memory");
    for (int p = 0; p < PIECES; ++p)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su32(sm + s * bytes + p * piece)), "l"(x + c * bytes + p * piece), "r"(piece), "r"(su32(&bar[s])) : "memory");
  };
  for (uint64_t kk = 0; kk < my && kk < STAGES; ++kk) load(kk);
  for (uint64_t kk = 0; kk < my; ++kk) {
    const int s = kk % STAGES;
    const uint32_t ph = (kk / STAGES) & 1;
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(su32(&bar[s])), "r"(ph) : "memory");
    const uint64_t c = blockIdx.x + kk * gridDim.x;
    for (int p = 0; p < PIECES; ++p)
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(y + c * bytes + p * piece), "r"(su32(sm + s * bytes + p * piece)), "r"(piece) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (kk + STAGES < my) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      load(kk + STAGES);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__global__ void copy128(const float4* __restrict__ a, float4* b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = __ldcs(a + i);
}
template <int STAGES, int PIECES>
void run(const char* x, char* y, size_t total, uint32_t bytes, int ctas) {
  auto fn = k<STAGES, PIECES>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, STAGES * bytes);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const uint64_t chunks = total / bytes;
  for (int w = 0; w < 2; ++w) fn<<<ctas, 32, STAGES * bytes>>>(x, y, chunks, bytes);
  cudaEventRecord(a);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) fn<<<ctas, 32, STAGES * bytes>>>(x, y, chunks, bytes);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("stages %d pieces %2d bytes %6u ctas %3d : %7.0f GB/s (read+write) %s\n", STAGES, PIECES, bytes, ctas,
         2.0 * chunks * bytes * reps / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  const size_t total = (size_t)1 << 30;
  char *x, *y; cudaMalloc(&x, total); cudaMalloc(&y, total); cudaMemset(x, 1, total);
  {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    copy128<<<148 * 8, 256>>>((const float4*)x, (float4*)y, total / 16);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) copy128<<<148 * 8, 256>>>((const float4*)x, (float4*)y, total / 16);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("LDG/STG copy: %7.0f GB/s\n", 2.0 * total * 5 / (ms * 1e-3) / 1e9);
  }
  run<2, 1>(x, y, total, 50176, 148);
  run<3, 1>(x, y, total, 50176, 148);
  run<3, 4>(x, y, total, 50176, 148);
  run<3, 16>(x, y, total, 50176, 148);
  run<4, 1>(x, y, total, 32768, 148);
  run<4, 8>(x, y, total, 32768, 148);
  run<6, 1>(x, y, total, 16384, 148);
  run<12, 1>(x, y, total, 8192, 148);
  run<3, 1>(x, y, total, 50176, 296);
  return 0;
}
