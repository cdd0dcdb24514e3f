// microbench_i8.cu -- tcgen05.mma kind::i8 instruction rate at the shapes of the correlation
// kernel (hygt_corr_tc.cu): M = 128, K = 32, N = 64 / 128 / 256, SWIZZLE_128B K-major operands in
// shared memory, one issuing thread, operands rotating over 8 slices (as the digit slices do),
// accumulating into one TMEM block or rotating over the TMEM blocks.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/microbench_i8 tools/microbench_i8.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

template <int NN, bool ROT>
__global__ void mma_rate(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];  // 16 slices of 64 rows x 128 B
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t base_sh;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < 16 * 8192 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = base_sh;
  if (threadIdx.x == 0) {
    const uint32_t s0 = smem_u32(sm);
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      // A: two adjacent slices (M = 128) starting at slice it % 7; B: NN / 64 slices from (it * 3) % 8 + 8 - NN / 64 ...
      const uint32_t a = s0 + (uint32_t)(it % 7) * 8192u;
      const uint32_t b = s0 + (uint32_t)(8 + (it * 3) % (8 - NN / 64 + 1)) * 8192u;
      const uint32_t d = tm + (ROT ? (uint32_t)((it % (512 / NN)) * NN) : 0u);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t da = desc_sw128(a) + 2u * j, db = desc_sw128(b) + 2u * j;
        const uint32_t acc = (it >= 512 / NN || j) ? 1u : 0u;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                     :: "r"(d), "l"(da), "l"(db), "r"(idesc_i8(NN)), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)));
    asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W%=;\n}\n"
                 :: "r"(smem_u32(&bar)));
    cycles[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tm));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* cyc;
  cudaMalloc(&cyc, sizeof(unsigned long long) * sms);
  const int iters = 4000, smem = 16 * 8192 + 1024;
  auto run = [&](auto kern, int nn, bool rot) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<sms, 128, smem>>>(iters, cyc);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("error %s\n", cudaGetErrorString(cudaGetLastError())); return; }
    std::vector<unsigned long long> h(sms);
    cudaMemcpy(h.data(), cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (auto v : h) mean += (double)v / sms;
    const double per = mean / (iters * 4.0);
    printf("tcgen05.mma kind::i8 M=128 N=%3d K=32 (%s accumulator): %.1f cycles/instr (math: %d), %.0f MAC/clk/SM\n", nn,
           rot ? "rotating" : "one", per, 128 * nn * 32 / 8192, 128.0 * nn * 32 / per);
  };
  run(mma_rate<64, false>, 64, false);
  run(mma_rate<64, true>, 64, true);
  run(mma_rate<128, false>, 128, false);
  run(mma_rate<128, true>, 128, true);
  run(mma_rate<256, false>, 256, false);
  run(mma_rate<256, true>, 256, true);
  return 0;
}
