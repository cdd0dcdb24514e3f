// microbench_pair.cu -- tcgen05.mma kind::f16 rate with CTA pairs (cta_group::2, M = 256) against
// single CTAs (M = 128), N = 128 / 256, K = 16, SWIZZLE_128B K-major operands resident in shared
// memory (random fp16 data), one accumulator chain or two interleaved accumulators; all SMs busy.
// Design input for hygt_gemm.cu (one N = 256 unit per tile, passes of 16 K steps into one
// accumulator). Build:
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/microbench_pair tools/microbench_pair.cu
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
__host__ __device__ constexpr uint32_t idesc_f16(int n, int m) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

// A: 128 rows x 4 K atoms (64 fp16 each) = 64 KB; B: BN rows x 4 atoms
template <bool PAIR, int NN, int NACC, int MM = PAIR ? 256 : 128>
__global__ void __cluster_dims__(PAIR ? 2 : 1, 1, 1) rate(int iters, int commit_every, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t base_sh;
  __shared__ __align__(8) uint64_t bar, cbar;
  constexpr int BN = PAIR ? NN / 2 : NN;
  const int warp = threadIdx.x >> 5;
  uint32_t rank = 0;
  if (PAIR) asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (warp == 0) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&base_sh)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&base_sh)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  uint32_t seed = 12345u + threadIdx.x * 7919u + blockIdx.x * 104729u;
  for (int i = threadIdx.x; i < (128 * 512 + BN * 512) / 4; i += blockDim.x) {
    seed = seed * 1664525u + 1013904223u;
    const uint32_t h0 = 0x3000u | ((seed >> 8) & 0x3ffu), h1 = 0x3000u | ((seed >> 18) & 0x3ffu);
    reinterpret_cast<uint32_t*>(sm)[i] = h0 | (h1 << 16) | ((seed & 1u) << 15);
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&cbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = base_sh;
  if (threadIdx.x == 0 && rank == 0) {
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 128 * 512);
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ka = 0; ka < 4; ++ka)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint64_t da = desc_sw128(a + ka * 16384 + 32 * j), db = desc_sw128(b + ka * BN * 128 + 32 * j);
          const uint32_t d = tm + (uint32_t)(((ka * 4 + j) % NACC) * NN);
          const uint32_t acc = (it | ka | j) ? 1u : 0u;
          if (PAIR)
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                         "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                         :: "r"(d), "l"(da), "l"(db), "r"(idesc_f16(NN, MM)), "r"(acc));
          else
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                         :: "r"(d), "l"(da), "l"(db), "r"(idesc_f16(NN, 128)), "r"(acc));
          if (commit_every && ((ka * 4 + j + 1) & (commit_every - 1)) == 0) {
            if (PAIR)
              asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                           :: "r"(smem_u32(&cbar)), "h"((uint16_t)3) : "memory");
            else
              asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&cbar)) : "memory");
          }
        }
    }
    if (PAIR)
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                   :: "r"(smem_u32(&bar)), "h"((uint16_t)1) : "memory");
    else
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)));
    asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W%=;\n}\n"
                 :: "r"(smem_u32(&bar)));
    cycles[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  if (warp == 0) {
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" :: "r"(tm));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tm));
  }
}

template <bool PAIR, int NN, int NACC, int MM = PAIR ? 256 : 128>
int run(int sms, unsigned long long* cyc, int ce = 0, int threads = 128, int extra = 0) {
  const int iters = 2000;
  constexpr int BN = PAIR ? NN / 2 : NN;
  const int smem = 128 * 512 + BN * 512 + 1024 + extra;
  cudaFuncSetAttribute(rate<PAIR, NN, NACC, MM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaMemset(cyc, 0, sizeof(unsigned long long) * sms);
  rate<PAIR, NN, NACC, MM><<<sms / 2 * 2, threads, smem>>>(iters, ce, cyc);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("error %s\n", cudaGetErrorString(cudaGetLastError())); return 1; }
  std::vector<unsigned long long> h(sms);
  cudaMemcpy(h.data(), cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
  double mean = 0;
  int n = 0;
  for (auto v : h) if (v) { mean += (double)v; ++n; }
  mean /= n;
  const double per = mean / (iters * 16.0);
  const double mac_per_sm = (double)MM * NN * 16 / (PAIR ? 2 : 1);
  printf("%s M=%d N=%3d accumulators %d, commit every %2d, %d threads, smem %d: %.1f cycles/instr, %.0f MAC/clk/SM (ideal cycles %.0f at 4096)\n",
         PAIR ? "cta_group::2" : "cta_group::1", MM, NN, NACC, ce, threads, smem, per, mac_per_sm / per, mac_per_sm / 4096);
  return 0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* cyc;
  cudaMalloc(&cyc, sizeof(unsigned long long) * sms);
  int e = 0;
  for (int ce : {0, 16, 4, 1}) {
    e |= run<true, 256, 1>(sms, cyc, ce);
    e |= run<true, 256, 2>(sms, cyc, ce);
    e |= run<false, 256, 1>(sms, cyc, ce);
    e |= run<false, 128, 1>(sms, cyc, ce);
  }
  return e;
}
