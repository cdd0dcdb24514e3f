// microbench_tc.cu -- design inputs for the tensor-core HyGT/KLT kernel (hygt_gemm.cu):
//   1. L2 -> SM read bandwidth (all SMs re-reading an L2-resident buffer), LDG.128 and
//      cp.async.bulk (TMA) into shared memory;
//   2. TMEM -> register bandwidth (tcgen05.ld.32x32b.x32) with 4 / 8 / 16 warps per SM;
//   3. tcgen05.mma kind::f16 (M = 128, K = 16, SWIZZLE_128B K-major operands) issue rate at
//      N = 64 / 128 / 256, one issuing thread.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/microbench_tc tools/microbench_tc.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 1;                                                               \
    }                                                                         \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// ---------------------------------------------------------------- 1. L2 read bandwidth ----
__global__ void l2_ldg(const uint4* __restrict__ buf, size_t n16, int iters, unsigned long long* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int it = 0; it < iters; ++it)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
      uint4 v;
      asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(buf + i));
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) atomicAdd(sink, 1ull);
}

// each CTA streams `chunks` 32 KB pieces of the buffer (offset by its id) through a 4-slot ring
__global__ void l2_tma(const uint8_t* __restrict__ buf, size_t bytes, int chunks, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[4];
  constexpr uint32_t CH = 32768;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const size_t nch = bytes / CH;
  uint32_t phase[4] = {0, 0, 0, 0};
  for (int k = 0; k < chunks + 4; ++k) {
    const int s = k & 3;
    if (k >= 4) {  // wait for the copy issued 4 steps ago
      asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W%=;\n}\n"
                   :: "r"(smem_u32(&bar[s])), "r"(phase[s]));
      phase[s] ^= 1;
    }
    if (k < chunks) {
      const size_t c = ((size_t)blockIdx.x * 7 + k) % nch;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[s])), "r"(CH));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(smem_u32(sm + s * CH)), "l"(buf + c * CH), "r"(CH), "r"(smem_u32(&bar[s])) : "memory");
    }
  }
  if (sm[5] == 0x7f && sm[77] == 0x3) atomicAdd(sink, 1ull);
}

// ---------------------------------------------------------------- 2. TMEM read rate -------
__global__ void tmem_ld(int iters, unsigned long long* cycles, unsigned long long* sink) {
  __shared__ uint32_t base_sh;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = base_sh;
  const int nw = blockDim.x >> 5;
  const int sub = warp & 3, slice = warp >> 2, slices = nw >> 2;  // warps sharing a subpartition split columns
  const int cols = 512 / slices;
  uint32_t acc = 0;
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
    for (int c = slice * cols; c < (slice + 1) * cols; c += 32) {
      uint32_t r[32];
      const uint32_t addr = tm + ((uint32_t)(sub * 32) << 16) + (uint32_t)c;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
            "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
            "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(addr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += r[j];
    }
  const unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (acc == 0x9999u) atomicAdd(sink, 1ull);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tm));
}

// ---------------------------------------------------------------- 3. MMA issue rate -------
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_f16(int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

template <int NN>
__global__ void mma_rate(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t base_sh;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&base_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < (128 * 128 + NN * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
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
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 128 * 128);
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t da = desc_sw128(a + 32 * j), db = desc_sw128(b + 32 * j);
        const uint32_t acc = (it | j) ? 1u : 0u;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                     :: "r"(tm), "l"(da), "l"(db), "r"(idesc_f16(NN)), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)));
    asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W%=;\n}\n"
                 :: "r"(smem_u32(&bar)));
    const unsigned long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tm));
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  // 1. L2 bandwidth on buffers of 8 / 16 / 32 MB (L2 resident), LDG and TMA
  for (size_t mb : {8, 16, 32, 64}) {
    const size_t bytes = mb << 20;
    uint8_t* buf;
    CK(cudaMalloc(&buf, bytes));
    CK(cudaMemset(buf, 1, bytes));
    const int iters = (int)(2048 / mb);
    l2_ldg<<<sms * 4, 512>>>((const uint4*)buf, bytes / 16, 2, sink);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    l2_ldg<<<sms * 4, 512>>>((const uint4*)buf, bytes / 16, iters, sink);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("L2 LDG.cg  buffer %3zu MB: %.1f GB/s\n", mb, (double)bytes * iters / (ms * 1e-3) / 1e9);
    CK(cudaFuncSetAttribute(l2_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768));
    const int chunks = 2048;
    for (int ctas_per_sm : {1}) {
      l2_tma<<<sms * ctas_per_sm, 32, 4 * 32768>>>(buf, bytes, 64, sink);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      l2_tma<<<sms * ctas_per_sm, 32, 4 * 32768>>>(buf, bytes, chunks, sink);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      printf("L2 TMA 32KB buffer %3zu MB: %.1f GB/s (%d CTA/SM)\n", mb, (double)sms * ctas_per_sm * chunks * 32768.0 / (ms * 1e-3) / 1e9, ctas_per_sm);
    }
    cudaFree(buf);
  }
  // 2. TMEM read rate
  unsigned long long* cyc;
  CK(cudaMalloc(&cyc, sizeof(unsigned long long) * sms));
  for (int warps : {4, 8, 16}) {
    const int iters = 200;
    tmem_ld<<<sms, warps * 32>>>(iters, cyc, sink);
    CK(cudaDeviceSynchronize());
    std::vector<unsigned long long> h(sms);
    CK(cudaMemcpy(h.data(), cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost));
    double mean = 0;
    for (auto v : h) mean += (double)v / sms;
    const double bytes = (double)iters * 128 * 512 * 4;  // the whole 128 x 512 fp32 TMEM per iteration
    printf("TMEM ld 32x32b.x32, %2d warps: %.1f B/clk per SM (%.0f cycles for %d full reads)\n", warps,
           bytes / mean, mean, iters);
  }
  // 3. MMA issue rate
  const int iters = 4000;
  auto run_mma = [&](auto kern, int nn) -> int {
    const int smem = 128 * 128 + nn * 128 + 1024;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<sms, 128, smem>>>(iters, cyc);
    CK(cudaDeviceSynchronize());
    std::vector<unsigned long long> h(sms);
    CK(cudaMemcpy(h.data(), cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost));
    double mean = 0;
    for (auto v : h) mean += (double)v / sms;
    const double per = mean / (iters * 4.0);
    printf("tcgen05.mma kind::f16 M=128 N=%3d K=16: %.1f cycles/instr (model 128*N/256 = %d), %.0f TFLOP/s chip at %d MHz\n",
           nn, per, 128 * nn / 256, 2.0 * 128 * nn * 16 / per * sms * clk_khz * 1e3 / 1e12, clk_khz / 1000);
    return 0;
  };
  if (run_mma(mma_rate<64>, 64)) return 1;
  if (run_mma(mma_rate<128>, 128)) return 1;
  if (run_mma(mma_rate<256>, 256)) return 1;
  return 0;
}
