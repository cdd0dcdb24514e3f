// microbench_ts2.cu -- design check for the CTA-pair TS form of the N = 256 composed operator
// (hygt_gemm.cu, hygt_gemm_ts_kernel): D[M = 256 output columns][N data rows] = OP . X^T with
//   * OP (the class operator, 256 x 256 K fp16) in TMEM, written by tcgen05.st.32x32b (thread =
//     output column = TMEM lane, TMEM column j = fp16 pair K 2j, 2j + 1, low half = even K):
//     each CTA of the pair holds its 128 output columns;
//   * X (data rows, K-major SWIZZLE_128B in shared memory): each CTA holds N / 2 rows;
//   * tcgen05.mma.cta_group::2.kind::f16 [d], [a_tmem], b_desc, idesc(M = 256, N).
// 1. correctness against a host reference (K = 256, both CTAs' D halves);
// 2. rate, all SMs busy: N = 64 / 128 / 256, one or two accumulators.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/microbench_ts2 tools/microbench_ts2.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
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
__device__ __forceinline__ uint32_t swz(int r, int q) { return (uint32_t)r * 128u + (uint32_t)((q ^ (r & 7)) << 4); }
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// OP: [256][256] fp16 row-major (row = output column m, K); X: [NN][256] fp16 (row n, K);
// D: [256][NN] fp32. 128 threads.
template <int NN, int NACC>
__global__ void __cluster_dims__(2, 1, 1) ts2(const __half* OP, const __half* X, float* D, int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  constexpr int BN = NN / 2;  // data rows in this CTA
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cta_rank();
  // this CTA's data rows rank * BN .. into 4 K atoms of BN x 128 B
  for (int i = tid; i < BN * 256; i += blockDim.x) {
    const int r = i / 256, k = i % 256;
    *reinterpret_cast<__half*>(sm + (k / 64) * BN * 128 + swz(r, (k % 64) / 8) + (k % 8) * 2) = X[(size_t)(rank * BN + r) * 256 + k];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  const uint32_t ta = tm;        // OP: columns [0, 128)
  const uint32_t td = tm + 128;  // D: columns [128, 128 + NACC NN)
  {  // thread = output column m = rank 128 + tid: its 256 K as 128 packed columns
    const uint32_t* src = reinterpret_cast<const uint32_t*>(OP + (size_t)(rank * 128 + tid) * 256);
    for (int c0 = 0; c0 < 128; c0 += 32) {
      uint32_t v[32];
      for (int i = 0; i < 32; ++i) v[i] = src[c0 + i];
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
          "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
          :: "r"(ta + ((uint32_t)(warp * 32) << 16) + c0), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]),
             "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
             "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]),
             "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0 && rank == 0) {
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ka = 0; ka < 4; ++ka)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint64_t db = desc_sw128(smem_u32(sm + ka * BN * 128)) + 2 * j;
          const uint32_t d = td + (uint32_t)((((it * 16 + ka * 4 + j) / 4) % NACC) * NN);
          const uint32_t acc = (ka | j) ? 1u : 0u;
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                       :: "r"(iters == 1 ? td : d), "r"(ta + (uint32_t)((ka * 4 + j) * 8)), "l"(db), "r"(idesc_f16(NN, 256)), "r"(acc));
        }
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 :: "r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
    if (cyc) cyc[blockIdx.x] = 0;  // written below after completion
    asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W%=;\n}\n" :: "r"(smem_u32(&bar)));
    if (cyc) cyc[blockIdx.x] = clock64() - t0;
  } else if (tid == 0) {
    asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W%=;\n}\n" :: "r"(smem_u32(&bar)));
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (iters == 1) {
    for (int c = 0; c < NN; c += 8) {
      uint32_t v[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                   : "r"(td + ((uint32_t)(warp * 32) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int i = 0; i < 8; ++i) D[(size_t)(rank * 128 + warp * 32 + lane) * NN + c + i] = __uint_as_float(v[i]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" :: "r"(tm));
}

template <int NN, int NACC>
int run() {
  std::vector<__half> A(256 * 256), X(NN * 256);
  std::vector<double> Af(A.size()), Xf(X.size());
  for (size_t i = 0; i < A.size(); ++i) { A[i] = __float2half((float)((int)(i * 37 % 101) - 50) / 32.f); Af[i] = __half2float(A[i]); }
  for (size_t i = 0; i < X.size(); ++i) { X[i] = __float2half((float)((int)(i * 53 % 97) - 48) / 64.f); Xf[i] = __half2float(X[i]); }
  __half *dA, *dX;
  float* dD;
  unsigned long long* dc;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dX, X.size() * 2);
  cudaMalloc(&dD, 256 * NN * 4);
  cudaMalloc(&dc, 8 * sms);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dX, X.data(), X.size() * 2, cudaMemcpyHostToDevice);
  const int smem = NN / 2 * 512;
  cudaFuncSetAttribute(ts2<NN, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  ts2<NN, NACC><<<2, 128, smem>>>(dA, dX, dD, 1, nullptr);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<float> D(256 * NN);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int m = 0; m < 256; ++m)
    for (int n = 0; n < NN; ++n) {
      double ref = 0;
      for (int k = 0; k < 256; ++k) ref += Af[(size_t)m * 256 + k] * Xf[(size_t)n * 256 + k];
      maxerr = fmax(maxerr, fabs(ref - D[(size_t)m * NN + n]));
    }
  const int iters = 500;
  cudaMemset(dc, 0, 8 * sms);
  ts2<NN, NACC><<<sms / 2 * 2, 128, smem>>>(dA, dX, dD, iters, dc);
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<unsigned long long> h(sms);
  cudaMemcpy(h.data(), dc, 8 * sms, cudaMemcpyDeviceToHost);
  double mean = 0;
  int n = 0;
  for (auto v : h) if (v) { mean += (double)v; ++n; }
  mean /= n;
  printf("TS pair M=256 N=%3d accumulators %d: max |D - ref| = %.3g, %.1f cycles per MMA (ideal %d)\n", NN, NACC, maxerr,
         mean / (iters * 16.0), NN / 2);
  cudaFree(dA); cudaFree(dX); cudaFree(dD); cudaFree(dc);
  return 0;
}

int main() {
  int e = 0;
  e |= run<64, 1>();
  e |= run<128, 1>();
  e |= run<128, 2>();
  e |= run<256, 1>();
  return e;
}
