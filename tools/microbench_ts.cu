// microbench_ts.cu -- design check for A-in-TMEM ("TS") tcgen05 MMAs:
//   1. correctness: A (128 x 64 fp16, SWIZZLE_128B K-major in smem) copied to TMEM with
//      tcgen05.cp.128x256b (4 K steps of 16), then D = A . B^T by tcgen05.mma kind::f16 with A
//      from TMEM; D read back (tcgen05.ld) and compared with a host reference;
//   2. rate: back-to-back TS MMAs at N = 64 / 128 / 256 against the SS-mode rate.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/microbench_ts tools/microbench_ts.cu
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
__host__ __device__ constexpr uint32_t idesc_f16(int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ uint32_t swz(int r, int q) { return (uint32_t)r * 128u + (uint32_t)((q ^ (r & 7)) << 4); }

// A: [128][64] fp16 row-major in global; B: [NN][64] fp16; D: [128][NN] fp32
template <int NN>
__global__ void ts_check(const __half* A, const __half* B, float* D, int iters, unsigned long long* cyc, int ts) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  unsigned char* sa = sm;
  unsigned char* sb = sm + 128 * 128;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 128 * 64; i += blockDim.x) {
    const int r = i / 64, k = i % 64;
    *reinterpret_cast<__half*>(sa + swz(r, k / 8) + (k % 8) * 2) = A[i];
  }
  for (int i = tid; i < NN * 64; i += blockDim.x) {
    const int r = i / 64, k = i % 64;
    *reinterpret_cast<__half*>(sb + swz(r, k / 8) + (k % 8) * 2) = B[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  const uint32_t ta = tm + 256;  // A in TMEM columns [256, 288): 64 fp16 per row = 32 columns
  const uint32_t td = tm;        // D in columns [0, NN)
  if (tid == 0) {
    const uint64_t da = desc_sw128(smem_u32(sa)), db = desc_sw128(smem_u32(sb));
    if (ts) {
#pragma unroll
      for (int j = 0; j < 4; ++j)  // 128 rows x 32 B (16 fp16 of K) per copy
        asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" :: "r"(ta + 8 * j), "l"(da + 2 * j));
    }
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t acc = j ? 1u : 0u;
        if (ts)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                       :: "r"(td), "r"(ta + 8 * j), "l"(db + 2 * j), "r"(idesc_f16(NN)), "r"(acc));
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                       :: "r"(td), "l"(da + 2 * j), "l"(db + 2 * j), "r"(idesc_f16(NN)), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)));
    asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W%=;\n}\n" :: "r"(smem_u32(&bar)));
    *cyc = clock64() - t0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4) {
    for (int c = 0; c < NN; c += 8) {
      uint32_t v[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                   : "r"(td + ((uint32_t)(warp * 32) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int i = 0; i < 8; ++i) D[(warp * 32 + lane) * NN + c + i] = __uint_as_float(v[i]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tm));
}

template <int NN>
int run(int ts) {
  std::vector<__half> A(128 * 64), B(NN * 64);
  std::vector<float> Af(128 * 64), Bf(NN * 64);
  for (int i = 0; i < 128 * 64; ++i) { Af[i] = (float)((i * 37 % 101) - 50) / 32.f; A[i] = __float2half(Af[i]); Af[i] = __half2float(A[i]); }
  for (int i = 0; i < NN * 64; ++i) { Bf[i] = (float)((i * 53 % 97) - 48) / 64.f; B[i] = __float2half(Bf[i]); Bf[i] = __half2float(B[i]); }
  __half *dA, *dB;
  float* dD;
  unsigned long long* dc;
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dD, 128 * NN * 4);
  cudaMalloc(&dc, 8);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  const int smem = 128 * 128 + NN * 128;
  cudaFuncSetAttribute(ts_check<NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  ts_check<NN><<<1, 128, smem>>>(dA, dB, dD, 1, dc, ts);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<float> D(128 * NN);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int r = 0; r < 128; ++r)
    for (int n = 0; n < NN; ++n) {
      double ref = 0;
      for (int k = 0; k < 64; ++k) ref += (double)Af[r * 64 + k] * Bf[n * 64 + k];
      maxerr = fmax(maxerr, fabs(ref - D[r * NN + n]));
    }
  const int iters = 2000;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  ts_check<NN><<<1, 128, smem>>>(dA, dB, dD, iters, dc, ts);
  cudaDeviceSynchronize();
  unsigned long long cyc = 0;
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  printf("%s N=%3d: max |D - ref| = %.3g, %.1f cycles per MMA (K = 16)\n", ts ? "TS (A in TMEM)" : "SS (A in smem)", NN,
         maxerr, (double)cyc / (iters * 4.0));
  cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dc);
  return 0;
}

int main() {
  for (int ts : {0, 1}) {
    if (run<64>(ts) || run<128>(ts) || run<256>(ts)) return 1;
  }
  return 0;
}
