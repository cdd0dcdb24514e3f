// microbench_contend.cu -- tcgen05.mma rate under contention from other warps of the same SM
// (design input for hygt_gemm.cu at N = 256, where the MMAs run at ~2x their ideal cycles).
// One CTA pair per two SMs, rank 0 issues back-to-back MMAs:
//   SS: cta_group::2 M = 256, N = 256, A and B from shared memory (the current kernel's form)
//   TS: cta_group::2 M = 256, N = 128, A from TMEM, B from shared memory (the TS form)
// while 8 background warps per CTA do, until the MMAs finish:
//   0 nothing, 1 STS.64 stream (the split's fp16 stores), 2 LDS.128 stream, 3 FFMA chains,
//   4 LDG.128 + STG.128 streaming HBM (the split's loads and the epilogue's stores), 5 = 1 + 4.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/microbench_contend tools/microbench_contend.cu
#include <cuda_fp16.h>
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

constexpr int OPS_BYTES = 128 * 512 * 2;  // A (128 rows x 256 K fp16) + B (128 rows x 256 K)
constexpr int BG_BYTES = 64 * 1024;       // background shared-memory region
constexpr int THREADS = 12 * 32;          // warps 0-3 TMEM / MMA, 4-11 background

template <bool TS>
__global__ void __cluster_dims__(2, 1, 1) contend(int iters, int mode, int commit_every, int cmode, int bg_warps, float4* gbuf, size_t gfloat4,
                                                  unsigned long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar, cbar[4];
  __shared__ volatile int done;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t rank;
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = tid; i < OPS_BYTES / 4; i += blockDim.x) {
    const uint32_t s = (uint32_t)i * 2654435761u;
    reinterpret_cast<uint32_t*>(sm)[i] = (0x3000u | ((s >> 8) & 0x3ffu)) | ((0x3000u | ((s >> 18) & 0x3ffu)) << 16);
  }
  if (tid == 0) done = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
    for (int i = 0; i < 4; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&cbar[i])), "r"((cmode & 7) == 3 ? (1 << 19) : 1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (warp < 4) {
    if (TS) {  // A (this CTA's 128 rows) into TMEM columns [0, 128)
      for (int c0 = 0; c0 < 128; c0 += 8) {
        uint32_t v[8];
        for (int i = 0; i < 8; ++i) v[i] = 0x3c003c00u ^ (uint32_t)((c0 + i + tid) & 0x3ff);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                     :: "r"(tm + ((uint32_t)(warp * 32) << 16) + c0), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]),
                        "r"(v[5]), "r"(v[6]), "r"(v[7]));
      }
      asm volatile("tcgen05.wait::st.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  auto issue_loop = [&](bool leader) {
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 128 * 512);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ka = 0; ka < 4; ++ka)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t acc = (ka | j) ? 1u : 0u;
          if (leader && (cmode & 32)) {  // one asm block per K atom: 4 MMAs, descriptor steps inside
            if (j == 0) {
              if (TS) {
                const uint64_t db = desc_sw128(b + ka * 64 * 128);
                asm volatile("{\n.reg .pred p;\n.reg .b64 bd;\n.reg .b32 ad;\nsetp.ne.b32 p, %4, 0;\n"
                             "mov.b64 bd, %2;\nmov.b32 ad, %1;\n"
                             "tcgen05.mma.cta_group::2.kind::f16 [%0], [ad], bd, %3, p;\n"
                             "add.s64 bd, bd, 2;\nadd.s32 ad, ad, 8;\n"
                             "tcgen05.mma.cta_group::2.kind::f16 [%0], [ad], bd, %3, 1;\n"
                             "add.s64 bd, bd, 2;\nadd.s32 ad, ad, 8;\n"
                             "tcgen05.mma.cta_group::2.kind::f16 [%0], [ad], bd, %3, 1;\n"
                             "add.s64 bd, bd, 2;\nadd.s32 ad, ad, 8;\n"
                             "tcgen05.mma.cta_group::2.kind::f16 [%0], [ad], bd, %3, 1;\n}\n"
                             :: "r"(tm + 256 + (uint32_t)((it & 1) * 128)), "r"(tm + (uint32_t)(ka * 32)), "l"(db),
                                "r"(idesc_f16(128, 256)), "r"((uint32_t)ka));
              } else {
                const uint64_t da = desc_sw128(a + ka * 16384), db = desc_sw128(b + ka * 16384);
                asm volatile("{\n.reg .pred p;\n.reg .b64 ad, bd;\nsetp.ne.b32 p, %4, 0;\n"
                             "mov.b64 ad, %1;\nmov.b64 bd, %2;\n"
                             "tcgen05.mma.cta_group::2.kind::f16 [%0], ad, bd, %3, p;\n"
                             "add.s64 ad, ad, 2;\nadd.s64 bd, bd, 2;\n"
                             "tcgen05.mma.cta_group::2.kind::f16 [%0], ad, bd, %3, 1;\n"
                             "add.s64 ad, ad, 2;\nadd.s64 bd, bd, 2;\n"
                             "tcgen05.mma.cta_group::2.kind::f16 [%0], ad, bd, %3, 1;\n"
                             "add.s64 ad, ad, 2;\nadd.s64 bd, bd, 2;\n"
                             "tcgen05.mma.cta_group::2.kind::f16 [%0], ad, bd, %3, 1;\n}\n"
                             :: "r"(tm + (uint32_t)((it & 1) * 256)), "l"(da), "l"(db), "r"(idesc_f16(256, 256)), "r"((uint32_t)ka));
              }
            }
          } else if (leader) {
            if (TS) {
              const uint64_t db = desc_sw128(b + ka * 64 * 128) + 2 * j;
              asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                           "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                           :: "r"(tm + 256 + (uint32_t)((it & 1) * 128)), "r"(tm + (uint32_t)((ka * 4 + j) * 8)), "l"(db),
                              "r"(idesc_f16(128, 256)), "r"(acc));
            } else {
              const uint64_t da = desc_sw128(a + ka * 16384) + 2 * j, db = desc_sw128(b + ka * 16384) + 2 * j;
              asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                           "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                           :: "r"(tm + (uint32_t)((it & 1) * 256)), "l"(da), "l"(db), "r"(idesc_f16(256, 256)), "r"(acc));
            }
          }
          if (commit_every && ((ka * 4 + j + 1) & (commit_every - 1)) == 0) {
            if ((cmode & 7) == 5) __syncwarp();
            if (leader || (cmode & 7) == 6) {
              const int ci = (ka * 4 + j) >> (commit_every == 16 ? 4 : commit_every == 4 ? 2 : 0);
              if ((cmode & 7) == 2)  // this CTA's barrier only
                asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                             :: "r"(smem_u32(&cbar[0])) : "memory");
              else
                asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                             :: "r"(smem_u32(&cbar[(cmode & 7) == 4 ? (ci & 3) : 0])), "h"((uint16_t)((cmode & 16) ? 1 : 3)) : "memory");
            }
          }
        }
    }
  };
  if (warp == 0) {
    if (rank == 0 && ((cmode & 7) >= 5 || (cmode & 64))) {  // the whole warp runs the loop, elect.sync picks the issuer
      uint32_t is_leader;
      asm volatile("{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\nselp.u32 %0, 1, 0, p;\n}\n" : "=r"(is_leader));
      const unsigned long long t0 = clock64();
      issue_loop(is_leader != 0);
      __syncwarp();
      if (is_leader) {
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                     :: "r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
        asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W%=;\n}\n" :: "r"(smem_u32(&bar)));
        cyc[blockIdx.x] = clock64() - t0;
        done = 1;
      }
      __syncwarp();
    } else if (lane == 0 && rank == 0) {
      const unsigned long long t0 = clock64();
      issue_loop(true);
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                   :: "r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
      asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W%=;\n}\n" :: "r"(smem_u32(&bar)));
      cyc[blockIdx.x] = clock64() - t0;
      done = 1;
    } else if (lane == 0 && !(cmode & 8)) {
      asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W%=;\n}\n" :: "r"(smem_u32(&bar)));
      done = 1;
    }
  } else if (warp >= 4 && warp < 4 + bg_warps && mode != 0) {
    const int bw = warp - 4;
    unsigned char* bg = sm + OPS_BYTES;
    float acc0 = (float)tid, acc1 = 1.f, acc2 = 2.f, acc3 = 3.f;
    size_t gi = ((size_t)blockIdx.x * 8 + bw) * 32 + lane;
    const size_t gstride = (size_t)gridDim.x * 8 * 32;
    uint32_t x = tid;
    while (!done) {
      if (mode == 1 || mode == 5) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
          *reinterpret_cast<uint2*>(bg + ((bw * 16 + r) * 512 + lane * 16) % BG_BYTES + (lane & 1) * 8) = make_uint2(x + r, x ^ r);
      }
      if (mode == 2) {
        uint4 s = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const uint4 v = *reinterpret_cast<const uint4*>(bg + ((bw * 16 + r) * 512 + lane * 16) % BG_BYTES);
          s.x ^= v.x; s.y += v.y;
        }
        x += s.x + s.y;
      }
      if (mode == 3) {
#pragma unroll
        for (int r = 0; r < 64; ++r) {
          acc0 = fmaf(acc0, 1.0001f, 0.5f); acc1 = fmaf(acc1, 0.9999f, 0.25f);
          acc2 = fmaf(acc2, 1.0002f, 0.5f); acc3 = fmaf(acc3, 0.9998f, 0.25f);
        }
      }
      if (mode == 6) {  // the split's conversion: scale, fp16 pack, unpack, residual, pack
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const float a0 = acc0 * 1.5f, a1 = acc1 * 1.5f;
          __half2 h = __floats2half2_rn(a0, a1);
          const float2 b = __half22float2(h);
          __half2 l = __floats2half2_rn(a0 - b.x, a1 - b.y);
          acc0 += __low2float(l) + 1e-3f;
          acc1 += __high2float(h) * 1e-6f;
        }
      }
      if (mode == 4 || mode == 5) {
        float4 v[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) v[r] = __ldcs(gbuf + (gi + r * gstride) % gfloat4);
#pragma unroll
        for (int r = 0; r < 4; ++r) __stcs(gbuf + (gi + r * gstride + gfloat4 / 2) % gfloat4, v[r]);
        gi += 4 * gstride;
      }
    }
    if (acc0 + acc1 + acc2 + acc3 == 1234.5f || x == 77u) gbuf[0] = make_float4(acc0, acc1, acc2, (float)x);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" :: "r"(tm));
}

template <bool TS>
void run(int sms, int mode, int commit_every, int cmode, int bg_warps, float4* g, size_t nf4, unsigned long long* cyc) {
  const int iters = 400;
  const int smem = OPS_BYTES + BG_BYTES;
  cudaFuncSetAttribute(contend<TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaMemset(cyc, 0, 8 * sms);
  contend<TS><<<sms / 2 * 2, THREADS, smem>>>(iters, mode, commit_every, cmode, bg_warps, g, nf4, cyc);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("error %s\n", cudaGetErrorString(cudaGetLastError())); return; }
  std::vector<unsigned long long> h(sms);
  cudaMemcpy(h.data(), cyc, 8 * sms, cudaMemcpyDeviceToHost);
  double mean = 0;
  int n = 0;
  for (auto v : h) if (v) { mean += (double)v; ++n; }
  mean /= n;
  static const char* names[] = {"none", "STS.64", "LDS.128", "FFMA", "LDG+STG HBM", "STS.64 + HBM", "fp16 split"};
  static const char* cnames[] = {"-", "multicast", "local", "multicast, count 2^19", "multicast, 4 barriers",
                                 "converged warp, elect.sync issue, syncwarp", "converged warp, all lanes commit", "-"};
  printf("%s  background %-13s x%d warps, commit every %2d (%s%s%s%s%s): %.1f cycles per MMA (ideal %d)\n",
         TS ? "TS M256 N128" : "SS M256 N256", names[mode], bg_warps, commit_every, cnames[commit_every ? (cmode & 7) : 0], (cmode & 8) ? ", peer not waiting" : "", (cmode & 16) ? ", mask 1" : "", (cmode & 32) ? ", asm block per atom" : "", (cmode & 64) ? ", converged" : "",
         mean / (iters * 16.0), TS ? 64 : 128);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 8 * sms);
  const size_t nf4 = (size_t)1 << 28;  // 4 GB
  float4* g;
  cudaMalloc(&g, nf4 * 16);
  cudaMemset(g, 0, nf4 * 16);
  for (int mode : {0, 6, 3})
    for (int cm : {1, 1 | 64, 1 | 32, 1 | 32 | 64}) {
      run<false>(sms, mode, 4, cm, 8, g, nf4, cyc);
      run<true>(sms, mode, 4, cm, 8, g, nf4, cyc);
    }
  return 0;
}
