// microbench2.cu -- data-movement probes for the HyGT tile design on B200.
//  1. random 64 B / 256 B / 1 KB row gathers from a 2 GiB array: LDG (row-cooperative lanes)
//     vs cp.async.bulk (TMA, one bulk copy per row) -> achieved GB/s
//  2. coefficient delivery: LDC (constant bank, per-warp class offset) vs LDS.128 broadcast
//  3. SHFL and LDS issued together: do they share a pipe?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// ---- 1a: LDG gathers: a group of ROWB/16 lanes reads one row (float4 per lane), sums it.
template <int ROWB>
__global__ void gather_ldg(const float4* __restrict__ x, const uint32_t* __restrict__ idx, uint64_t rows, float* out) {
  constexpr int LPR = ROWB / 16 < 32 ? ROWB / 16 : 32;  // lanes per row
  constexpr int RPW = 32 / LPR;
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  float acc = 0.f;
  for (uint64_t r0 = warp * RPW; r0 < rows; r0 += nwarps * RPW) {
    const uint64_t r = r0 + lane / LPR;
    if (r < rows) {
      const uint64_t row = idx[r];
#pragma unroll
      for (int k = 0; k < ROWB / 16 / LPR; ++k) {
        const float4 v = __ldcs(x + row * (ROWB / 16) + (lane % LPR) + k * LPR);
        acc += v.x + v.y + v.z + v.w;
      }
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

// ---- 1b: TMA bulk gathers: each lane copies one row (cp.async.bulk global->shared), 2 stages.
template <int ROWB>
__global__ void gather_tma(const char* __restrict__ x, const uint32_t* __restrict__ idx, uint64_t rows, float* out) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar[2];
  const int tid = threadIdx.x;
  const int R = blockDim.x;  // rows per stage = threads
  char* buf[2] = {sm, sm + (size_t)R * ROWB};
  if (tid == 0) {
    for (int s = 0; s < 2; ++s) asm volatile("mbarrier.init.shared.b64 [%0], %1;" :: "r"(smem_u32(&bar[s])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  float acc = 0.f;
  uint32_t phase[2] = {0, 0};
  uint64_t it = 0;
  for (uint64_t r0 = blockIdx.x * (uint64_t)R; r0 < rows; r0 += gridDim.x * (uint64_t)R, ++it) {
    const int s = it & 1;
    const uint64_t r = r0 + tid;
    const int nvalid = (int)((rows - r0) < (uint64_t)R ? (rows - r0) : R);
    if (tid == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[s])), "r"(nvalid * ROWB));
    __syncthreads();
    if (r < rows) {
      const uint64_t row = idx[r];
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(smem_u32(buf[s] + (size_t)tid * ROWB)), "l"(x + row * ROWB), "r"(ROWB), "r"(smem_u32(&bar[s])) : "memory");
    }
    // wait
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }"
                 :: "r"(smem_u32(&bar[s])), "r"(phase[s]) : "memory");
    phase[s] ^= 1;
    const float4* v = reinterpret_cast<const float4*>(buf[s] + (size_t)tid * ROWB);
    acc += v[0].x;
    __syncthreads();
  }
  if (acc == 12345.f) out[0] = acc;
}

// ---- 2: coefficient delivery. Each warp uses class (warp % 35); reads the 208 floats of
// that class sequentially (config-2 sized table, 35 x 832 B = 29 KB) and FMAs them.
__constant__ float4 ctab[35 * 52];
__global__ void coef_ldc(float* out, int reps) {
  const int cls = (threadIdx.x >> 5) % 35 + blockIdx.x % 3;
  float a = threadIdx.x, b = 1.f;
  for (int r = 0; r < reps; ++r) {
#pragma unroll 4
    for (int k = 0; k < 52; ++k) {
      const float4 q = ctab[(cls % 35) * 52 + k];
      a = fmaf(a, q.x, q.y);
      b = fmaf(b, q.z, q.w);
    }
  }
  if (a + b == 12345.f) out[0] = a;
}
__global__ void coef_lds(const float4* g, float* out, int reps) {
  __shared__ float4 tab[35 * 52];
  for (int i = threadIdx.x; i < 35 * 52; i += blockDim.x) tab[i] = g[i];
  __syncthreads();
  const int cls = (threadIdx.x >> 5) % 35 + blockIdx.x % 3;
  float a = threadIdx.x, b = 1.f;
  for (int r = 0; r < reps; ++r) {
#pragma unroll 4
    for (int k = 0; k < 52; ++k) {
      const float4 q = tab[(cls % 35) * 52 + k];
      a = fmaf(a, q.x, q.y);
      b = fmaf(b, q.z, q.w);
    }
  }
  if (a + b == 12345.f) out[0] = a;
}

// ---- 3: SHFL alone, LDS alone, both interleaved.
template <bool DO_SHFL, bool DO_LDS>
__global__ void mix(float* out, int reps) {
  __shared__ float tab[32 * 64];
  for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) tab[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float s[4] = {1, 2, 3, 4}, l[4] = {0, 0, 0, 0};
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (DO_SHFL) s[k] = __shfl_xor_sync(0xffffffffu, s[k], k + 1);
      if (DO_LDS) l[k] += tab[((r * 4 + k) & 63) * 32 + lane];
    }
  }
  if (s[0] + s[1] + s[2] + s[3] + l[0] + l[1] + l[2] + l[3] == 12345.f) out[0] = 1;
}

template <class F>
float timeit(F f, int reps = 5) {
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  f();
  cudaEventRecord(s);
  for (int r = 0; r < reps; ++r) f();
  cudaEventRecord(e);
  cudaEventSynchronize(e);
  float ms;
  cudaEventElapsedTime(&ms, s, e);
  return ms / reps;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = (size_t)2 << 30;
  char* x;
  float* out;
  CK(cudaMalloc(&x, bytes));
  CK(cudaMemset(x, 1, bytes));
  CK(cudaMalloc(&out, 1024));
  const uint64_t maxrows = bytes / 64;
  uint32_t* idx;
  CK(cudaMalloc(&idx, maxrows * 4));
  // idx: a class-bucketed order -- rows of "class" c (= row % 35) in ascending order, classes
  // one after another (global sort), or within chunks of 16384 rows (chunked sort)
  uint32_t* h = (uint32_t*)malloc(maxrows * 4);
  auto fill = [&](uint64_t rows, uint64_t chunk) {
    uint64_t k = 0;
    for (uint64_t c0 = 0; c0 < rows; c0 += chunk) {
      const uint64_t c1 = c0 + chunk < rows ? c0 + chunk : rows;
      for (int c = 0; c < 35; ++c)
        for (uint64_t r = c0; r < c1; ++r)
          if ((r * 2654435761u >> 7) % 35 == (uint64_t)c) h[k++] = (uint32_t)r;
    }
    cudaMemcpy(idx, h, rows * 4, cudaMemcpyHostToDevice);
  };
  auto seq = [&](uint64_t rows) { for (uint64_t r = 0; r < rows; ++r) h[r] = (uint32_t)r; cudaMemcpy(idx, h, rows * 4, cudaMemcpyHostToDevice); };
  struct { const char* name; int rb; } cases[] = {{"64B", 64}, {"256B", 256}, {"1KB", 1024}};
  for (auto cs : cases) {
    const uint64_t rows = bytes / cs.rb;
    for (int mode = 0; mode < 3; ++mode) {
      if (mode == 0) seq(rows); else fill(rows, mode == 1 ? 16384 : rows);
      const char* mname = mode == 0 ? "sequential" : mode == 1 ? "chunk16K-bucketed" : "global-bucketed";
      float ms;
      if (cs.rb == 64) ms = timeit([&] { gather_ldg<64><<<sms * 8, 256>>>((const float4*)x, idx, rows, out); });
      else if (cs.rb == 256) ms = timeit([&] { gather_ldg<256><<<sms * 8, 256>>>((const float4*)x, idx, rows, out); });
      else ms = timeit([&] { gather_ldg<1024><<<sms * 8, 256>>>((const float4*)x, idx, rows, out); });
      printf("LDG gather %-5s %-18s: %7.0f GB/s (+idx)\n", cs.name, mname, bytes / (ms * 1e-3) / 1e9);
      int thr = cs.rb == 1024 ? 64 : 128;
      size_t smem = 2 * (size_t)thr * cs.rb;
      float ms2;
      if (cs.rb == 64) { cudaFuncSetAttribute(gather_tma<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); ms2 = timeit([&] { gather_tma<64><<<sms * 4, thr, smem>>>(x, idx, rows, out); }); }
      else if (cs.rb == 256) { cudaFuncSetAttribute(gather_tma<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); ms2 = timeit([&] { gather_tma<256><<<sms * 4, thr, smem>>>(x, idx, rows, out); }); }
      else { cudaFuncSetAttribute(gather_tma<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); ms2 = timeit([&] { gather_tma<1024><<<sms * 4, thr, smem>>>(x, idx, rows, out); }); }
      cudaError_t e = cudaGetLastError();
      printf("TMA gather %-5s %-18s: %7.0f GB/s %s\n", cs.name, mname, bytes / (ms2 * 1e-3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  float4* g;
  CK(cudaMalloc(&g, 35 * 52 * 16));
  cudaMemset(g, 0, 35 * 52 * 16);
  const int reps = 64;
  const double warp_instr = (double)sms * 8 * 8 * reps * 52;  // 8 blocks x 8 warps
  float ms = timeit([&] { coef_ldc<<<sms * 8, 256>>>(out, reps); });
  printf("LDC.128 coef (per-warp class)  : %.2f warp-loads/clk/SM (at 1.9 GHz)\n", warp_instr / (ms * 1e-3) / sms / 1.9e9);
  ms = timeit([&] { coef_lds<<<sms * 8, 256>>>(g, out, reps); });
  printf("LDS.128 coef (per-warp class)  : %.2f warp-loads/clk/SM\n", warp_instr / (ms * 1e-3) / sms / 1.9e9);
  const double wi = (double)sms * 8 * 8 * 4096 * 4;
  float a = timeit([&] { mix<true, false><<<sms * 8, 256>>>(out, 4096); });
  float b = timeit([&] { mix<false, true><<<sms * 8, 256>>>(out, 4096); });
  float c = timeit([&] { mix<true, true><<<sms * 8, 256>>>(out, 4096); });
  printf("SHFL only %.3f ms (%.2f/clk/SM), LDS only %.3f ms (%.2f/clk/SM), both %.3f ms\n",
         a, wi / (a * 1e-3) / sms / 1.9e9, b, wi / (b * 1e-3) / sms / 1.9e9, c);
  return 0;
}
