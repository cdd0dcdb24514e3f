// microbench_tma2.cu -- per-row TMA gather + scatter throughput (rows of ROWB bytes addressed by
// an index array), one warp per CTA issuing one bulk copy per lane, ring of S stages of 32 rows.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int ROWB, int S, bool STORE>
__global__ void __launch_bounds__(32 * 4) k(const char* x, char* y, const uint32_t* idx, uint64_t rows) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar[4][S];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned char* my = sm + (size_t)w * S * 32 * ROWB;
  if (lane == 0) for (int i = 0; i < S; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[w][i])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncwarp();
  const uint64_t gw = (uint64_t)blockIdx.x * 4 + w, nw = (uint64_t)gridDim.x * 4;
  const uint64_t batches = rows / 32;
  const uint64_t my_b = batches > gw ? (batches - 1 - gw) / nw + 1 : 0;
  auto load = [&](uint64_t kk) {
    const int s = kk % S;
    const uint64_t b = gw + kk * nw;
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[w][s])), "r"(32 * ROWB) : "memory");
    __syncwarp();
    const uint64_t row = idx[b * 32 + lane];
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su32(my + (s * 32 + lane) * ROWB)), "l"(x + row * ROWB), "r"(ROWB), "r"(su32(&bar[w][s])) : "memory");
  };
  for (uint64_t kk = 0; kk < my_b && kk < S - 1; ++kk) load(kk);
  for (uint64_t kk = 0; kk < my_b; ++kk) {
    const int s = kk % S;
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(su32(&bar[w][s])), "r"((uint32_t)(kk / S) & 1u) : "memory");
    if (STORE) {
      const uint64_t b = gw + kk * nw;
      const uint64_t row = idx[b * 32 + lane];
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(y + row * ROWB), "r"(su32(my + (s * 32 + lane) * ROWB)), "r"(ROWB) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(1) : "memory");  // stage kk-1 free
    }
    __syncwarp();
    if (kk + S - 1 < my_b) load(kk + S - 1);
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
template <int ROWB, int S, bool STORE>
void run(const char* x, char* y, const uint32_t* idx, uint64_t rows, const char* what) {
  auto fn = k<ROWB, S, STORE>;
  const size_t smem = (size_t)4 * S * 32 * ROWB;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 128, smem);
  const int ctas = 148 * std::max(occ, 1);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  fn<<<ctas, 128, smem>>>(x, y, idx, rows);
  cudaEventRecord(a);
  for (int r = 0; r < 3; ++r) fn<<<ctas, 128, smem>>>(x, y, idx, rows);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("%-10s rowB %5d stages %2d store %d occ %d: %7.0f GB/s (%s)\n", what, ROWB, S, (int)STORE, occ,
         (STORE ? 2.0 : 1.0) * rows * ROWB * 3 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  const size_t total = (size_t)1 << 32;
  char *x, *y; cudaMalloc(&x, total); cudaMalloc(&y, total); cudaMemset(x, 1, total);
  for (int rb : {256, 1024}) {
    const uint64_t rows = total / rb;
    std::vector<uint32_t> h(rows);
    for (uint64_t i = 0; i < rows; ++i) h[i] = (uint32_t)i;
    // class-bucketed order: 35 classes, random class per row -> rows of one class ascending
    std::mt19937 g(1);
    std::vector<uint32_t> cls(rows);
    for (auto& c : cls) c = g() % 35;
    std::stable_sort(h.begin(), h.end(), [&](uint32_t a, uint32_t b) { return cls[a] < cls[b]; });
    uint32_t* idx; cudaMalloc(&idx, rows * 4);
    cudaMemcpy(idx, h.data(), rows * 4, cudaMemcpyHostToDevice);
    uint32_t* seq; cudaMalloc(&seq, rows * 4);
    for (uint64_t i = 0; i < rows; ++i) h[i] = (uint32_t)i;
    cudaMemcpy(seq, h.data(), rows * 4, cudaMemcpyHostToDevice);
    if (rb == 256) {
      run<256, 4, false>(x, y, seq, rows, "seq");
      run<256, 4, true>(x, y, seq, rows, "seq");
      run<256, 4, true>(x, y, idx, rows, "bucketed");
      run<256, 6, true>(x, y, idx, rows, "bucketed");
    } else {
      run<1024, 2, true>(x, y, seq, rows, "seq");
      run<1024, 2, true>(x, y, idx, rows, "bucketed");
      run<1024, 3, true>(x, y, idx, rows, "bucketed");
    }
    cudaFree(idx); cudaFree(seq);
  }
  return 0;
}
