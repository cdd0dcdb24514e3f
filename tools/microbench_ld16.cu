// microbench_ld16.cu -- fragment layout of tcgen05.ld.16x256b (design check for a staging-free
// epilogue): TMEM lane l, column c is written with 1000 l + c through tcgen05.st.32x32b (thread =
// lane), then warp 0 reads lanes 0-15 with tcgen05.ld.16x256b.x2 and prints what each thread got.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/microbench_ld16 tools/microbench_ld16.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void k(uint32_t* out) {
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" :: "r"((uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  // warp w writes lanes 32w .. 32w + 31, columns 0..15
  uint32_t v[16];
  for (int c = 0; c < 16; ++c) v[c] = (uint32_t)((warp * 32 + lane) * 1000 + c);
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
               :: "r"(tm + ((uint32_t)(warp * 32) << 16)), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]),
                  "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
  asm volatile("tcgen05.wait::st.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tm));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 8; ++i) out[lane * 8 + i] = r[i];
  }
  if (warp == 1) {  // the same from lane 16 (second half of the quadrant): base lane in bits 16+
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tm + ((uint32_t)(32 + 16) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 8; ++i) out[256 + lane * 8 + i] = r[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" :: "r"(tm));
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 512 * 4);
  k<<<1, 128>>>(d);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("error %s\n", cudaGetErrorString(cudaGetLastError())); return 1; }
  uint32_t h[512];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  for (int part = 0; part < 2; ++part) {
    printf(part ? "warp 1, base lane 48:\n" : "warp 0, base lane 0:\n");
    for (int t = 0; t < 32; ++t) {
      printf("t%2d:", t);
      for (int i = 0; i < 8; ++i) printf(" (%u,%u)", h[part * 256 + t * 8 + i] / 1000, h[part * 256 + t * 8 + i] % 1000);
      printf("\n");
    }
  }
  return 0;
}
