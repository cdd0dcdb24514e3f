// microbench3.cu -- shared-memory wavefronts per warp instruction for broadcast-style loads.
// mode: 0 LDS.32 uniform, 1 LDS.64 uniform, 2 LDS.128 uniform, 3 LDS.128 2-unique (lane&1),
//       4 LDS.128 4-unique (lane&3), 5 LDS.128 8-unique (lane&7), 6 LDS.128 32 distinct (conflict-free)
//       7 LDS.64 2-unique, 8 LDS.64 4-unique
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, int iters) {
  __shared__ float4 tab[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) tab[i] = make_float4(i, i, i, i);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float acc = 0;
  int base = 0;
  for (int it = 0; it < iters; ++it) {
    base = (base + 37) & 511;
    if (MODE == 0) { acc += reinterpret_cast<const float*>(tab)[base * 4]; }
    if (MODE == 1) { float2 v = reinterpret_cast<const float2*>(tab)[base * 2]; acc += v.x + v.y; }
    if (MODE == 2) { float4 v = tab[base]; acc += v.x + v.y + v.z + v.w; }
    if (MODE == 3) { float4 v = tab[base + (lane & 1)]; acc += v.x + v.y + v.z + v.w; }
    if (MODE == 4) { float4 v = tab[base + (lane & 3)]; acc += v.x + v.y + v.z + v.w; }
    if (MODE == 5) { float4 v = tab[base + (lane & 7)]; acc += v.x + v.y + v.z + v.w; }
    if (MODE == 6) { float4 v = tab[base + lane]; acc += v.x + v.y + v.z + v.w; }
    if (MODE == 7) { float2 v = reinterpret_cast<const float2*>(tab)[base * 2 + (lane & 1)]; acc += v.x + v.y; }
    if (MODE == 8) { float2 v = reinterpret_cast<const float2*>(tab)[base * 2 + (lane & 3)]; acc += v.x + v.y; }
  }
  if (acc == 1234.5f) out[0] = acc;
}
int main() {
  float* out; cudaMalloc(&out, 64);
  const int iters = 4096;
  k<0><<<148, 256>>>(out, iters); k<1><<<148, 256>>>(out, iters); k<2><<<148, 256>>>(out, iters);
  k<3><<<148, 256>>>(out, iters); k<4><<<148, 256>>>(out, iters); k<5><<<148, 256>>>(out, iters);
  k<6><<<148, 256>>>(out, iters); k<7><<<148, 256>>>(out, iters); k<8><<<148, 256>>>(out, iters);
  cudaDeviceSynchronize();
  printf("done\n");
  return 0;
}
