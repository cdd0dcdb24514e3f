// hygt_capi.cu -- libhygt_gpu.so: the extern "C" boundary (include/hygt_gpu.h), class
// bucketing, kernel dispatch, the fixed-point and KLT paths and the device-side synthetic
// workload generators. Built for sm_100a only (see __graft_entry__.build()).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <unordered_map>
#include <new>
#include <string>
#include <vector>

#include <cub/block/block_scan.cuh>

#include "../../include/hygt_gpu.h"
#include "hygt_kernels.cuh"
#include "hygt_tile.cuh"
#include "hygt_segment.cuh"
#include "hygt_plan.h"
#include "hygt_jit.h"
#include "hygt_gemm.h"
#include "hygt_knobs.h"

using namespace hygt_gpu;
#include "hygt_dispatch.h"
#include "hygt_nvtx.h"

// ============================================================================ errors =====
namespace {
thread_local std::string g_err_msg;
thread_local int g_err_status = 0;

int fail(int status, const std::string& msg) {
  g_err_status = status;
  g_err_msg = msg;
  return status;
}
int ok() {
  g_err_status = 0;
  g_err_msg.clear();
  return HYGT_OK;
}
#define CU(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(HYGT_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
}  // namespace

int hygt_set_error(int status, const char* msg) { return fail(status, msg ? msg : ""); }

extern "C" int hygt_last_error(char* buf, size_t len) {
  if (buf && len) {
    std::strncpy(buf, g_err_msg.c_str(), len - 1);
    buf[len - 1] = 0;
  }
  return g_err_status;
}

// ============================================================================ plan =======
struct hygt_plan {
  int kind = 0;  // 0 float, 1 fixed
  hygt_plan_options opt{};  // resolved creation options (include/hygt_gpu.h)
  double input_limit = 0;   // largest max|x| the plan's arithmetic form keeps finite
  int log2n = 0, rounds = 0, classes = 0, lanes_log2 = 0;
  int algo = 0;  // 0 standard, 1 scale-folded
  uint32_t perm_mask = 0;
  int num_sms = 148;
  uint64_t chunk_rows = 0;  // bucketing locality window (rows); 0 = global
  // float tables per direction (0 = forward, 1 = inverse)
  float2* d_coef[2] = {nullptr, nullptr};
  uint32_t stream_len[2] = {0, 0};
  uint16_t* d_gidx[2] = {nullptr, nullptr};
  uint64_t gmask[2] = {0, 0};
  // fixed point
  int angle_bits = 0, precision_bits = 0;
  uint16_t* d_codes = nullptr;
  int32_t* d_cos = nullptr;
  int32_t* d_sin = nullptr;
  uint16_t* d_fgather[2] = {nullptr, nullptr};  // [C][R+1][N]
  int2* d_ftab[2] = {nullptr, nullptr};          // [C][R*log2N][N/2] (c, s) per pair and step
  // staged fixed-point kernel (N = 16): element-pair (c, s', c, s') units, sort workspace
  bool stagefx = false;
  int4* d_fxtab[2] = {nullptr, nullptr};
  uint16_t* d_fxgt[2] = {nullptr, nullptr};
  uint32_t fx_rows = 0, fx_block_words = 0;
  size_t fx_smem[2] = {0, 0};
  void* d_fx_ws = nullptr;
  size_t fx_ws_bytes = 0;
  // tile path (N <= 32): lane-interleaved tables staged into shared memory by each CTA
  bool tile = false;
  int tile_l = 0, tile_vpt = 1;
  uint32_t tile_rows = 8192;
  float4* d_tcoef[2] = {nullptr, nullptr};
  uint32_t tunits[2] = {0, 0};
  uint4* d_tgidx[2] = {nullptr, nullptr};
  size_t tile_smem[2] = {0, 0};
  // stage path (N = 16): TMA-staged tiles, element-ordered tables
  bool stage = false;
  uint32_t stage_rows = 0, stage_cw = 0, stage_block_words = 0;
  float4* d_scoef[2] = {nullptr, nullptr};
  uint16_t* d_sgtab[2] = {nullptr, nullptr};
  size_t stage_smem[2] = {0, 0};
  // seg2 path (N = 64): thread-per-row over global class buckets, element-ordered tables
  bool seg2 = false;
  size_t seg2_smem[2] = {0, 0};
  // cls path (N = 64): one launch per class, class tables as kernel parameters (hygt_cls.cuh)
  bool cls = false;
  std::vector<unsigned char> cls_blk[2];  // [C] parameter blocks per direction
  unsigned cls_grid = 0;
  int cls_vpt = 2;  // rows per thread
  JitClsKernels cls_jit;  // the same chain with per-class NVRTC kernels (coefficients immediate)
  // JIT path (N <= 64): NVRTC-specialised kernels, coefficients as immediates
  JitKernels jit;
  // segment path (N >= 64): same interleaved tables, one class staged per CTA segment
  bool seg = false;
  int seg_variant = 0;
  size_t seg_smem[2] = {0, 0};
  size_t seg_energy_smem = 0;
  unsigned long long* d_fixed_err = nullptr;
  bool fx_int32 = false;  // fixed point: the int32 kernels are provably safe for this plan
  // fixed point, per-class NVRTC chain (hygt_jit.cpp): kernels and a plan-owned bucket workspace
  JitClsKernels fx_jit;
  void* d_fx_bws = nullptr;
  size_t fx_bws_bytes = 0;
  std::mutex* fixed_mu = nullptr;
  // composed-operator path (N = 64 / 128 / 256): per-class M_c / M_c^T on the tensor cores
  bool gemm = false;
  GemmOperands gemm_ops[2];
};

namespace {

template <class T>
int upload(T** dst, const T* src, size_t n) {
  if (n == 0) {
    *dst = nullptr;
    return HYGT_OK;
  }
  CU(cudaMalloc(reinterpret_cast<void**>(dst), n * sizeof(T)));
  CU(cudaMemcpy(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice));
  return HYGT_OK;
}

void free_plan(hygt_plan* p) {
  if (!p) return;
  for (int d = 0; d < 2; ++d) {
    cudaFree(p->d_coef[d]);
    cudaFree(p->d_gidx[d]);
    cudaFree(p->d_fgather[d]);
    cudaFree(p->d_ftab[d]);
    cudaFree(p->d_fxtab[d]);
    cudaFree(p->d_fxgt[d]);
    cudaFree(p->d_tcoef[d]);
    cudaFree(p->d_tgidx[d]);
    cudaFree(p->d_scoef[d]);
    cudaFree(p->d_sgtab[d]);
  }
  cudaFree(p->d_codes);
  cudaFree(p->d_cos);
  cudaFree(p->d_sin);
  cudaFree(p->d_fixed_err);
  cudaFree(p->d_fx_ws);
  jit_release(p->jit);
  jit_cls_release(p->cls_jit);
  jit_cls_release(p->fx_jit);
  cudaFree(p->d_fx_bws);
  gemm_release(p->gemm_ops[0]);
  gemm_release(p->gemm_ops[1]);
  delete p->fixed_mu;
  delete p;
}

// Options with the defaults filled in; HYGT_ERR_ARGUMENT for malformed ones.
int resolve_options(const hygt_plan_options* in, hygt_plan_options& out) {
  out = hygt_plan_options{};
  out.size = sizeof(hygt_plan_options);
  out.kernel = HYGT_KERNEL_AUTO;
  out.allow_nvrtc = 1;
  out.cta_pairs = 1;
  out.stage_tile_rows = 0;
  if (!in) return HYGT_OK;
  if (in->size < sizeof(uint32_t) || in->size > sizeof(hygt_plan_options))
    return fail(HYGT_ERR_ARGUMENT, "hygt_plan_options: size must be sizeof(hygt_plan_options)");
  hygt_plan_options o = out;
  std::memcpy(&o, in, in->size);
  if (o.kernel < HYGT_KERNEL_AUTO || o.kernel > HYGT_KERNEL_TENSOR)
    return fail(HYGT_ERR_ARGUMENT, "hygt_plan_options: unknown kernel family");
  if (o.allow_nvrtc < 0) o.allow_nvrtc = 1;
  if (o.cta_pairs < 0) o.cta_pairs = 1;
  if (o.stage_tile_rows != 0 && (o.stage_tile_rows < 128 || o.stage_tile_rows > 1016 || o.stage_tile_rows % 8))
    return fail(HYGT_ERR_ARGUMENT, "hygt_plan_options: stage_tile_rows must be a multiple of 8 in [128, 1016]");
  out = o;
  out.size = sizeof(hygt_plan_options);
  return HYGT_OK;
}

int check_perms(int log2n, int rounds, int classes, const uint16_t* perms, uint32_t mask) {
  if (!perms) return HYGT_OK;
  if (rounds > 32) return fail(HYGT_ERR_ARGUMENT, "hygt_plan_create: permutations need rounds <= 32");
  const int n = 1 << log2n;
  std::vector<char> seen(n);
  for (int c = 0; c < classes; ++c)
    for (int r = 0; r < rounds; ++r) {
      if (!((mask >> r) & 1u)) continue;
      std::fill(seen.begin(), seen.end(), 0);
      const uint16_t* p = perms + ((size_t)c * rounds + r) * n;
      for (int i = 0; i < n; ++i) {  // model.hpp:37-44
        if (p[i] >= n || seen[p[i]]) return fail(HYGT_ERR_ARGUMENT, "permutation: not a bijection");
        seen[p[i]] = 1;
      }
    }
  return HYGT_OK;
}

}  // namespace

void hygt_smem_attr(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> set;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  size_t& cur = set[{dev, fn}];
  if (bytes <= cur) return;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess) cur = bytes;
  cudaGetLastError();
}

namespace {
// Development knobs (hygt_knobs.h): the test hook's value, or the measured-best default.
int env_int(const char* name, int dflt) { return knob(name, dflt); }

// Kernels' dynamic shared-memory limits are per function, shared by every plan; plans need
// different sizes, so the attribute only ever grows (a smaller later plan must not shrink it
// under an earlier, larger one).
// The attribute is set per (device, function): a process driving several GPUs sets it on each
// device its plans are created on.
void smem_attr(const void* fn, size_t bytes) { hygt_smem_attr(fn, bytes); }
template <typename F>
void smem_attr(F* fn, size_t bytes) {
  smem_attr(reinterpret_cast<const void*>(fn), bytes);
}

}  // namespace

// ======================================================================= bucketing =======
namespace {

constexpr int BK_THREADS = 1024;
constexpr int BK_PER = 16;
constexpr uint64_t BK_TILE = (uint64_t)BK_THREADS * BK_PER;  // rows per histogram tile

struct WsLayout {
  size_t err = 0, idx = 0, counts = 0, base = 0, seg = 0, total = 0;
  uint64_t tiles = 0, chunks = 0, tiles_per_chunk = 0;
};

WsLayout ws_layout(int classes, uint64_t chunk_rows, uint64_t count) {
  WsLayout w;
  auto al = [](size_t v) { return (v + 255) & ~size_t(255); };
  w.tiles = (count + BK_TILE - 1) / BK_TILE;
  if (w.tiles == 0) w.tiles = 1;
  w.tiles_per_chunk = chunk_rows ? std::max<uint64_t>(1, chunk_rows / BK_TILE) : w.tiles;
  w.chunks = (w.tiles + w.tiles_per_chunk - 1) / w.tiles_per_chunk;
  const size_t cp1 = (size_t)classes + 1;
  w.err = 0;
  w.idx = 256;
  w.counts = al(w.idx + count * sizeof(uint32_t));
  w.base = al(w.counts + w.tiles * cp1 * sizeof(uint32_t));
  w.seg = al(w.base + w.tiles * cp1 * sizeof(uint32_t));
  w.total = al(w.seg + w.chunks * cp1 * sizeof(uint32_t));
  return w;
}

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// Class ids of BK_PER consecutive rows per thread (128-bit loads when aligned).
__device__ __forceinline__ void load_ids16(const uint16_t* __restrict__ cls, uint64_t r0,
                                           uint64_t count, uint32_t (&q)[BK_PER / 2]) {
  if (r0 + BK_PER <= count && (reinterpret_cast<uintptr_t>(cls + r0) & 15) == 0) {
#pragma unroll
    for (int w = 0; w < BK_PER / 8; ++w) {
      const uint4 v = __ldcs(reinterpret_cast<const uint4*>(cls + r0) + w);
      q[4 * w] = v.x; q[4 * w + 1] = v.y; q[4 * w + 2] = v.z; q[4 * w + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int w = 0; w < BK_PER / 2; ++w) q[w] = 0;
    for (int h = 0; h < BK_PER; ++h)
      if (r0 + h < count) q[h >> 1] |= (uint32_t)cls[r0 + h] << (16 * (h & 1));
  }
}

// Per-tile class histogram, written class-major: counts[c * tiles + tile].
__global__ void __launch_bounds__(BK_THREADS) bucket_hist_kernel(const uint16_t* __restrict__ cls,
                                                                 uint64_t count, int classes,
                                                                 uint32_t* counts, uint64_t tiles,
                                                                 uint32_t* err) {
  extern __shared__ uint32_t cnt[];
  for (int i = threadIdx.x; i <= classes; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  const uint64_t r0 = (uint64_t)blockIdx.x * BK_TILE + (uint64_t)threadIdx.x * BK_PER;
  uint32_t q[BK_PER / 2];
  load_ids16(cls, r0, count, q);
  bool bad = false;
#pragma unroll
  for (int h = 0; h < BK_PER; ++h) {
    int c = (q[h >> 1] >> (16 * (h & 1))) & 0xffff;
    if (c >= classes) {
      c = classes;
      bad |= r0 + h < count;
    }
    if (r0 + h < count) atomicAdd(&cnt[c], 1u);
  }
  if (bad) atomicOr(err, 1u);
  __syncthreads();
  for (int i = threadIdx.x; i <= classes; i += blockDim.x) counts[(size_t)i * tiles + blockIdx.x] = cnt[i];
}

// One CTA per chunk: exclusive scan of the chunk's (class, tile) counts in class-major order
// (contiguous in the class-major count layout). Writes per-tile class bases (class-major) and
// the chunk's class run ends.
__global__ void __launch_bounds__(BK_THREADS) bucket_scan_kernel(const uint32_t* counts,
                                                                 uint32_t* base,
                                                                 uint32_t* seg_end,
                                                                 uint64_t tiles,
                                                                 uint64_t tiles_per_chunk,
                                                                 int classes, uint64_t count) {
  using Scan = cub::BlockScan<uint32_t, BK_THREADS>;
  __shared__ typename Scan::TempStorage tmp;
  const uint64_t t0 = (uint64_t)blockIdx.x * tiles_per_chunk;
  const uint64_t tn = umin64(tiles_per_chunk, tiles - t0);
  const uint64_t cp1 = (uint64_t)classes + 1;
  const uint64_t entries = tn * cp1;
  const uint64_t per = (entries + BK_THREADS - 1) / BK_THREADS;
  const uint64_t e0 = umin64(entries, per * threadIdx.x);
  const uint64_t e1 = umin64(entries, e0 + per);
  auto at = [&](uint64_t e) { return (e / tn) * tiles + t0 + (e % tn); };
  uint32_t local = 0;
  for (uint64_t e = e0; e < e1; ++e) local += counts[at(e)];
  uint32_t excl;
  Scan(tmp).ExclusiveSum(local, excl);
  uint32_t run = (uint32_t)umin64(count, t0 * BK_TILE) + excl;
  for (uint64_t e = e0; e < e1; ++e) {
    const uint32_t v = counts[at(e)];
    base[at(e)] = run;
    run += v;
    if (e % tn == tn - 1) seg_end[(uint64_t)blockIdx.x * cp1 + e / tn] = run;
  }
}

// Per tile: local counting sort in shared memory, then each class run of the tile is written
// contiguously to its place in the bucketed index list (coalesced stores).
__global__ void __launch_bounds__(BK_THREADS) bucket_scatter_kernel(
    const uint16_t* __restrict__ cls, uint64_t count, int classes, const uint32_t* base,
    uint64_t tiles, uint32_t* idx) {
  extern __shared__ uint32_t sm_sc[];
  uint32_t* lcnt = sm_sc;                                   // [C+2] local run starts / cursors
  uint32_t* gbase = lcnt + ((classes + 2 + 3) & ~3);        // [C+1] global bases of this tile
  uint32_t* ent = gbase + ((classes + 1 + 3) & ~3);         // [BK_TILE] (class << 16 | row)
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < classes + 2; i += blockDim.x) lcnt[i] = 0;
  for (int i = tid; i <= classes; i += blockDim.x) gbase[i] = base[(size_t)i * tiles + blockIdx.x];
  __syncthreads();
  const uint64_t row0 = (uint64_t)blockIdx.x * BK_TILE;
  const uint64_t r0 = row0 + (uint64_t)tid * BK_PER;
  const int rows = (int)umin64(BK_TILE, count - row0);
  uint32_t q[BK_PER / 2];
  load_ids16(cls, r0, count, q);
#pragma unroll
  for (int h = 0; h < BK_PER; ++h) {
    int c = (q[h >> 1] >> (16 * (h & 1))) & 0xffff;
    c = c < classes ? c : classes;
    if (r0 + h < count) atomicAdd(&lcnt[c + 1], 1u);
  }
  __syncthreads();
  if (tid < 32) {  // exclusive scan of the local counts
    uint32_t carry = 0;
    for (int b = 1; b < classes + 2; b += 32) {
      const int i = b + lane;
      uint32_t v0 = i < classes + 2 ? lcnt[i] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t n = __shfl_up_sync(0xffffffffu, v0, o);
        if (lane >= o) v0 += n;
      }
      if (i < classes + 2) lcnt[i] = v0 + carry;
      carry += __shfl_sync(0xffffffffu, v0, 31);
    }
  }
  __syncthreads();
  // gbase[c] - lcnt[c] turns a local sorted position into the global one
  for (int i = tid; i <= classes; i += blockDim.x) gbase[i] -= lcnt[i];
  __syncthreads();
#pragma unroll
  for (int h = 0; h < BK_PER; ++h) {
    int c = (q[h >> 1] >> (16 * (h & 1))) & 0xffff;
    c = c < classes ? c : classes;
    if (r0 + h < count) {
      const uint32_t lp = atomicAdd(&lcnt[c], 1u);
      ent[lp] = ((uint32_t)c << 16) | (uint32_t)(tid * BK_PER + h);
    }
  }
  __syncthreads();
  for (int j = tid; j < rows; j += blockDim.x) {
    const uint32_t e = ent[j];
    idx[gbase[e >> 16] + j] = (uint32_t)row0 + (e & 0xffffu);
  }
}

__global__ void validate_classes_kernel(const uint16_t* cls, uint64_t count, int classes,
                                        uint32_t* err) {
  bool bad = false;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x)
    bad |= cls[i] >= classes;
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
}

int run_bucket(const hygt_plan* p, int classes, uint64_t chunk_rows, const uint16_t* d_cls,
               uint64_t count, void* d_ws, size_t ws_bytes, cudaStream_t st) {
  const WsLayout w = ws_layout(classes, chunk_rows, count);
  if (!d_ws || ws_bytes < w.total) return fail(HYGT_ERR_ARGUMENT, "hygt_bucket: workspace too small");
  char* ws = static_cast<char*>(d_ws);
  uint32_t* err = reinterpret_cast<uint32_t*>(ws + w.err);
  if (count == 0) return ok();
  if (!d_cls) return ok();
  if (classes == 1) {
    validate_classes_kernel<<<std::min<uint64_t>((count + 255) / 256, (uint64_t)p->num_sms * 8),
                              256, 0, st>>>(d_cls, count, classes, err);
    CU(cudaGetLastError());
    return ok();
  }
  const size_t smem = ((size_t)classes + 1) * sizeof(uint32_t);
  uint32_t* idx = reinterpret_cast<uint32_t*>(ws + w.idx);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(ws + w.counts);
  uint32_t* base = reinterpret_cast<uint32_t*>(ws + w.base);
  uint32_t* seg = reinterpret_cast<uint32_t*>(ws + w.seg);
  bucket_hist_kernel<<<w.tiles, BK_THREADS, smem, st>>>(d_cls, count, classes, cnt, w.tiles, err);
  CU(cudaGetLastError());
  bucket_scan_kernel<<<w.chunks, BK_THREADS, 0, st>>>(cnt, base, seg, w.tiles,
                                                      w.tiles_per_chunk, classes, count);
  CU(cudaGetLastError());
  const size_t smem_sc = (size_t)(((classes + 2 + 3) & ~3) + ((classes + 1 + 3) & ~3)) * 4 + BK_TILE * 4;
  smem_attr(bucket_scatter_kernel, 112 * 1024);  // thread-safe, idempotent
  bucket_scatter_kernel<<<w.tiles, BK_THREADS, smem_sc, st>>>(d_cls, count, classes, base, w.tiles, idx);
  CU(cudaGetLastError());
  return ok();
}

}  // namespace

namespace hygt_gpu {
// Class bucketing for other translation units (the KLT path): workspace size and offsets.
size_t bucket_ws_bytes(int classes, uint64_t chunk_rows, uint64_t count) {
  return ws_layout(classes, chunk_rows, count).total;
}
int bucket_rows(int classes, uint64_t chunk_rows, const uint16_t* d_cls, uint64_t count,
                void* d_ws, size_t ws_bytes, bool run, cudaStream_t st, const uint32_t** idx,
                const uint32_t** seg_end, uint32_t* nseg) {
  const WsLayout w = ws_layout(classes, chunk_rows, count);
  hygt_plan tmp;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&tmp.num_sms, cudaDevAttrMultiProcessorCount, dev);
  if (run) {
    const int s = run_bucket(&tmp, classes, chunk_rows, d_cls, count, d_ws, ws_bytes, st);
    if (s) return s;
  }
  char* ws = static_cast<char*>(d_ws);
  *idx = reinterpret_cast<const uint32_t*>(ws + w.idx);
  *seg_end = reinterpret_cast<const uint32_t*>(ws + w.seg);
  *nseg = (uint32_t)(w.chunks * (classes + 1));
  return HYGT_OK;
}
}  // namespace hygt_gpu

// ======================================================================= dispatch ========
namespace {

constexpr int APPLY_THREADS = 256;

size_t apply_smem(const hygt_plan* p, int dir) {
  if (!p->gmask[dir]) return 0;
  return (size_t)(APPLY_THREADS / 32) * 32 * (1u << p->log2n) / (1u << p->lanes_log2) * sizeof(float);
}


// ---- tile path --------------------------------------------------------------------------
void default_tile_layout(int log2n, int* l, int* vpt) {
  switch (log2n) {
    case 2: *l = 0; *vpt = 2; break;
    case 3: *l = 1; *vpt = 2; break;
    case 4: *l = 1; *vpt = 2; break;
    case 5: *l = 2; *vpt = 2; break;
    default: *l = -1; *vpt = 0;
  }
}

int tile_scratch_floats(int log2n, int l, int vpt) {
  const int n = 1 << log2n, tpv = 1 << l, v = 32 / tpv, rows = v * vpt;
  const int want = (v / 4) % 8;
  return n * (rows + ((want - rows % 8) % 8 + 8) % 8);
}

int run_tile(const hygt_plan* p, int dir, const float* x, float* y, const uint16_t* d_cls,
             uint64_t count, double* energy, uint32_t* err, cudaStream_t st) {
  TileFn fn = select_tile(p->log2n, p->tile_l, p->tile_vpt, p->algo == 0, dir == 0, energy != nullptr);
  if (!fn) return fail(HYGT_ERR_ARGUMENT, "hygt: no tile kernel for this layout");
  TileParams P{};
  P.x = x;
  P.y = y;
  P.cls = d_cls;
  P.count = count;
  P.classes = p->classes;
  P.rounds = p->rounds;
  P.coef = p->d_tcoef[dir];
  P.units = p->tunits[dir];
  P.gidx = p->d_tgidx[dir];
  P.gmask = p->gmask[dir];
  P.tile_rows = p->tile_rows;
  P.energy = energy;
  P.err = err;
  P.load_policy = env_int("HYGT_LOAD_POLICY", 1);
  int occ = 0;
  const int tthreads = p->tile_vpt >= 8 ? 256 : TILE_THREADS;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, tthreads, p->tile_smem[dir]));
  if (occ < 1) return fail(HYGT_ERR_CUDA, "hygt: tile kernel does not fit on an SM");
  const uint64_t tiles = (count + p->tile_rows - 1) / p->tile_rows;
  const uint64_t ctas = std::min<uint64_t>(tiles, (uint64_t)p->num_sms * occ);
  fn<<<(unsigned)ctas, tthreads, p->tile_smem[dir], st>>>(P);
  CU(cudaGetLastError());
  return ok();
}

// Lane-interleaved tables of layout (l, vpt) for both directions: coefficient float4 units
// [C][units][TPV] and gather words [C][R+1][words][TPV] holding byte offsets into the
// permutation scratch (stride from the layout). Returns the per-class table bytes.
int build_interleaved(hygt_plan* p, const double* angles, const uint16_t* perms, int l, int vpt,
                      size_t* coef_bytes_per_class, size_t* gidx_bytes_per_class) {
  const Layout ly{p->log2n, l};
  const int tpv = ly.tpv(), e = ly.e();
  for (int d = 0; d < 2; ++d) {
    DirTables t;
    if (!build_direction(ly, p->rounds, p->classes, angles, perms, p->perm_mask, d == 0, p->algo == 0, t))
      return fail(HYGT_ERR_NUMERICAL, "hygt: table build failed");
    const uint32_t units = t.stream_len / 2;
    std::vector<float4> il((size_t)p->classes * units * tpv);
    for (int c = 0; c < p->classes; ++c)
      for (int lt = 0; lt < tpv; ++lt)
        for (uint32_t u = 0; u < units; ++u) {
          const Float2* w = &t.coef[((size_t)c * tpv + lt) * t.stream_len + 2 * u];
          il[((size_t)c * units + u) * tpv + lt] = make_float4(w[0].x, w[0].y, w[1].x, w[1].y);
        }
    const int words = (e + 7) / 8;
    const uint32_t stride_bytes = 4u * (uint32_t)(tile_scratch_floats(p->log2n, l, vpt) >> p->log2n);
    std::vector<uint4> gi;
    if (t.gmask) {
      gi.assign((size_t)p->classes * (p->rounds + 1) * words * tpv, make_uint4(0, 0, 0, 0));
      for (int c = 0; c < p->classes; ++c)
        for (int k = 0; k <= p->rounds; ++k)
          for (int lt = 0; lt < tpv; ++lt) {
            const uint16_t* src = &t.gidx[(((size_t)c * (p->rounds + 1) + k) * tpv + lt) * e];
            for (int w = 0; w < words; ++w) {
              uint32_t q[4] = {0, 0, 0, 0};
              for (int h = 0; h < 8 && 8 * w + h < e; ++h)  // byte offsets into the scratch
                q[h / 2] |= (uint32_t)(src[8 * w + h] * stride_bytes) << (16 * (h & 1));
              gi[(((size_t)c * (p->rounds + 1) + k) * words + w) * tpv + lt] = make_uint4(q[0], q[1], q[2], q[3]);
            }
          }
    }
    if ((size_t)tile_scratch_floats(p->log2n, l, vpt) * 4 > 65535)
      return fail(HYGT_ERR_ARGUMENT, "hygt: permutation scratch exceeds 16-bit offsets");
    int s = upload(&p->d_tcoef[d], il.data(), il.size());
    if (!s && !gi.empty()) s = upload(&p->d_tgidx[d], gi.data(), gi.size());
    if (s) return s;
    p->tunits[d] = units;
    coef_bytes_per_class[d] = (size_t)units * tpv * sizeof(float4);
    gidx_bytes_per_class[d] = gi.empty() ? 0 : (size_t)(p->rounds + 1) * words * tpv * sizeof(uint4);
  }
  return HYGT_OK;
}

int setup_tile(hygt_plan* p, const double* angles, const uint16_t* perms) {
  int l = -1, vpt = 0;
  default_tile_layout(p->log2n, &l, &vpt);
  const int el = env_int("HYGT_TILE_L", -1), ev = env_int("HYGT_TILE_VPT", -1);
  if (el >= 0 && ev > 0 && select_tile(p->log2n, el, ev, false, true, false)) {
    l = el;
    vpt = ev;
  }
  if (l < 0 || env_int("HYGT_TILE", 1) == 0) return HYGT_OK;
  const int tthreads = vpt >= 8 ? 256 : TILE_THREADS;
  const int rows = (vpt >= 8 ? 16 : 8) * tthreads;  // the tile sort loads 8 or 16 ids per thread
  size_t cb[2], gb[2];
  const int vpt_real = vpt >= 8 ? vpt - 8 : vpt;
  if (int s = build_interleaved(p, angles, perms, l, vpt_real, cb, gb)) return s;
  size_t smem_max = 0;
  for (int d = 0; d < 2; ++d) {
    p->tile_smem[d] = tile_smem_bytes(cb[d] * p->classes, gb[d] * p->classes, p->classes, rows,
                                      tthreads / 32, tile_scratch_floats(p->log2n, l, vpt_real));
    smem_max = std::max(smem_max, p->tile_smem[d]);
  }
  if (smem_max > 200 * 1024) return HYGT_OK;  // tables too large: stay on another path
  for (int d = 0; d < 2; ++d)
    for (int en = 0; en < 2; ++en) {
      TileFn fn = select_tile(p->log2n, l, vpt, p->algo == 0, d == 0, en == 1);
      if (fn) smem_attr(fn, (int)p->tile_smem[d]);
    }
  cudaGetLastError();  // no sticky error from the attribute calls
  p->tile = true;
  p->tile_l = l;
  p->tile_vpt = vpt;
  p->tile_rows = (uint32_t)rows;
  return HYGT_OK;
}

// ---- stage path (hygt_stage.cuh) ----------------------------------------------------------
unsigned long long* g_stage_trace = nullptr;  // debug hook, see hygt_debug_stage_trace
// Element-ordered tables: per class, per execution step (round, pass) N/4 float4 units of the
// per-element coefficient k_i of y_i = x_i + k_i x_{i^2^p} (scale-folded: k_m = t1, k_n = -t2;
// standard: N/4 units of c_i then N/4 units of s'_i with s'_m = s, s'_n = -s), then N/4 units of
// final scales (scale-folded only). Gathers: [C][R+1][N] u16 scratch offsets src * 128.
// Element-ordered tables of both directions into p->d_scoef / p->d_sgtab (stage and seg2 paths).
// Host copies of one direction's element tables: coef [C][cw] float4, gt [C][gs] u16 with
// gs = stage_gstride / 2 (gather offsets src * 128 per step).
int elem_tables_host(hygt_plan* p, const double* angles, const uint16_t* perms, int d,
                     std::vector<float4>& coef, std::vector<uint16_t>& gt, uint32_t* cw_out) {
  const int n = 1 << p->log2n, nc = n / 4, C = p->classes, R = p->rounds;
  const bool standard = p->algo == 0;
  const uint32_t step_units = (uint32_t)nc * (standard ? 2 : 1);
  const uint32_t cw = (uint32_t)R * p->log2n * step_units + (standard ? 0u : (uint32_t)nc);
  {
    std::vector<ClassProgram> progs;
    if (!build_programs(p->log2n, R, C, angles, perms, p->perm_mask, d == 0, standard, progs))
      return fail(HYGT_ERR_NUMERICAL, "hygt: element table build failed");
    coef.assign((size_t)C * cw, make_float4(0.f, 0.f, 0.f, 0.f));
    const uint32_t gs = stage_gstride(p->log2n, R) / 2;  // u16 per class
    gt.assign((size_t)C * gs, 0);
    std::vector<float> kc(n), ks(n);
    for (int c = 0; c < C; ++c) {
      float4* cc = &coef[(size_t)c * cw];
      uint32_t step = 0;
      int in_pass = 0;
      for (const ProgOp& op : progs[c].ops) {
        if (op.kind == 0) {
          if (standard) {
            kc[op.m] = kc[op.n] = op.a;
            ks[op.m] = op.b;
            ks[op.n] = -op.b;
          } else {
            kc[op.m] = op.a;
            kc[op.n] = op.b;  // build_programs stores -k2 for the n side
          }
          if (++in_pass == n / 2) {
            for (int u = 0; u < nc; ++u) {
              cc[step * step_units + u] = make_float4(kc[4 * u], kc[4 * u + 1], kc[4 * u + 2], kc[4 * u + 3]);
              if (standard)
                cc[step * step_units + nc + u] =
                    make_float4(ks[4 * u], ks[4 * u + 1], ks[4 * u + 2], ks[4 * u + 3]);
            }
            ++step;
            in_pass = 0;
          }
        } else if (op.kind == 2) {
          const std::vector<float>& sc = progs[c].scales;
          for (int u = 0; u < nc; ++u)
            cc[(size_t)R * p->log2n * step_units + u] = make_float4(sc[4 * u], sc[4 * u + 1], sc[4 * u + 2], sc[4 * u + 3]);
        }
      }
      if (step != (uint32_t)R * p->log2n) return fail(HYGT_ERR_NUMERICAL, "hygt: element table step count");
      uint64_t gm = 0;
      const auto g = exec_gathers(p->log2n, R, perms ? perms + (size_t)c * R * n : nullptr,
                                  p->perm_mask, d == 0, &gm);
      for (int k = 0; k <= R; ++k)
        for (size_t i = 0; i < g[k].size(); ++i)
          gt[(size_t)c * gs + (size_t)k * n + i] = (uint16_t)(g[k][i] * 128);
    }
  }
  *cw_out = cw;
  return HYGT_OK;
}

int build_elem_tables(hygt_plan* p, const double* angles, const uint16_t* perms, uint32_t* cw_out) {
  for (int d = 0; d < 2; ++d) {
    std::vector<float4> coef;
    std::vector<uint16_t> gt;
    if (int s = elem_tables_host(p, angles, perms, d, coef, gt, cw_out)) return s;
    int s = upload(&p->d_scoef[d], coef.data(), coef.size());
    if (!s && p->gmask[d]) s = upload(&p->d_sgtab[d], gt.data(), gt.size());
    if (s) return s;
  }
  return HYGT_OK;
}

int setup_stage(hygt_plan* p, const double* angles, const uint16_t* perms) {
  StageFn probe = select_stage(p->log2n, p->algo == 0, true);
  if (!probe || env_int("HYGT_STAGE", 1) == 0 || p->classes > STAGE_MAX_CLASSES) return HYGT_OK;
  const int C = p->classes, R = p->rounds;
  const bool standard = p->algo == 0;
  uint32_t cw = 0;
  if (int s = build_elem_tables(p, angles, perms, &cw)) return s;
  // Tile rows: one batch of 32 * VPT sorted positions per consumer warp, including the padding
  // of every class run to VPT; rows are indexed with 10 bits in the sort entries.
  const long long tenv = p->opt.stage_tile_rows > 0 ? p->opt.stage_tile_rows : env_int("HYGT_STAGE_ROWS", -1);
  uint32_t T = (uint32_t)std::max(0, STAGE_WARPS * 32 * STAGE_VPT - (STAGE_VPT - 1) * C);
  if (tenv > 0) T = (uint32_t)tenv;
  T = std::min<uint32_t>(T, 1016) / 8 * 8;
  size_t smem[2] = {0, 0};
  for (; T >= 128; T -= 8) {
    for (int d = 0; d < 2; ++d)
      smem[d] = stage_smem_layout(p->log2n, STAGE_VPT, STAGE_WARPS, C, cw, R, T, p->gmask[d] != 0).total;
    if (std::max(smem[0], smem[1]) <= 227 * 1024) break;
  }
  if (T < 128) return HYGT_OK;  // tables too large for the staged layout
  for (int d = 0; d < 2; ++d) {
    smem_attr(select_stage(p->log2n, standard, d == 0), (int)smem[d]);
    p->stage_smem[d] = smem[d];
  }
  cudaGetLastError();
  p->stage = true;
  p->stage_rows = T;
  p->stage_cw = cw;
  p->stage_block_words = stage_block_words(T, STAGE_VPT, C);
  for (uint32_t t : {7u * 128u, 8u * 128u})
    smem_attr(select_stage_sort(STAGE_VPT, t), (int)(STAGE_SORT_WARPS * stage_sort_warp_bytes(C, p->stage_block_words)));
  cudaGetLastError();
  return HYGT_OK;
}

// Workspace of the stage path: error word, then one sorted entry block per tile.
size_t stage_ws_bytes(const hygt_plan* p, uint64_t count) {
  const uint64_t tiles = (count + p->stage_rows - 1) / p->stage_rows;
  return 256 + tiles * p->stage_block_words * 2;
}

// Per-tile class sort of the staged kernels into d_ws (error word, then one entry block per tile).
int stage_sort(int classes, uint32_t T, uint32_t block_words, int vpt, int num_sms, const uint16_t* d_cls,
               uint64_t count, void* d_ws, cudaStream_t st) {
  if (count == 0) return ok();
  StageSortParams S{};
  S.cls = d_cls;
  S.count = count;
  S.classes = classes;
  S.tile_rows = T;
  S.block_words = block_words;
  S.ent = reinterpret_cast<uint16_t*>(static_cast<char*>(d_ws) + 256);
  S.err = static_cast<uint32_t*>(d_ws);
  const uint64_t tiles = (count + T - 1) / T;
  StageSortFn fn = select_stage_sort(vpt, T);
  const size_t smem = (size_t)STAGE_SORT_WARPS * stage_sort_warp_bytes(classes, block_words);
  if (smem > 48 * 1024) smem_attr(fn, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 32 * STAGE_SORT_WARPS, smem);
  if (occ < 1) occ = 1;
  const uint64_t ctas = std::min<uint64_t>((tiles + STAGE_SORT_WARPS - 1) / STAGE_SORT_WARPS, (uint64_t)num_sms * occ);
  fn<<<(unsigned)ctas, 32 * STAGE_SORT_WARPS, smem, st>>>(S);
  CU(cudaGetLastError());
  return ok();
}

int run_stage_sort(const hygt_plan* p, const uint16_t* d_cls, uint64_t count, void* d_ws,
                   size_t ws_bytes, cudaStream_t st) {
  if (!d_ws || ws_bytes < stage_ws_bytes(p, count)) return fail(HYGT_ERR_ARGUMENT, "hygt: workspace too small");
  return stage_sort(p->classes, p->stage_rows, p->stage_block_words, STAGE_VPT, p->num_sms, d_cls, count, d_ws, st);
}

bool stage_usable(const hygt_plan* p, const float* x, const float* y, const double* energy) {
  (void)x; (void)y;
  return p->stage && !energy;  // run_apply has checked the 16 B row alignment
}

int run_stage(const hygt_plan* p, int dir, const float* x, float* y, const uint16_t* d_cls,
              uint64_t count, void* d_ws, size_t ws_bytes, uint32_t flags, cudaStream_t st) {
  const bool sorted = d_cls && p->classes > 1;
  if (sorted && !(flags & HYGT_REUSE_BUCKETS))
    if (int s = run_stage_sort(p, d_cls, count, d_ws, ws_bytes, st)) return s;
  if (sorted && (!d_ws || ws_bytes < stage_ws_bytes(p, count)))
    return fail(HYGT_ERR_ARGUMENT, "hygt: workspace too small");
  // The debug build (trace hook set) is a separate instantiation with the same smem layout.
  StageFn fn = select_stage(p->log2n, p->algo == 0, dir == 0, g_stage_trace != nullptr);
  if (g_stage_trace) smem_attr(fn, (int)p->stage_smem[dir]);
  StageParams P{};
  P.x = x;
  P.y = y;
  P.count = count;
  P.classes = p->classes;
  P.rounds = p->rounds;
  P.coef = p->d_scoef[dir];
  P.cw = p->stage_cw;
  P.gtab = p->d_sgtab[dir];
  P.gmask = p->gmask[dir];
  P.tile_rows = p->stage_rows;
  P.ent = sorted ? reinterpret_cast<const uint16_t*>(static_cast<const char*>(d_ws) + 256) : nullptr;
  P.block_words = p->stage_block_words;
  if (!sorted && d_cls) {  // one class: the kernel validates the ids itself (ResidualDataset)
    if (!d_ws || ws_bytes < 256) return fail(HYGT_ERR_ARGUMENT, "hygt: workspace too small");
    P.cls = d_cls;
    P.err = static_cast<uint32_t*>(d_ws);
  }
  P.trace = g_stage_trace;
  P.debug_skip = g_stage_trace ? (uint32_t)env_int("HYGT_STAGE_DEBUG_SKIP", 0) : 0u;
  const uint64_t tiles = (count + p->stage_rows - 1) / p->stage_rows;
  const uint64_t ctas = std::min<uint64_t>(tiles, (uint64_t)p->num_sms);
  fn<<<(unsigned)ctas, (STAGE_WARPS + 1) * 32, p->stage_smem[dir], st>>>(P);
  CU(cudaGetLastError());
  return ok();
}

// ---- segment path -----------------------------------------------------------------------

struct SegVariant {
  int log2n, l, vpt;
  bool prefetch;
};
// Instantiated segment layouts; the first of each N is the default.
constexpr SegVariant kSegVariants[] = {
    {6, 1, 1, true}, {6, 1, 2, false}, {6, 2, 2, true}, {6, 0, 1, false},
    {7, 2, 1, true}, {7, 2, 2, false},
    {8, 2, 1, false}, {8, 2, 1, true}, {8, 1, 1, false}, {8, 3, 2, false}, {8, 2, 2, false},
};
// default variant per log2 N (measured on B200): N=64 -> (L=1, VPT=2),
// N=128 -> (L=2, VPT=1, prefetch), N=256 -> (L=2, VPT=2) (36.6% vs 35.7% for (L=1, VPT=1))
int default_seg_variant(int log2n) { return log2n == 6 ? 1 : log2n == 7 ? 4 : log2n == 8 ? 10 : -1; }

int setup_segment(hygt_plan* p, const double* angles, const uint16_t* perms) {
  if (p->tile || env_int("HYGT_SEGMENT", 1) == 0) return HYGT_OK;
  int variant = default_seg_variant(p->log2n);
  const int want = env_int("HYGT_SEG_VARIANT", -1);
  if (want >= 0 && want < (int)(sizeof(kSegVariants) / sizeof(kSegVariants[0])) &&
      kSegVariants[want].log2n == p->log2n)
    variant = want;
  if (variant < 0) return HYGT_OK;
  const SegVariant sv = kSegVariants[variant];
  size_t cb[2], gb[2];
  if (int s = build_interleaved(p, angles, perms, sv.l, sv.vpt, cb, gb)) return s;
  for (int d = 0; d < 2; ++d) {
    // the permutation scratch exists only when the plan has permutations
    p->seg_smem[d] = cb[d] + gb[d] +
                     (p->gmask[d] ? (size_t)(SEG_THREADS / 32) * tile_scratch_floats(p->log2n, sv.l, sv.vpt) * 4 : 0);
    if (d == 0)  // fused energy: per-warp fp64 partial sums [E][32] (seg_energy_smem)
      p->seg_energy_smem = (p->seg_smem[0] + 7) / 8 * 8 + (size_t)(SEG_THREADS / 32) * ((1u << p->log2n) >> sv.l) * 32 * 8;
    if (p->seg_smem[d] > 220 * 1024) return HYGT_OK;
    SegFn fn = select_seg(variant, p->algo == 0, d == 0, false);
    if (fn) smem_attr(fn, (int)p->seg_smem[d]);
  }
  // fused energy (forward only): its per-warp partial sums must fit next to the tables
  if (p->seg_energy_smem <= 227 * 1024) {
    SegFn fe = select_seg(variant, p->algo == 0, true, true);
    if (fe) smem_attr(fe, (int)p->seg_energy_smem);
  } else {
    p->seg_energy_smem = 0;  // energy requests use the bucketed apply kernel instead
  }
  cudaGetLastError();  // attribute calls must not leave a sticky error for the next launch check
  p->seg = true;
  p->seg_variant = variant;
  p->chunk_rows = 0;  // global class buckets
  return HYGT_OK;
}

int setup_seg2(hygt_plan* p, const double* angles, const uint16_t* perms) {
  if (!select_seg2(p->log2n, p->algo == 0, true) || env_int("HYGT_SEG2", 1) == 0) return HYGT_OK;
  uint32_t cw = 0;
  if (int s = build_elem_tables(p, angles, perms, &cw)) return s;
  for (int d = 0; d < 2; ++d) {
    p->seg2_smem[d] = seg2_smem_bytes(p->log2n, SEG2_VPT, SEG2_WARPS, cw, stage_gstride(p->log2n, p->rounds));
    if (p->seg2_smem[d] > 227 * 1024) return HYGT_OK;
    smem_attr(select_seg2(p->log2n, p->algo == 0, d == 0), (int)p->seg2_smem[d]);
  }
  cudaGetLastError();
  p->stage_cw = cw;
  p->seg2 = true;
  p->chunk_rows = 0;  // global class buckets
  return HYGT_OK;
}

// ---- cls path (hygt_cls.cuh) ----------------------------------------------------------------
int setup_cls(hygt_plan* p, const double* angles, const uint16_t* perms) {
  if (p->algo == 1 && !p->jit.ok && jit_cls_supported(p->log2n, p->classes, p->rounds) &&
      p->opt.allow_nvrtc && env_int("HYGT_CLS_JIT", 1) != 0) {
    std::string err;
    if (jit_cls_build(p->log2n, p->rounds, p->classes, angles, perms, p->perm_mask, false, p->cls_jit, err)) {
      jit_cls_release(p->cls_jit);  // stay on the precompiled kernels
      if (env_int("HYGT_JIT_REQUIRED", 0)) return fail(HYGT_ERR_CUDA, err);
    } else {
      p->cls = true;
      p->chunk_rows = 0;  // global class buckets
      return HYGT_OK;
    }
  }
  const size_t bytes = cls_param_bytes(p->log2n, p->rounds);
  if (!bytes || p->algo != 1 || p->classes < 2 || env_int("HYGT_CLS", 1) == 0) return HYGT_OK;
  const int C = p->classes;
  const uint32_t gs = stage_gstride(p->log2n, p->rounds) / 2;
  for (int d = 0; d < 2; ++d) {
    std::vector<float4> coef;
    std::vector<uint16_t> gt;
    uint32_t cw = 0;
    if (int s = elem_tables_host(p, angles, perms, d, coef, gt, &cw)) return s;
    p->cls_blk[d].assign((size_t)C * bytes, 0);
    for (int c = 0; c < C; ++c)
      cls_fill(p->log2n, p->rounds, p->cls_blk[d].data() + (size_t)c * bytes, &coef[(size_t)c * cw], cw,
               &gt[(size_t)c * gs], (uint32_t)p->gmask[d]);
  }
  p->cls_vpt = env_int("HYGT_CLS_VPT", 1) == 2 ? 2 : 1;
  for (int d = 0; d < 2; ++d)
    smem_attr(cls_kernel(p->log2n, p->rounds, d == 0, p->cls_vpt), cls_smem_bytes(p->log2n, p->cls_vpt));
  cudaGetLastError();
  int occ = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, cls_kernel(p->log2n, p->rounds, true, p->cls_vpt), 32,
                                                   cls_smem_bytes(p->log2n, p->cls_vpt)));
  if (occ < 1) return HYGT_OK;
  // grids of a fraction of the SMs' warp slots: each warp takes several batches (its next
  // batch's rows prefetched), and the PDL chain keeps grids of several classes in flight
  const int div = std::max(1, env_int("HYGT_CLS_GRID_DIV", 1));
  p->cls_grid = (unsigned)std::max(1, p->num_sms * occ / div);
  p->cls = true;
  p->chunk_rows = 0;  // global class buckets
  return HYGT_OK;
}

int run_cls(const hygt_plan* p, int dir, const float* x, float* y, const WsLayout& w, char* ws,
            cudaStream_t st) {
  if (p->cls_jit.ok) {
    if (jit_cls_launch(p->cls_jit, dir, x, y, reinterpret_cast<const uint32_t*>(ws + w.idx),
                       reinterpret_cast<const uint32_t*>(ws + w.seg), p->classes, st))
      return fail(HYGT_ERR_CUDA, std::string("hygt: class launch failed: ") + cudaGetErrorString(cudaGetLastError()));
    return ok();
  }
  const cudaError_t e = cls_launch_chain(p->log2n, p->rounds, dir == 0, p->cls_blk[dir].data(), p->classes, x, y,
                                         reinterpret_cast<const uint32_t*>(ws + w.idx),
                                         reinterpret_cast<const uint32_t*>(ws + w.seg), p->cls_grid, p->cls_vpt, st);
  if (e != cudaSuccess) return fail(HYGT_ERR_CUDA, std::string("hygt: class launch failed: ") + cudaGetErrorString(e));
  return ok();
}

int run_seg2(const hygt_plan* p, int dir, const float* x, float* y, uint64_t count,
             const WsLayout& w, char* ws, cudaStream_t st) {
  Seg2Fn fn = select_seg2(p->log2n, p->algo == 0, dir == 0);
  Seg2Params P{};
  P.x = x;
  P.y = y;
  P.idx = reinterpret_cast<const uint32_t*>(ws + w.idx);
  P.seg_end = reinterpret_cast<const uint32_t*>(ws + w.seg);
  P.classes = p->classes;
  P.rounds = p->rounds;
  P.count = count;
  P.coef = p->d_scoef[dir];
  P.cw = p->stage_cw;
  P.gtab = p->d_sgtab[dir];
  P.gstride = stage_gstride(p->log2n, p->rounds);
  P.gmask = p->gmask[dir];
  const uint64_t min_span = 4096;
  uint64_t ctas = std::min<uint64_t>((uint64_t)p->num_sms, (count + min_span - 1) / min_span);
  if (ctas < 1) ctas = 1;
  P.cta_span = (count + ctas - 1) / ctas;
  fn<<<(unsigned)ctas, SEG2_WARPS * 32, p->seg2_smem[dir], st>>>(P);
  CU(cudaGetLastError());
  return ok();
}

int run_segment(const hygt_plan* p, int dir, const float* x, float* y, uint64_t count,
                double* energy, const WsLayout& w, char* ws, bool bucketed, cudaStream_t st) {
  SegFn fn = select_seg(p->seg_variant, p->algo == 0, dir == 0, energy != nullptr);
  SegParams P{};
  P.x = x;
  P.y = y;
  P.idx = reinterpret_cast<const uint32_t*>(ws + w.idx);
  P.seg_end = reinterpret_cast<const uint32_t*>(ws + w.seg);
  P.classes = p->classes;
  P.rounds = p->rounds;
  P.count = count;
  P.coef = p->d_tcoef[dir];
  P.units = p->tunits[dir];
  P.gidx = p->d_tgidx[dir];
  P.gmask = p->gmask[dir];
  P.energy = energy;
  (void)bucketed;
  const size_t smem = energy ? p->seg_energy_smem : p->seg_smem[dir];
  int occ = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, SEG_THREADS, smem));
  if (occ < 1) return fail(HYGT_ERR_CUDA, "hygt: segment kernel does not fit on an SM");
  const uint64_t ctas_max = (uint64_t)p->num_sms * occ;
  const uint64_t min_span = 2048;
  uint64_t ctas = std::min<uint64_t>(ctas_max, (count + min_span - 1) / min_span);
  if (ctas < 1) ctas = 1;
  P.cta_span = (count + ctas - 1) / ctas;
  fn<<<(unsigned)ctas, SEG_THREADS, smem, st>>>(P);
  CU(cudaGetLastError());
  return ok();
}

// Composed-operator path: M_c (forward) and M_c^T (inverse) per class, fp64 on the host, then
// the fp16 hi/lo operand stages of hygt_gemm.cu. Default for N = 128 / 256, where the butterfly
// kernels are bound by coefficient delivery through the LSU (measured at N = 128,
// 35 classes, R = 4: 27 % of HBM against 59 %); HYGT_GEMM=1 takes it at N = 64 as well (the
// per-class NVRTC chain is faster there), HYGT_GEMM=0 never.
int setup_gemm(hygt_plan* p, const double* angles, const uint16_t* perms) {
  const int n = 1 << p->log2n;
  if (!gemm_supported(n, p->classes)) {
    if (p->opt.kernel == HYGT_KERNEL_TENSOR)
      return fail(HYGT_ERR_ARGUMENT, "hygt_plan_create: the tensor-core path needs N in {64, 128, 256} and <= 512 classes");
    return HYGT_OK;
  }
  const int want = p->opt.kernel == HYGT_KERNEL_TENSOR ? 1 : p->opt.kernel == HYGT_KERNEL_BUTTERFLY ? 0
                                                                                  : env_int("HYGT_GEMM", -1);
  if (want == 0 || (want < 0 && n < 128)) return HYGT_OK;
  const size_t a = (size_t)p->rounds * p->log2n * n / 2;
  std::vector<double> fwd((size_t)p->classes * n * n), inv((size_t)p->classes * n * n);
  for (int c = 0; c < p->classes; ++c) {
    double* m = &fwd[(size_t)c * n * n];
    compose_operator(p->log2n, p->rounds, angles + (size_t)c * a,
                     perms ? perms + (size_t)c * p->rounds * n : nullptr, p->perm_mask, m);
    double* t = &inv[(size_t)c * n * n];
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < n; ++k) t[(size_t)i * n + k] = m[(size_t)k * n + i];
  }
  if (int s = gemm_build(n, p->classes, fwd.data(), p->gemm_ops[0])) return s;
  if (int s = gemm_build(n, p->classes, inv.data(), p->gemm_ops[1])) return s;
  for (int d = 0; d < 2; ++d) {
    p->gemm_ops[d].pair = p->opt.cta_pairs != 0 && env_int("HYGT_GEMM_PAIR", 1) != 0;
    p->gemm_ops[d].wide = env_int("HYGT_GEMM_WIDE", 1) != 0;  // merged accumulator, one unit per tile
    p->gemm_ops[d].ts = env_int("HYGT_GEMM_TS", 1) != 0;      // N = 256: operator in TMEM
    p->gemm_ops[d].dbg = env_int("HYGT_GEMM_DBG", 0);  // diagnostics only (hygt_gemm.h)
  }
  p->gemm = true;
  p->chunk_rows = 0;  // global class buckets
  return HYGT_OK;
}

int run_apply(const hygt_plan* p, int dir, const float* x, float* y, const uint16_t* d_cls,
              uint64_t count, double* energy, void* d_ws, size_t ws_bytes, uint32_t flags,
              cudaStream_t st) {
  if (!p || p->kind != 0) return fail(HYGT_ERR_ARGUMENT, "hygt: not a float plan");
  if (count == 0) return ok();
  if (!x || !y) return fail(HYGT_ERR_ARGUMENT, "hygt: null data pointer");
  if (count > 0xFFFFFFFFull) return fail(HYGT_ERR_ARGUMENT, "hygt: at most 2^32-1 rows per call");
  {  // rows are moved in chunks of min(4, N) floats
    const uintptr_t al = (uintptr_t)4 << (p->log2n < 2 ? p->log2n : 2);
    if (((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & (al - 1)) != 0)
      return fail(HYGT_ERR_ARGUMENT, "hygt: x and y must be aligned to min(16, 4N) bytes");
  }
  const WsLayout w = ws_layout(p->classes, p->chunk_rows, count);
  if (p->gemm) {
    if (((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) != 0)
      return fail(HYGT_ERR_ARGUMENT, "hygt: x and y must be aligned to 16 bytes");
    const bool bk = d_cls && p->classes > 1;
    if (bk) {
      if (!d_ws || ws_bytes < w.total) return fail(HYGT_ERR_ARGUMENT, "hygt: workspace too small");
      if (!(flags & HYGT_REUSE_BUCKETS)) {
        const int s = run_bucket(p, p->classes, 0, d_cls, count, d_ws, ws_bytes, st);
        if (s) return s;
      }
    }
    const char* ws = static_cast<const char*>(d_ws);
    return gemm_run(p->gemm_ops[dir], x, y, bk ? reinterpret_cast<const uint32_t*>(ws + w.idx) : nullptr,
                    bk ? reinterpret_cast<const uint32_t*>(ws + w.seg) : nullptr, count, energy, st);
  }
  if (p->jit.ok && !energy) {
    const bool bk = d_cls && p->classes > 1;
    if (d_cls) {
      if (!d_ws || ws_bytes < w.total) return fail(HYGT_ERR_ARGUMENT, "hygt: workspace too small");
      if (!(flags & HYGT_REUSE_BUCKETS)) {
        const int s = run_bucket(p, p->classes, p->chunk_rows, d_cls, count, d_ws, ws_bytes, st);
        if (s) return s;
      }
    }
    char* ws = static_cast<char*>(d_ws);
    if (jit_launch(p->jit, dir, x, y, bk ? reinterpret_cast<const uint32_t*>(ws + w.idx) : nullptr,
                   bk ? reinterpret_cast<const uint32_t*>(ws + w.seg) : nullptr,
                   bk ? (uint32_t)(w.chunks * (p->classes + 1)) : 0u, count, p->classes,
                   p->num_sms, st))
      return fail(HYGT_ERR_CUDA, std::string("hygt: jit launch failed: ") + cudaGetErrorString(cudaGetLastError()));
    return ok();
  }
  if (stage_usable(p, x, y, energy)) return run_stage(p, dir, x, y, d_cls, count, d_ws, ws_bytes, flags, st);
  const bool bucketed = d_cls && p->classes > 1;
  // per-class launch chain (N = 32 / 64)
  if (p->cls && bucketed && !energy) {
    if (!d_ws || ws_bytes < w.total) return fail(HYGT_ERR_ARGUMENT, "hygt: workspace too small");
    if (!(flags & HYGT_REUSE_BUCKETS)) {
      const int s = run_bucket(p, p->classes, 0, d_cls, count, d_ws, ws_bytes, st);
      if (s) return s;
    }
    return run_cls(p, dir, x, y, w, static_cast<char*>(d_ws), st);
  }
  if (p->tile) {
    if (d_cls && (!d_ws || ws_bytes < 256)) return fail(HYGT_ERR_ARGUMENT, "hygt: workspace too small");
    return run_tile(p, dir, x, y, d_cls, count, energy,
                    d_cls ? reinterpret_cast<uint32_t*>(static_cast<char*>(d_ws) + w.err) : nullptr, st);
  }
  if (p->seg2 && bucketed && !energy) {
    if (!d_ws || ws_bytes < w.total) return fail(HYGT_ERR_ARGUMENT, "hygt: workspace too small");
    if (!(flags & HYGT_REUSE_BUCKETS)) {
      const int s = run_bucket(p, p->classes, 0, d_cls, count, d_ws, ws_bytes, st);
      if (s) return s;
    }
    return run_seg2(p, dir, x, y, count, w, static_cast<char*>(d_ws), st);
  }
  if (p->seg && bucketed && (!energy || p->seg_energy_smem)) {
    if (!d_ws || ws_bytes < w.total) return fail(HYGT_ERR_ARGUMENT, "hygt: workspace too small");
    if (!(flags & HYGT_REUSE_BUCKETS)) {
      const int s = run_bucket(p, p->classes, 0, d_cls, count, d_ws, ws_bytes, st);
      if (s) return s;
    }
    return run_segment(p, dir, x, y, count, energy, w, static_cast<char*>(d_ws), true, st);
  }
  if (d_cls) {
    if (!d_ws || ws_bytes < w.total) return fail(HYGT_ERR_ARGUMENT, "hygt: workspace too small");
    if (!(flags & HYGT_REUSE_BUCKETS)) {
      const int s = run_bucket(p, p->classes, p->chunk_rows, d_cls, count, d_ws, ws_bytes, st);
      if (s) return s;
    }
  }
  ApplyParams P{};
  P.x = x;
  P.y = y;
  char* ws = static_cast<char*>(d_ws);
  P.idx = bucketed ? reinterpret_cast<const uint32_t*>(ws + w.idx) : nullptr;
  P.seg_end = bucketed ? reinterpret_cast<const uint32_t*>(ws + w.seg) : nullptr;
  P.nseg = bucketed ? (uint32_t)(w.chunks * (p->classes + 1)) : 0;
  P.classes = p->classes;
  P.count = count;
  P.coef = p->d_coef[dir];
  P.stream_len = p->stream_len[dir];
  P.gidx = p->d_gidx[dir];
  P.gmask = p->gmask[dir];
  P.rounds = p->rounds;
  P.energy = energy;
  ApplyFn fn = select_apply(p->log2n, p->lanes_log2, p->algo == 0, dir == 0, energy != nullptr);
  if (!fn) return fail(HYGT_ERR_ARGUMENT, "hygt: no kernel for this dimension/layout");
  const size_t smem = apply_smem(p, dir);
  int occ = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, APPLY_THREADS, smem));
  if (occ < 1) occ = 1;
  const uint64_t rows_per_warp_step = 32u >> p->lanes_log2;
  const uint64_t warps_per_cta = APPLY_THREADS / 32;
  const uint64_t max_ctas = (uint64_t)p->num_sms * occ;
  uint64_t ctas = (count + rows_per_warp_step * warps_per_cta - 1) / (rows_per_warp_step * warps_per_cta);
  ctas = std::min(ctas, max_ctas);
  const uint64_t warps = ctas * warps_per_cta;
  uint64_t span = (count + warps - 1) / warps;
  span = (span + rows_per_warp_step - 1) / rows_per_warp_step * rows_per_warp_step;
  P.warp_span = span;
  fn<<<(unsigned)ctas, APPLY_THREADS, smem, st>>>(P);
  CU(cudaGetLastError());
  return ok();
}

}  // namespace

// ======================================================================= float API =======
extern "C" int hygt_plan_create(int log2_n, int rounds, int class_count, const double* angles,
                                const uint16_t* perms, uint32_t perm_mask, uint32_t flags,
                                hygt_plan** out) {
  return hygt_plan_create_ex(log2_n, rounds, class_count, angles, perms, perm_mask, flags, nullptr, out);
}

extern "C" int hygt_plan_create_ex(int log2_n, int rounds, int class_count, const double* angles,
                                   const uint16_t* perms, uint32_t perm_mask, uint32_t flags,
                                   const hygt_plan_options* opts, hygt_plan** out) {
  HYGT_NVTX("hygt_plan_create_ex");
  if (!out) return fail(HYGT_ERR_ARGUMENT, "hygt_plan_create: null out");
  *out = nullptr;
  hygt_plan_options opt;
  if (int s = resolve_options(opts, opt)) return s;
  if (log2_n < 1 || log2_n > 16) return fail(HYGT_ERR_ARGUMENT, "HyGTModel: log2_n out of range [1, 16]");
  if (log2_n > 8) return fail(HYGT_ERR_ARGUMENT, "hygt_plan_create: GPU path supports log2_n <= 8");
  if (rounds < 1) return fail(HYGT_ERR_ARGUMENT, "num_parameters: log2_n and rounds must be >= 1");
  if (class_count < 1 || class_count > 4096)
    return fail(HYGT_ERR_ARGUMENT, "hygt_plan_create: class_count must be in [1, 4096]");
  if (!angles) return fail(HYGT_ERR_ARGUMENT, "hygt_plan_create: null angles");
  if (perms && perm_mask == 0) perms = nullptr;
  if (int s = check_perms(log2_n, rounds, class_count, perms, perm_mask)) return s;
  for (size_t i = 0, n = (size_t)class_count * rounds * log2_n * ((size_t)1 << (log2_n - 1)); i < n; ++i)
    if (!std::isfinite(angles[i])) return fail(HYGT_ERR_ARGUMENT, "hygt_plan_create: non-finite angle");

  hygt_plan* p = new (std::nothrow) hygt_plan();
  if (!p) return fail(HYGT_ERR_CUDA, "out of host memory");
  p->kind = 0;
  p->opt = opt;
  p->log2n = log2_n;
  p->rounds = rounds;
  p->classes = class_count;
  p->perm_mask = perms ? perm_mask : 0;
  int l = env_int("HYGT_LANES_LOG2", -1);
  if (l < 0 || !select_apply(log2_n, l, false, true, false)) l = default_lane_log2(log2_n);
  p->lanes_log2 = l;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, dev);
  if (p->num_sms <= 0) p->num_sms = 148;
  // Locality window of the class bucketing: short rows (<= 128 B) are bucketed inside one
  // histogram tile so a warp's gathered rows stay within ~1 MB of HBM; longer rows bucket globally.
  const long long chunk_env = env_int("HYGT_CHUNK_ROWS", -1);
  p->chunk_rows = chunk_env >= 0 ? (uint64_t)chunk_env : (log2_n <= 5 ? BK_TILE : 0);

  const Layout ly{log2_n, l};
  bool standard = (flags & HYGT_PLAN_FORCE_STANDARD) != 0;
  DirTables t[2];
  for (int attempt = 0; attempt < 2; ++attempt) {
    bool good = true;
    for (int d = 0; d < 2 && good; ++d)
      good = build_direction(ly, rounds, class_count, angles, perms, p->perm_mask, d == 0,
                             standard, t[d]);
    if (good) break;
    if (flags & HYGT_PLAN_FORCE_FAST) {
      free_plan(p);
      return fail(HYGT_ERR_NUMERICAL, "hygt_plan_create: scale-folded form unsafe for these angles");
    }
    standard = true;
  }
  p->algo = standard ? 0 : 1;
  // input range: the scale-folded form's (hygt_plan.h), or the standard rotations' (orthogonal:
  // |value| <= sqrt(N) max|x| within fp32)
  p->input_limit = standard ? std::ldexp(1.0, 127 - (log2_n + 1) / 2)
                            : std::min(fast_input_limit(log2_n, t[0].sigma_min), fast_input_limit(log2_n, t[1].sigma_min));
  for (int d = 0; d < 2; ++d) {
    int s = upload(&p->d_coef[d], reinterpret_cast<const float2*>(t[d].coef.data()), t[d].coef.size());
    if (!s) s = upload(&p->d_gidx[d], t[d].gidx.data(), t[d].gmask ? t[d].gidx.size() : 0);
    if (s) {
      free_plan(p);
      return s;
    }
    p->stream_len[d] = t[d].stream_len;
    p->gmask[d] = t[d].gmask;
    ApplyFn fns[2] = {select_apply(log2_n, l, standard, d == 0, false),
                      select_apply(log2_n, l, standard, d == 0, d == 0)};
    for (ApplyFn fn : fns)
      if (fn && apply_smem(p, d) > 48 * 1024)
        smem_attr(fn, (int)apply_smem(p, d));
  }
  cudaGetLastError();
  // The staged kernel (N = 16) matches the NVRTC path's kernel time without its bucketing pass
  // or its seconds of compilation at plan creation; HYGT_JIT=2 forces the JIT path anyway.
  const bool stage_first = select_stage(log2_n, standard, true) && env_int("HYGT_STAGE", 1) != 0 &&
                           class_count <= STAGE_MAX_CLASSES && env_int("HYGT_JIT", 1) != 2;
  if (!stage_first && opt.allow_nvrtc && opt.kernel != HYGT_KERNEL_TENSOR &&
      jit_supported(log2_n, class_count, rounds) && env_int("HYGT_JIT", 1) != 0) {
    std::string err;
    if (jit_build(log2_n, rounds, class_count, angles, perms, p->perm_mask, p->algo == 0, p->jit, err)) {
      jit_release(p->jit);  // stay on the precompiled kernels
      if (env_int("HYGT_JIT_REQUIRED", 0)) {
        free_plan(p);
        return fail(HYGT_ERR_CUDA, err);
      }
    }
    // class runs long enough that a CTA range stays inside one or two class bodies
    if (p->jit.ok) p->chunk_rows = chunk_env >= 0 ? (uint64_t)chunk_env : ((uint64_t)1 << 18);
  }
  if (opt.kernel == HYGT_KERNEL_TENSOR) {  // every call runs on the composed-operator path
    if (int s = setup_gemm(p, angles, perms)) {
      free_plan(p);
      return s;
    }
    *out = p;
    return ok();
  }
  if (int s = setup_tile(p, angles, perms)) {
    free_plan(p);
    return s;
  }
  if (int s = setup_stage(p, angles, perms)) {
    free_plan(p);
    return s;
  }
  if (int s = setup_segment(p, angles, perms)) {
    free_plan(p);
    return s;
  }
  if (int s = setup_seg2(p, angles, perms)) {
    free_plan(p);
    return s;
  }
  if (int s = setup_cls(p, angles, perms)) {
    free_plan(p);
    return s;
  }
  if (int s = setup_gemm(p, angles, perms)) {
    free_plan(p);
    return s;
  }
  *out = p;
  return ok();
}

// Debug hook (not part of the public header): per-tile clock64 events of CTA 0 of the staged
// kernel are written to dev[k * 8 + e] (k < 64) while set; nullptr switches it off.
extern "C" void hygt_debug_stage_trace(void* dev) {
  g_stage_trace = static_cast<unsigned long long*>(dev);
}

extern "C" int hygt_plan_destroy(hygt_plan* plan) {
  free_plan(plan);
  return ok();
}

extern "C" int hygt_plan_algorithm(const hygt_plan* plan) { return plan ? plan->algo : -1; }

extern "C" double hygt_plan_input_limit(const hygt_plan* plan) {
  if (!plan) return 0.0;
  // the tensor-core path scales every row by a power of two of its own: any finite input
  if (plan->gemm) return std::ldexp(1.0, 127 - (plan->log2n + 1) / 2);
  return plan->kind == 0 ? plan->input_limit : 1048576.0;  // fixed point: |x| <= 2^20 (fixedpoint.hpp:145)
}

extern "C" int hygt_plan_path(const hygt_plan* plan) {
  return plan ? (plan->gemm ? 8 : plan->jit.ok ? 3 : plan->stage ? 4 : plan->cls_jit.ok ? 7 : plan->cls ? 6 : plan->tile ? 1 : plan->seg2 ? 5 : plan->seg ? 2 : 0) : -1;
}

extern "C" size_t hygt_workspace_bytes(const hygt_plan* plan, uint64_t count) {
  if (!plan) return 0;
  if (plan->gemm) return ws_layout(plan->classes, 0, count).total;
  if (plan->stage && !plan->jit.ok) return std::max<size_t>(stage_ws_bytes(plan, count), 256);
  if (plan->tile && !plan->jit.ok && !plan->cls) return 256;
  return ws_layout(plan->classes, plan->chunk_rows, count).total;
}

extern "C" int hygt_bucket(const hygt_plan* plan, const uint16_t* d_cls, uint64_t count,
                           void* d_ws, size_t ws_bytes, void* stream) {
  HYGT_NVTX("hygt_bucket");
  if (!plan) return fail(HYGT_ERR_ARGUMENT, "hygt_bucket: null plan");
  if (plan->gemm)
    return plan->classes > 1 ? run_bucket(plan, plan->classes, 0, d_cls, count, d_ws, ws_bytes, as_stream(stream)) : ok();
  if (plan->stage && !plan->jit.ok)  // per-tile class sort of the staged kernel
    return plan->classes > 1 ? run_stage_sort(plan, d_cls, count, d_ws, ws_bytes, as_stream(stream)) : ok();
  if (plan->tile && !plan->jit.ok && !plan->cls) return ok();  // tile plans sort each tile in shared memory
  return run_bucket(plan, plan->classes, plan->chunk_rows, d_cls, count, d_ws, ws_bytes,
                    as_stream(stream));
}

extern "C" int hygt_forward_f32(const hygt_plan* plan, const float* d_x, float* d_y,
                                const uint16_t* d_cls, uint64_t count, void* d_ws,
                                size_t ws_bytes, uint32_t flags, void* stream) {
  HYGT_NVTX("hygt_forward_f32");
  return run_apply(plan, 0, d_x, d_y, d_cls, count, nullptr, d_ws, ws_bytes, flags,
                   as_stream(stream));
}

extern "C" int hygt_inverse_f32(const hygt_plan* plan, const float* d_y, float* d_x,
                                const uint16_t* d_cls, uint64_t count, void* d_ws,
                                size_t ws_bytes, uint32_t flags, void* stream) {
  HYGT_NVTX("hygt_inverse_f32");
  return run_apply(plan, 1, d_y, d_x, d_cls, count, nullptr, d_ws, ws_bytes, flags,
                   as_stream(stream));
}

extern "C" int hygt_forward_energy_f32(const hygt_plan* plan, const float* d_x, float* d_y,
                                       const uint16_t* d_cls, uint64_t count, double* d_energy,
                                       void* d_ws, size_t ws_bytes, uint32_t flags,
                                       void* stream) {
  HYGT_NVTX("hygt_forward_energy_f32");
  if (!d_energy) return fail(HYGT_ERR_ARGUMENT, "hygt_forward_energy_f32: null energy");
  return run_apply(plan, 0, d_x, d_y, d_cls, count, d_energy, d_ws, ws_bytes, flags,
                   as_stream(stream));
}

extern "C" int hygt_sync_status(const hygt_plan* plan, void* d_ws, void* stream) {
  (void)plan;
  CU(cudaStreamSynchronize(as_stream(stream)));
  if (!d_ws) return ok();
  uint32_t err = 0;
  CU(cudaMemcpy(&err, d_ws, sizeof(err), cudaMemcpyDeviceToHost));
  if (err) {
    CU(cudaMemset(d_ws, 0, sizeof(uint32_t)));
    return fail(HYGT_ERR_ARGUMENT, "ResidualDataset: class id out of range");
  }
  return ok();
}

// ===================================================================== fixed point =======
namespace {

constexpr int FX_THREADS = 256;

struct FixedParams {
  const int64_t* x;
  int64_t* y;
  const uint16_t* cls;
  uint64_t count;
  int classes, log2n, rounds, angle_bits, precision_bits;
  const uint16_t* codes;  // [C][A]
  const int32_t* cos_tab;
  const int32_t* sin_tab;
  const uint16_t* gather;  // [C][R+1][N]
  uint64_t gmask;
  unsigned long long* err;  // min over (row << 3 | status)
};

// One warp per row; the row lives in shared memory as int64 (fixedpoint.hpp:154-182: int64
// products, rounding shift, |value| > 2^46 -> OverflowError).
template <bool FWD>
__global__ void __launch_bounds__(FX_THREADS) fixed_kernel(const FixedParams P) {
  extern __shared__ int64_t fx_smem[];
  const int n = 1 << P.log2n, half = n / 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t* buf = fx_smem + (size_t)warp * 2 * n;
  int64_t* tmp = buf + n;
  const uint64_t warps = (uint64_t)gridDim.x * (FX_THREADS / 32);
  const uint32_t mask = (1u << P.angle_bits) - 1u;
  const int prec = P.precision_bits;
  const int64_t rnd = (int64_t)1 << (prec - 1);
  const int64_t in_lim = (int64_t)1 << 20, val_lim = (int64_t)1 << 46;  // fixedpoint.hpp:142-143
  const size_t a_count = (size_t)P.rounds * P.log2n * half;
  for (uint64_t row = (uint64_t)blockIdx.x * (FX_THREADS / 32) + warp; row < P.count; row += warps) {
    const int64_t* xr = P.x + row * n;
    bool bad_in = false;
    for (int i = lane; i < n; i += 32) {
      const int64_t v = xr[i];
      buf[i] = v;
      bad_in |= v > in_lim || v < -in_lim;  // fixedpoint.hpp:145-150
    }
    int status = __any_sync(0xffffffffu, bad_in) ? 1 : 0;
    const int c = P.cls ? (int)P.cls[row] : 0;
    if (c >= P.classes) status = 1;  // dataset.hpp:47
    __syncwarp();
    if (!status) {
      const uint16_t* codes = P.codes + (size_t)c * a_count;
      const uint16_t* gsrc = P.gather + (size_t)c * (P.rounds + 1) * n;
      auto gather = [&](int step) {
        const uint16_t* gs = gsrc + (size_t)step * n;
        for (int i = lane; i < n; i += 32) tmp[i] = buf[gs[i]];
        __syncwarp();
        for (int i = lane; i < n; i += 32) buf[i] = tmp[i];
        __syncwarp();
      };
      if (P.gmask & 1ull) gather(0);
      for (int k = 0; k < P.rounds && !status; ++k) {
        const int r = FWD ? k : P.rounds - 1 - k;
        for (int pp = 0; pp < P.log2n && !status; ++pp) {
          const int d = FWD ? pp : P.log2n - 1 - pp;
          const uint32_t kk = 1u << d;
          const size_t base = ((size_t)r * P.log2n + d) * half;
          bool over = false;
          for (int j = lane; j < half; j += 32) {
            const uint32_t m = j + (j & (0u - kk)), nn = m + kk;
            uint32_t code = codes[base + j];
            if (!FWD) code = (0u - code) & mask;  // fixedpoint.hpp:170
            const int64_t cs = P.cos_tab[code], sn = P.sin_tab[code];
            const int64_t a = buf[m], b = buf[nn];
            const int64_t ym = (cs * a + sn * b + rnd) >> prec;  // arithmetic shift
            const int64_t yn = (cs * b - sn * a + rnd) >> prec;
            buf[m] = ym;
            buf[nn] = yn;
            over |= ym > val_lim || ym < -val_lim || yn > val_lim || yn < -val_lim;
          }
          if (__any_sync(0xffffffffu, over)) status = 4;  // fixedpoint.hpp:177-179
          __syncwarp();
        }
        if (!status && ((P.gmask >> (k + 1)) & 1ull)) gather(k + 1);
      }
    }
    int64_t* yr = P.y + row * n;
    for (int i = lane; i < n; i += 32) yr[i] = buf[i];
    if (status && lane == 0) atomicMin(P.err, (unsigned long long)((row << 3) | (uint64_t)status));
    __syncwarp();
  }
}

// Thread-per-row fixed-point kernel for N <= 64. Same arithmetic as fixed_kernel:
// y_m = (c a + s b + 2^(prec-1)) >> prec, y_n = (c b - s a + 2^(prec-1)) >> prec
// (fixedpoint.hpp:170-176), with the TrigTable lookups (and the inverse's code negation) done at
// plan creation into (c, s) int2 pairs in reference pair order per execution step. Tables of up
// to 48 KB are staged into shared memory; larger ones are read through L1.
// Values are held as int32. The plan selects this kernel only when fixed_int32_safe() proves,
// from the plan's own TrigTable gains and R * log2N, that no value of a valid row (|x| <= 2^20,
// checked, fixedpoint.hpp:145-150) reaches 2^30: then the reference's 2^46 overflow test
// (fixedpoint.hpp:177-179) cannot fire and the products fit IMAD.WIDE (32 x 32 -> 64).
template <int LOG2N, bool FWD>
__global__ void __launch_bounds__(FX_THREADS) fixed_row_kernel(const FixedParams P, const int2* __restrict__ tab,
                                                               uint32_t tab_smem_pairs) {
  constexpr int N = 1 << LOG2N, HALF = N / 2;
  extern __shared__ __align__(16) int32_t fxr_smem[];  // [table pairs] then scratch [N][FX_THREADS]
  const int tid = threadIdx.x;
  const int prec = P.precision_bits;
  const int64_t rnd = (int64_t)1 << (prec - 1);
  const int steps = P.rounds * LOG2N;
  const int2* s_tab = reinterpret_cast<const int2*>(fxr_smem);
  int32_t* scr = fxr_smem + 2 * tab_smem_pairs;
  for (uint32_t i = tid; i < tab_smem_pairs; i += FX_THREADS)
    reinterpret_cast<int2*>(fxr_smem)[i] = __ldg(tab + i);
  __syncthreads();
  for (uint64_t row = (uint64_t)blockIdx.x * FX_THREADS + tid; row < P.count;
       row += (uint64_t)gridDim.x * FX_THREADS) {
    int status = 0;
    const int c = P.cls ? (int)P.cls[row] : 0;
    if (c >= P.classes) status = 1;  // dataset.hpp:47
    int32_t v[N];
    const longlong2* xr = reinterpret_cast<const longlong2*>(P.x + row * N);
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
      const longlong2 q = __ldcs(xr + i);
      if (q.x > (1 << 20) || q.x < -(1 << 20) || q.y > (1 << 20) || q.y < -(1 << 20)) status = 1;
      v[2 * i] = (int32_t)q.x;
      v[2 * i + 1] = (int32_t)q.y;
    }
    if (!status) {
      const size_t tbase = (size_t)c * steps * HALF;
      const int2* t = tab_smem_pairs ? s_tab + tbase : tab + tbase;
      const uint16_t* gsrc = P.gather + (size_t)c * (P.rounds + 1) * N;
      auto gather = [&](int step) {
        const uint16_t* gs = gsrc + (size_t)step * N;
#pragma unroll
        for (int i = 0; i < N; ++i) scr[i * FX_THREADS + tid] = v[i];
#pragma unroll
        for (int i = 0; i < N; i += 8) {
          const uint4 g = __ldg(reinterpret_cast<const uint4*>(gs + i));
          const uint32_t w[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            v[i + 2 * h] = scr[(w[h] & 0xffffu) * FX_THREADS + tid];
            v[i + 2 * h + 1] = scr[(w[h] >> 16) * FX_THREADS + tid];
          }
        }
      };
      if (P.gmask & 1ull) gather(0);
      for (int k = 0; k < P.rounds; ++k) {
#pragma unroll
        for (int pp = 0; pp < LOG2N; ++pp) {
          const int d = FWD ? pp : LOG2N - 1 - pp;
          const int2* u = t + (size_t)(k * LOG2N + pp) * HALF;
#pragma unroll
          for (int j = 0; j < HALF; j += 2) {
            const int4 q = tab_smem_pairs ? *reinterpret_cast<const int4*>(u + j)
                                          : __ldg(reinterpret_cast<const int4*>(u + j));
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int jj = j + h;
              const int m = jj + (jj & -(1 << d)), n = m + (1 << d);  // hypercube.hpp:73-74
              const int64_t cs = h ? q.z : q.x, sn = h ? q.w : q.y;
              const int32_t a = v[m], b = v[n];
              v[m] = (int32_t)((cs * a + sn * b + rnd) >> prec);
              v[n] = (int32_t)((cs * b - sn * a + rnd) >> prec);
            }
          }
        }
        if ((P.gmask >> (k + 1)) & 1ull) gather(k + 1);
      }
    }
    longlong2* yr = reinterpret_cast<longlong2*>(P.y + row * N);
#pragma unroll
    for (int i = 0; i < N / 2; ++i) __stcs(yr + i, make_longlong2(v[2 * i], v[2 * i + 1]));
    if (status) atomicMin(P.err, (unsigned long long)((row << 3) | (uint64_t)status));
  }
}

using FixedRowFn = void (*)(FixedParams, const int2*, uint32_t);
FixedRowFn select_fixed_row(int log2n, bool fwd) {
  switch (log2n) {
    case 1: return fwd ? fixed_row_kernel<1, true> : fixed_row_kernel<1, false>;
    case 2: return fwd ? fixed_row_kernel<2, true> : fixed_row_kernel<2, false>;
    case 3: return fwd ? fixed_row_kernel<3, true> : fixed_row_kernel<3, false>;
    case 4: return fwd ? fixed_row_kernel<4, true> : fixed_row_kernel<4, false>;
    case 5: return fwd ? fixed_row_kernel<5, true> : fixed_row_kernel<5, false>;
    case 6: return fwd ? fixed_row_kernel<6, true> : fixed_row_kernel<6, false>;
    default: return nullptr;
  }
}

// Staged fixed-point path (hygt_stage_fixed.cuh). Returns a status, or -1 when the sort pass met
// invalid class ids (the caller re-runs the row kernel, which reports the first failing row).
// Called with the plan mutex held.
int run_fixed_staged(const hygt_plan* p, int dir, const int64_t* x, int64_t* y, const uint16_t* cls,
                     uint64_t count, uint64_t* first_bad, cudaStream_t st) {
  hygt_plan* mp = const_cast<hygt_plan*>(p);  // the sort workspace is plan-owned, guarded by fixed_mu
  const bool sorted = cls != nullptr;
  if (sorted) {
    const uint64_t tiles = (count + p->fx_rows - 1) / p->fx_rows;
    const size_t need = 256 + tiles * p->fx_block_words * 2;
    if (mp->fx_ws_bytes < need) {
      cudaFree(mp->d_fx_ws);
      mp->d_fx_ws = nullptr;
      mp->fx_ws_bytes = 0;
      CU(cudaMalloc(&mp->d_fx_ws, need));
      mp->fx_ws_bytes = need;
    }
    CU(cudaMemsetAsync(mp->d_fx_ws, 0, 4, st));
    if (int s = stage_sort(p->classes, p->fx_rows, p->fx_block_words, STAGE_FX_VPT, p->num_sms, cls, count, mp->d_fx_ws, st))
      return s;
  }
  StageFxParams F{};
  F.x = x;
  F.y = y;
  F.count = count;
  F.classes = p->classes;
  F.rounds = p->rounds;
  F.precision_bits = p->precision_bits;
  F.tab = p->d_fxtab[dir];
  F.gtab = p->d_fxgt[dir];
  F.gmask = p->gmask[dir];
  F.tile_rows = p->fx_rows;
  F.ent = sorted ? reinterpret_cast<const uint16_t*>(static_cast<char*>(mp->d_fx_ws) + 256) : nullptr;
  F.block_words = p->fx_block_words;
  F.err = p->d_fixed_err;
  const uint64_t tiles = (count + p->fx_rows - 1) / p->fx_rows;
  StageFxFn fn = select_stage_fixed(p->log2n, dir == 0);
  fn<<<(unsigned)std::min<uint64_t>(tiles, (uint64_t)p->num_sms), (STAGE_FX_WARPS + 1) * 32, p->fx_smem[dir], st>>>(F);
  CU(cudaGetLastError());
  unsigned long long key = 0;
  uint32_t bad_ids = 0;
  CU(cudaMemcpyAsync(&key, p->d_fixed_err, sizeof(key), cudaMemcpyDeviceToHost, st));
  if (sorted) CU(cudaMemcpyAsync(&bad_ids, mp->d_fx_ws, sizeof(bad_ids), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (bad_ids) return -1;
  if (key == ~0ull) return ok();
  if (first_bad) *first_bad = key >> 3;
  return fail(HYGT_ERR_ARGUMENT, "fixed transform: input magnitude exceeds 2^20");
}

// Per-class NVRTC chain for fixed plans (hygt_jit.cpp). Same contract as run_fixed_staged:
// a status, or -1 when the bucketing met invalid class ids. Called with the plan mutex held.
int run_fixed_jit(const hygt_plan* p, int dir, const int64_t* x, int64_t* y, const uint16_t* cls,
                  uint64_t count, uint64_t* first_bad, cudaStream_t st) {
  hygt_plan* mp = const_cast<hygt_plan*>(p);  // the bucket workspace is plan-owned, guarded by fixed_mu
  const bool bucketed = cls && p->classes > 1;
  const uint32_t* idx = nullptr;
  const uint32_t* seg = nullptr;
  if (cls) {
    const WsLayout w = ws_layout(p->classes, 0, count);
    if (mp->fx_bws_bytes < w.total) {
      cudaFree(mp->d_fx_bws);
      mp->d_fx_bws = nullptr;
      mp->fx_bws_bytes = 0;
      CU(cudaMalloc(&mp->d_fx_bws, w.total));
      mp->fx_bws_bytes = w.total;
    }
    CU(cudaMemsetAsync(mp->d_fx_bws, 0, 4, st));
    if (int s = run_bucket(p, p->classes, 0, cls, count, mp->d_fx_bws, mp->fx_bws_bytes, st)) return s;
    if (bucketed) {
      idx = reinterpret_cast<const uint32_t*>(static_cast<char*>(mp->d_fx_bws) + w.idx);
      seg = reinterpret_cast<const uint32_t*>(static_cast<char*>(mp->d_fx_bws) + w.seg);
    }
  }
  if (jit_fixed_launch(p->fx_jit, dir, x, y, idx, seg, p->classes, count, p->d_fixed_err, st))
    return fail(HYGT_ERR_CUDA, std::string("hygt: fixed class launch failed: ") + cudaGetErrorString(cudaGetLastError()));
  unsigned long long key = 0;
  uint32_t bad_ids = 0;
  CU(cudaMemcpyAsync(&key, p->d_fixed_err, sizeof(key), cudaMemcpyDeviceToHost, st));
  if (cls) CU(cudaMemcpyAsync(&bad_ids, mp->d_fx_bws, sizeof(bad_ids), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (bad_ids) return -1;
  if (key == ~0ull) return ok();
  if (first_bad) *first_bad = key >> 3;
  return fail(HYGT_ERR_ARGUMENT, "fixed transform: input magnitude exceeds 2^20");
}

int run_fixed(const hygt_plan* p, int dir, const int64_t* x, int64_t* y, const uint16_t* cls,
              uint64_t count, uint64_t* first_bad, cudaStream_t st) {
  if (!p || p->kind != 1) return fail(HYGT_ERR_ARGUMENT, "hygt: not a fixed-point plan");
  if (first_bad) *first_bad = count;
  if (count == 0) return ok();
  if (!x || !y) return fail(HYGT_ERR_ARGUMENT, "hygt: null data pointer");
  std::lock_guard<std::mutex> lock(*p->fixed_mu);
  const unsigned long long init = ~0ull;
  CU(cudaMemcpyAsync(p->d_fixed_err, &init, sizeof(init), cudaMemcpyHostToDevice, st));
  FixedParams P{x, y, cls, count, p->classes, p->log2n, p->rounds, p->angle_bits,
                p->precision_bits, p->d_codes, p->d_cos, p->d_sin, p->d_fgather[dir],
                p->gmask[dir], p->d_fixed_err};
  const bool aligned16 = (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(y) & 15) == 0;
  if (p->fx_jit.ok && aligned16 && count < 0xFFFFFFFFull) {  // u32 row ids
    const int s = run_fixed_jit(p, dir, x, y, cls, count, first_bad, st);
    if (s != -1) return s;  // -1: invalid class ids -> the exact first failing row from below
    CU(cudaMemcpyAsync(p->d_fixed_err, &init, sizeof(init), cudaMemcpyHostToDevice, st));
  } else if (p->stagefx && aligned16) {
    const int s = run_fixed_staged(p, dir, x, y, cls, count, first_bad, st);
    if (s != -1) return s;  // -1: invalid class ids -> the exact first failing row from below
    CU(cudaMemcpyAsync(p->d_fixed_err, &init, sizeof(init), cudaMemcpyHostToDevice, st));
  }
  FixedRowFn rfn = p->d_ftab[dir] ? select_fixed_row(p->log2n, dir == 0) : nullptr;
  if (rfn) {
    const size_t pairs = (size_t)p->classes * p->rounds * p->log2n * ((1u << p->log2n) / 2);
    const uint32_t smem_pairs = pairs * sizeof(int2) <= 48 * 1024 ? (uint32_t)pairs : 0u;
    const size_t smem = smem_pairs * sizeof(int2) +
                        (p->gmask[dir] ? (size_t)FX_THREADS * (1u << p->log2n) * sizeof(int32_t) : 0);
    if (smem > 48 * 1024) smem_attr(rfn, (int)smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, rfn, FX_THREADS, smem);
    const uint64_t ctas = std::min<uint64_t>((count + FX_THREADS - 1) / FX_THREADS,
                                             (uint64_t)p->num_sms * std::max(occ, 1));
    rfn<<<(unsigned)ctas, FX_THREADS, smem, st>>>(P, p->d_ftab[dir], smem_pairs);
  } else {
    const size_t smem = (size_t)(FX_THREADS / 32) * 2 * (1u << p->log2n) * sizeof(int64_t);
    const uint64_t ctas = std::min<uint64_t>((count + 7) / 8, (uint64_t)p->num_sms * 8);
    if (dir == 0) fixed_kernel<true><<<(unsigned)ctas, FX_THREADS, smem, st>>>(P);
    else fixed_kernel<false><<<(unsigned)ctas, FX_THREADS, smem, st>>>(P);
  }
  CU(cudaGetLastError());
  unsigned long long key = 0;
  CU(cudaMemcpyAsync(&key, p->d_fixed_err, sizeof(key), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (key == ~0ull) return ok();
  const uint64_t row = key >> 3;
  const int status = (int)(key & 7);
  if (first_bad) *first_bad = row;
  if (status == 4) return fail(HYGT_ERR_OVERFLOW, "fixed transform: intermediate exceeds 2^46");
  if (cls) {
    uint16_t c = 0;
    CU(cudaMemcpy(&c, cls + row, sizeof(c), cudaMemcpyDeviceToHost));
    if (c >= p->classes) return fail(HYGT_ERR_ARGUMENT, "ResidualDataset: class id out of range");
  }
  return fail(HYGT_ERR_ARGUMENT, "fixed transform: input magnitude exceeds 2^20");
}

}  // namespace

namespace {
// Norm bound for the rounded integer butterflies of forward_fixed / inverse_fixed
// (fixedpoint.hpp:170-176). One pass maps a pair (a, b) to (round((c a + s b) / 2^p),
// round((c b - s a) / 2^p)) with (c, s) = TrigTable[code]; the exact part has L2 gain
// g_code = sqrt(c^2 + s^2) / 2^p and each rounding adds at most 1/2 per element, so over the
// N/2 disjoint pairs of a pass ||x'|| <= g ||x|| + sqrt(N)/2 with g the largest gain among the
// codes the plan uses (the inverse's negated codes have the same gain). Permutations keep the
// norm, and |value| <= ||x||. Inputs are at most 2^20 per element (checked per row,
// fixedpoint.hpp:142-150), so after T = R log2N passes
//   |value| <= g^T sqrt(N) 2^20 + sqrt(N)/2 * sum_{i<T} g^i.
// The int32 kernels are safe when this stays below 2^30 (products c*a then fit IMAD.WIDE and
// the int64 sums cannot wrap); the bound is evaluated in long double, monotone in every term.
bool fixed_int32_safe(int log2n, int rounds, int classes, size_t a, const uint16_t* codes,
                      const int32_t* ct, const int32_t* sn, int prec) {
  long double g = 0;
  for (size_t i = 0; i < a * (size_t)classes; ++i) {
    const long double c = ct[codes[i]], s = sn[codes[i]];
    g = std::max(g, sqrtl(c * c + s * s) / (long double)((int64_t)1 << prec));
  }
  const long double rn = sqrtl((long double)((size_t)1 << log2n));
  long double bound = rn * 1048576.0L;
  const int T = rounds * log2n;
  for (int t = 0; t < T; ++t) {
    bound = g * bound + rn / 2;
    if (bound >= 1073741824.0L) return false;
  }
  return true;
}
}  // namespace

extern "C" int hygt_fixed_plan_create(int log2_n, int rounds, int class_count, int angle_bits,
                                      int precision_bits, const uint16_t* codes,
                                      const uint16_t* perms, uint32_t perm_mask,
                                      hygt_plan** out) {
  return hygt_fixed_plan_create_ex(log2_n, rounds, class_count, angle_bits, precision_bits, codes, perms,
                                   perm_mask, nullptr, out);
}

extern "C" int hygt_fixed_plan_create_ex(int log2_n, int rounds, int class_count, int angle_bits,
                                         int precision_bits, const uint16_t* codes,
                                         const uint16_t* perms, uint32_t perm_mask,
                                         const hygt_plan_options* opts, hygt_plan** out) {
  HYGT_NVTX("hygt_fixed_plan_create_ex");
  if (!out) return fail(HYGT_ERR_ARGUMENT, "hygt_fixed_plan_create: null out");
  *out = nullptr;
  hygt_plan_options opt;
  if (int s = resolve_options(opts, opt)) return s;
  if (log2_n < 1 || log2_n > 16) return fail(HYGT_ERR_ARGUMENT, "QuantizedHyGTModel: log2_n out of range [1, 16]");
  if (log2_n > 8) return fail(HYGT_ERR_ARGUMENT, "hygt_fixed_plan_create: GPU path supports log2_n <= 8");
  if (angle_bits < 1 || angle_bits > 12)
    return fail(HYGT_ERR_ARGUMENT, "QuantizedHyGTModel: angle_bits out of range [1, 12]");
  if (precision_bits < 4 || precision_bits > 15)
    return fail(HYGT_ERR_ARGUMENT, "TrigTable: precision_bits out of range [4, 15]");
  if (rounds < 1) return fail(HYGT_ERR_ARGUMENT, "num_parameters: log2_n and rounds must be >= 1");
  if (class_count < 1 || class_count > 65535) return fail(HYGT_ERR_ARGUMENT, "hygt_fixed_plan_create: class_count");
  if (!codes) return fail(HYGT_ERR_ARGUMENT, "hygt_fixed_plan_create: null codes");
  const size_t n = (size_t)1 << log2_n;
  const size_t a = (size_t)rounds * log2_n * n / 2;
  for (size_t i = 0; i < a * class_count; ++i)
    if (codes[i] > (1u << angle_bits) - 1u)
      return fail(HYGT_ERR_ARGUMENT, "QuantizedHyGTModel: code exceeds 2^angle_bits");
  if (perms && perm_mask == 0) perms = nullptr;
  if (int s = check_perms(log2_n, rounds, class_count, perms, perm_mask)) return s;

  hygt_plan* p = new (std::nothrow) hygt_plan();
  if (!p) return fail(HYGT_ERR_CUDA, "out of host memory");
  p->kind = 1;
  p->opt = opt;
  p->log2n = log2_n;
  p->rounds = rounds;
  p->classes = class_count;
  p->angle_bits = angle_bits;
  p->precision_bits = precision_bits;
  p->perm_mask = perms ? perm_mask : 0;
  p->fixed_mu = new std::mutex();
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, dev);
  // TrigTable (fixedpoint.hpp:37-52), evaluated on the host exactly as the reference does.
  const size_t size = (size_t)1 << angle_bits;
  std::vector<int32_t> ct(size), sn(size);
  const double scale = (double)((int64_t)1 << precision_bits);
  for (size_t q = 0; q < size; ++q) {
    const double ang = 2.0 * 3.14159265358979323846 * (double)q / (double)size;
    ct[q] = (int32_t)std::lround(std::cos(ang) * scale);
    sn[q] = (int32_t)std::lround(std::sin(ang) * scale);
  }
  int s = upload(&p->d_cos, ct.data(), size);
  if (!s) s = upload(&p->d_sin, sn.data(), size);
  if (!s) s = upload(&p->d_codes, codes, a * class_count);
  if (!s) {
    unsigned long long* e = nullptr;
    if (cudaMalloc(&e, sizeof(*e)) != cudaSuccess) s = fail(HYGT_ERR_CUDA, "cudaMalloc");
    p->d_fixed_err = e;
  }
  // The int32 kernels (staged N = 16, thread-per-row N <= 64, per-class NVRTC chain) hold values
  // in 32 bits. They are used only when a bound computed from this plan's own table proves that
  // no value can reach 2^31 (so the reference's 2^46 test, fixedpoint.hpp:177-179, cannot fire
  // either); otherwise every row runs on the int64 fixed_kernel, which applies that test.
  const bool int32_ok = fixed_int32_safe(log2_n, rounds, class_count, a, codes, ct.data(), sn.data(),
                                         precision_bits);
  p->fx_int32 = int32_ok;
  for (int d = 0; d < 2 && !s; ++d) {
    std::vector<uint16_t> g((size_t)class_count * (rounds + 1) * n, 0);
    for (int c = 0; c < class_count; ++c) {
      uint64_t gm = 0;
      const auto gs = exec_gathers(log2_n, rounds, perms ? perms + (size_t)c * rounds * n : nullptr,
                                   p->perm_mask, d == 0, &gm);
      p->gmask[d] = gm;
      for (int k = 0; k <= rounds; ++k)
        for (size_t i = 0; i < n && !gs[k].empty(); ++i)
          g[((size_t)c * (rounds + 1) + k) * n + i] = (uint16_t)gs[k][i];
    }
    s = upload(&p->d_fgather[d], g.data(), g.size());
    if (!s && int32_ok && log2_n == 4 && class_count <= STAGE_MAX_CLASSES && env_int("HYGT_FIXED_STAGE", 1) != 0) {
      // element-pair (c, s', c, s') units per execution step for the staged kernel, and its
      // permutation offsets (src * 128 into the [element][lane] int32 scratch)
      const uint32_t mask = (1u << angle_bits) - 1u;
      const size_t steps = (size_t)rounds * log2_n, half = n / 2;
      std::vector<int4> tab((size_t)class_count * steps * half);
      std::vector<int32_t> ce(n), se(n);
      for (int c = 0; c < class_count; ++c)
        for (size_t k = 0; k < (size_t)rounds; ++k)
          for (int pp = 0; pp < log2_n; ++pp) {
            const int r = d == 0 ? (int)k : rounds - 1 - (int)k;
            const int dd = d == 0 ? pp : log2_n - 1 - pp;
            const uint32_t kk = 1u << dd;
            const size_t base = ((size_t)r * log2_n + dd) * half;  // model.hpp:77-79
            for (uint32_t j = 0; j < half; ++j) {
              const uint32_t m = j + (j & (0u - kk)), nn = m + kk;  // hypercube.hpp:73-74
              uint32_t code = codes[(size_t)c * a + base + j];
              if (d == 1) code = (0u - code) & mask;  // fixedpoint.hpp:170
              ce[m] = ce[nn] = ct[code];
              se[m] = sn[code];
              se[nn] = -sn[code];
            }
            int4* u = &tab[((size_t)c * steps + k * log2_n + pp) * half];
            for (size_t j = 0; j < half; ++j) u[j] = make_int4(ce[2 * j], se[2 * j], ce[2 * j + 1], se[2 * j + 1]);
          }
      const uint32_t gs = stage_gstride(log2_n, rounds) / 2;
      std::vector<uint16_t> gt((size_t)class_count * gs, 0);
      for (int c = 0; c < class_count; ++c) {
        uint64_t gm = 0;
        const auto g = exec_gathers(log2_n, rounds, perms ? perms + (size_t)c * rounds * n : nullptr,
                                    p->perm_mask, d == 0, &gm);
        for (int k = 0; k <= rounds; ++k)
          for (size_t i = 0; i < g[k].size(); ++i) gt[(size_t)c * gs + (size_t)k * n + i] = (uint16_t)(g[k][i] * 128);
      }
      s = upload(&p->d_fxtab[d], tab.data(), tab.size());
      if (!s) s = upload(&p->d_fxgt[d], gt.data(), gt.size());
      if (!s && d == 1) {  // both directions built: size the tiles to the shared memory
        uint32_t T = (uint32_t)std::max(0, STAGE_FX_WARPS * 32 * STAGE_FX_VPT - (STAGE_FX_VPT - 1) * class_count);
        T = std::min<uint32_t>(T, 1016) / 8 * 8;
        size_t sm[2] = {0, 0};
        for (; T >= 64; T -= 8) {
          for (int e = 0; e < 2; ++e)
            sm[e] = stage_fx_smem_layout(log2_n, STAGE_FX_VPT, STAGE_FX_WARPS, class_count, rounds, T, p->gmask[e] != 0).total;
          if (std::max(sm[0], sm[1]) <= 227 * 1024) break;
        }
        if (T >= 64) {
          for (int e = 0; e < 2; ++e) {
            smem_attr(select_stage_fixed(log2_n, e == 0), (int)sm[e]);
            p->fx_smem[e] = sm[e];
          }
          cudaGetLastError();
          p->fx_rows = T;
          p->fx_block_words = stage_block_words(T, STAGE_FX_VPT, class_count);
          p->stagefx = true;
        }
      }
    }
    if (!s && int32_ok && log2_n <= 6 && env_int("HYGT_FIXED_ROW", 1) != 0) {
      // (c, s) per pair of the thread-per-row kernel, in execution order
      const uint32_t mask = (1u << angle_bits) - 1u;
      const size_t steps = (size_t)rounds * log2_n, half = n / 2;
      std::vector<int2> tab((size_t)class_count * steps * half);
      for (int c = 0; c < class_count; ++c)
        for (size_t k = 0; k < (size_t)rounds; ++k)
          for (int pp = 0; pp < log2_n; ++pp) {
            const int r = d == 0 ? (int)k : rounds - 1 - (int)k;
            const int dd = d == 0 ? pp : log2_n - 1 - pp;
            const size_t base = ((size_t)r * log2_n + dd) * half;  // model.hpp:77-79
            int2* u = &tab[((size_t)c * steps + k * log2_n + pp) * half];
            for (size_t j = 0; j < half; ++j) {
              uint32_t code = codes[(size_t)c * a + base + j];
              if (d == 1) code = (0u - code) & mask;  // fixedpoint.hpp:170
              u[j] = make_int2(ct[code], sn[code]);
            }
          }
      s = upload(&p->d_ftab[d], tab.data(), tab.size());
    }
  }
  if (s) {
    free_plan(p);
    return s;
  }
  if (!s && int32_ok && opt.allow_nvrtc && jit_fixed_supported(log2_n, rounds, class_count) &&
      env_int("HYGT_FIXED_JIT", 1) != 0) {
    std::string err;
    if (jit_fixed_build(log2_n, rounds, class_count, angle_bits, precision_bits, codes, ct.data(), sn.data(),
                        perms, p->perm_mask, p->fx_jit, err))
      jit_cls_release(p->fx_jit);  // stay on the precompiled kernels
  }
  *out = p;
  return ok();
}

extern "C" int hygt_forward_i64(const hygt_plan* plan, const int64_t* d_x, int64_t* d_y,
                                const uint16_t* d_cls, uint64_t count, uint64_t* first_bad,
                                void* stream) {
  HYGT_NVTX("hygt_forward_i64");
  return run_fixed(plan, 0, d_x, d_y, d_cls, count, first_bad, as_stream(stream));
}

extern "C" int hygt_inverse_i64(const hygt_plan* plan, const int64_t* d_y, int64_t* d_x,
                                const uint16_t* d_cls, uint64_t count, uint64_t* first_bad,
                                void* stream) {
  HYGT_NVTX("hygt_inverse_i64");
  return run_fixed(plan, 1, d_y, d_x, d_cls, count, first_bad, as_stream(stream));
}

// ======================================================================= synthetic =======
namespace {

__device__ __forceinline__ uint64_t smix(uint64_t z) {  // SplitMix64 finaliser
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double u01(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }
__device__ __forceinline__ float gauss(uint64_t seed, uint64_t row, uint32_t k) {
  const uint64_t h = smix(seed ^ smix(row * 0x100000001B3ull + (k >> 1)));
  double a = u01(h), b = u01(smix(h));
  if (a <= 0.0) a = 0x1.0p-53;
  const double r = sqrt(-2.0 * log(a));
  return (float)((k & 1) ? r * sin(6.283185307179586 * b) : r * cos(6.283185307179586 * b));
}

__global__ void synth_classes_kernel(uint16_t* cls, uint64_t count, uint64_t row0, int classes,
                                     uint64_t seed) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x)
    cls[i] = (uint16_t)(smix(seed ^ smix(row0 + i)) % (uint64_t)classes);
}

// One warp per row; the bs x bs block sits in shared memory. Separable AR(1) recursion
// (u_0 = z_0, u_k = rho u_{k-1} + sqrt(1-rho^2) z_k) along columns then rows gives covariance
// A (x) A with A_ij = rho^|i-j| (ar1_covariance_2d, statistics.hpp:287-305).
__global__ void synth_rows_kernel(float* x, uint64_t count, uint64_t row0, int bs,
                                  const uint16_t* cls, const float* rho_c, float sigma,
                                  float edge_frac, float edge_amp, float edge_noise,
                                  uint64_t seed) {
  __shared__ float tile[8][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* t = tile[warp];
  const int n = bs * bs;
  for (uint64_t i = (uint64_t)blockIdx.x * 8 + warp; i < count; i += (uint64_t)gridDim.x * 8) {
    const uint64_t row = row0 + i;
    const float rho = rho_c ? rho_c[cls ? cls[i] : 0] : 0.9f;
    const float q = sqrtf(1.f - rho * rho);
    const bool edge = u01(smix(seed ^ 0xED6Eull ^ smix(row))) < (double)edge_frac;
    if (!edge) {
      if (lane < bs) {  // column recursion
        float prev = 0.f;
        for (int r = 0; r < bs; ++r) {
          const float z = gauss(seed, row, r * bs + lane);
          prev = r == 0 ? z : rho * prev + q * z;
          t[r * bs + lane] = prev;
        }
      }
      __syncwarp();
      if (lane < bs) {  // row recursion
        float prev = 0.f;
        for (int c = 0; c < bs; ++c) {
          const float u = t[lane * bs + c];
          prev = c == 0 ? u : rho * prev + q * u;
          t[lane * bs + c] = prev;
        }
      }
      __syncwarp();
      for (int k = lane; k < n; k += 32) x[i * n + k] = sigma * t[k];
    } else {
      const uint64_t h = smix(seed ^ 0x5EDull ^ smix(row));
      const double phi = 3.141592653589793 * u01(h);
      const double delta = (u01(smix(h)) - 0.5) * 0.5 * bs;
      const double cph = cos(phi), sph = sin(phi), mid = 0.5 * (bs - 1);
      for (int k = lane; k < n; k += 32) {
        const int r = k / bs, c = k % bs;
        const double d = (c - mid) * cph + (r - mid) * sph - delta;
        x[i * n + k] = (float)(edge_amp * (d >= 0 ? 1.0 : -1.0)) + edge_noise * gauss(seed ^ 0xE, row, k);
      }
    }
    __syncwarp();
  }
}

}  // namespace

extern "C" int hygt_synth_classes(uint16_t* d_cls, uint64_t count, uint64_t row0,
                                  int class_count, uint64_t seed, void* stream) {
  if (!d_cls || class_count < 1) return fail(HYGT_ERR_ARGUMENT, "hygt_synth_classes: bad args");
  if (!count) return ok();
  synth_classes_kernel<<<(unsigned)std::min<uint64_t>((count + 255) / 256, 148 * 16), 256, 0,
                         as_stream(stream)>>>(d_cls, count, row0, class_count, seed);
  CU(cudaGetLastError());
  return ok();
}

extern "C" int hygt_synth_rows_f32(float* d_x, uint64_t count, uint64_t row0, int block_size,
                                   const uint16_t* d_cls, const float* d_rho_per_class,
                                   int class_count, float sigma, float edge_fraction,
                                   float edge_amplitude, float edge_noise, uint64_t seed,
                                   void* stream) {
  (void)class_count;
  if (!d_x || block_size < 1 || block_size > 16)
    return fail(HYGT_ERR_ARGUMENT, "hygt_synth_rows_f32: block_size in [1, 16]");
  if (!count) return ok();
  synth_rows_kernel<<<(unsigned)std::min<uint64_t>((count + 7) / 8, 148 * 32), 256, 0,
                      as_stream(stream)>>>(d_x, count, row0, block_size, d_cls, d_rho_per_class,
                                           sigma, edge_fraction, edge_amplitude, edge_noise, seed);
  CU(cudaGetLastError());
  return ok();
}
