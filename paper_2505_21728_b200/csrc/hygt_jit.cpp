// hygt_jit.cpp -- plan-specialised HyGT kernels for short rows (N <= 64), compiled at plan
// creation with NVRTC for sm_100a.
//
// The transform of each class is emitted as straight-line CUDA: every butterfly is two FFMAs
// whose coefficients are immediates (no coefficient loads at all), every permutation is a
// compile-time register renaming (no shared-memory round trip), and the final scales are
// immediate multiplies. One kernel per direction holds all classes behind a switch on the row's
// class; rows are class-sorted per tile in shared memory (as in hygt_tile.cuh) so warps are
// class-uniform and only one case body is live per warp. A row is owned by one lane; HBM traffic
// stays coalesced through a bank-swizzled per-warp transpose buffer (cooperative 128-bit loads of
// the warp's 32 rows, then each lane reads its own row).
//
// Reference arithmetic: butterflies and order as transform.hpp:45-66 / model.hpp:77-79, gathers
// as transform.hpp:75-80 (inverse: scatter first, :88-93); coefficients from hygt_plan.cpp.
#include "hygt_jit.h"
#include "hygt_knobs.h"

#include <nvrtc.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <mutex>
#include <sstream>
#include <thread>
#include <string>
#include <unordered_map>
#include <vector>

namespace hygt_gpu {

namespace {

bool env_on(const char* name) { return knob(name, 0) != 0; }    // development knob set and non-zero
bool env_off(const char* name) { return knob(name, 1) == 0; }   // development knob set to 0

std::string lit(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  char b[40];
  std::snprintf(b, sizeof b, "__int_as_float(0x%08x)", u);
  return b;
}

// Chunk swizzle of the transpose buffer: row r, 16-byte chunk q -> q ^ swz(r).
const char* kSwizzle[] = {
    /*log2n=2*/ "0", /*3*/ "((r >> 2) & 1)", /*4*/ "((r >> 1) & 3)", /*5*/ "(r & 7)", /*6*/ "(r & 7)"};

const char* kPrologue = R"CUDA(
typedef unsigned int u32;
typedef unsigned long long u64;
typedef unsigned short u16;
#define FULL 0xffffffffu
// Rows are visited in class-bucketed order (idx: position -> row; seg_end: [chunks][C+1] run
// ends, bin C = invalid ids). Each CTA streams a contiguous range of positions, so all its warps
// sit in the same class run -- one class body hot in the instruction cache. idx == 0: identity
// order, single class.
extern "C" __global__ void __launch_bounds__(WARPS * 32, MINB)
hygt_jit_kernel(const float* __restrict__ x, float* __restrict__ y, const u32* __restrict__ idx,
                const u32* __restrict__ seg_end, u32 nseg, u64 count, int C, u64 span) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float4* wb = (float4*)sm + (size_t)warp * 32 * NQ;
  const u64 beg = (u64)blockIdx.x * span;
  if (beg >= count) return;
  const u64 end = beg + span < count ? beg + span : count;
  const float4* x4 = (const float4*)x;
  float4* y4 = (float4*)y;
  // per-lane walk over the run ends (positions only increase)
  u32 f = 0;
  if (idx) {
    u32 lo = 0, hi = nseg;
    const u64 p = beg + (u64)warp * 32 + lane;
    while (lo < hi) {
      const u32 mid = (lo + hi) >> 1;
      if ((u64)__ldg(seg_end + mid) <= p) lo = mid + 1; else hi = mid;
    }
    f = lo;
  }
  auto meta = [&](u64 p, u32& row, u32& c) {
    if (p >= end) { row = 0; c = 0; return; }
    if (!idx) { row = (u32)p; c = 0; return; }
    while (f < nseg && (u64)__ldg(seg_end + f) <= p) ++f;
    c = f % (u32)(C + 1);
    row = __ldg(idx + p);
  };
  float4 pre[NQ];
  u32 row_n, c_n;
  auto issue = [&](u64 p0n, u32 rown) {
    const int nr = end - p0n < 32 ? (int)(end - p0n) : 32;
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
      const int cc = lane + 32 * k, r = cc / NQ, q = cc % NQ;
      const u32 rr = __shfl_sync(FULL, rown, r);
      if (r < nr) pre[k] = LOADX(x4 + (size_t)rr * NQ + q);
    }
  };
  u64 p0 = beg + (u64)warp * 32;
  meta(p0 + lane, row_n, c_n);
  if (p0 < end) issue(p0, row_n);
  for (; p0 < end; p0 += WARPS * 32) {
    const u32 row = row_n, c = c_n;
    const int nrows = end - p0 < 32 ? (int)(end - p0) : 32;
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
      const int cc = lane + 32 * k, r = cc / NQ, q = cc % NQ;
      if (r < nrows) wb[r * NQ + (q ^ SWZ)] = pre[k];
    }
    const u64 p1 = p0 + WARPS * 32;
    if (p1 < end) {
      meta(p1 + lane, row_n, c_n);
      issue(p1, row_n);
    }
    __syncwarp();
    float v[N];
    {
      const int r = lane;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const float4 a = wb[r * NQ + (q ^ SWZ)];
        v[4 * q] = a.x; v[4 * q + 1] = a.y; v[4 * q + 2] = a.z; v[4 * q + 3] = a.w;
      }
    }
    switch (c) {
)CUDA";

const char* kEpilogue = R"CUDA(
      default: break;  // invalid class id: the row passes through unchanged (error flagged)
    }
    {
      const int r = lane;
#pragma unroll
      for (int q = 0; q < NQ; ++q) wb[r * NQ + (q ^ SWZ)] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
      const int cc = lane + 32 * k, r = cc / NQ, q = cc % NQ;
      const u32 rr = __shfl_sync(FULL, row, r);
      if (r < nrows) __stcs(y4 + (size_t)rr * NQ + q, wb[r * NQ + (q ^ SWZ)]);
    }
    __syncwarp();
  }
}
)CUDA";

// Straight-line body of one class in SSA form: every butterfly defines two new values, gathers
// only rename (the generator tracks which value holds logical sample i), so the front end sees
// scalar code with no arrays to promote. Reads and finally rewrites v[0..n).
void emit_body(std::ostringstream& o, const ClassProgram& pr, int n, bool standard) {
  std::vector<std::string> cur(n);
  for (int i = 0; i < n; ++i) cur[i] = "v[" + std::to_string(i) + "]";
  int k = 0;
  auto fresh = [&]() { return "t" + std::to_string(k++); };
  for (const ProgOp& op : pr.ops) {
    if (op.kind == 0) {
      const std::string a = cur[op.m], b = cur[op.n], ym = fresh(), yn = fresh();
      if (!standard)  // a' = a + t1 b ; b' = b - t2 a   (op.b = -t2)
        o << "const float " << ym << "=fmaf(" << b << "," << lit(op.a) << "," << a << ");const float "
          << yn << "=fmaf(" << a << "," << lit(op.b) << "," << b << ");\n";
      else  // y_m = c a + s b ; y_n = c b - s a   (givens.hpp:44-47)
        o << "const float " << ym << "=fmaf(" << a << "," << lit(op.a) << "," << b << "*" << lit(op.b)
          << ");const float " << yn << "=fmaf(" << b << "," << lit(op.a) << ",-(" << a << "*"
          << lit(op.b) << "));\n";
      cur[op.m] = ym;
      cur[op.n] = yn;
    } else if (op.kind == 1) {
      const auto& g = pr.gathers[op.arg];
      std::vector<std::string> nxt(n);
      for (int i = 0; i < n; ++i) nxt[i] = cur[g[i]];
      cur.swap(nxt);
    } else {
      for (int i = 0; i < n; ++i) {
        const std::string t = fresh();
        o << "const float " << t << "=" << cur[i] << "*" << lit(pr.scales[i]) << ";";
        cur[i] = t;
      }
      o << "\n";
    }
  }
  // all samples were rewritten by the first pass, so these assignments never read an
  // already-overwritten input
  for (int i = 0; i < n; ++i) o << "v[" << i << "]=" << cur[i] << ";";
  o << "\n";
}

std::string generate(int log2n, int classes, int warps, int minb, bool standard,
                     const std::vector<ClassProgram>& progs) {
  const int n = 1 << log2n;
  std::ostringstream o;
  o << "#define LOADX __ldg\n";
  o << "#define N " << n << "\n#define NQ " << n / 4 << "\n#define WARPS " << warps
    << "\n#define MINB " << minb << "\n#define SWZ " << kSwizzle[log2n - 2] << "\n";
  o << kPrologue;
  for (int c = 0; c < classes; ++c) {
    o << "      case " << c << ": {\n";
    emit_body(o, progs[c], n, standard);
    o << "      } break;\n";
  }
  o << kEpilogue;
  return o.str();
}

// ---- per-class kernels (plan path "clsjit") -------------------------------------------------
// One kernel per class and direction, launched over that class's bucketed run (the launch chain
// of hygt_cls.cuh): the class body above between a cp.async row stage-in and a coalesced
// stage-out through a per-warp slot area. One warp per CTA, one row per lane.
const char* kClsPrologue = R"CUDA(
typedef unsigned int u32;
typedef unsigned long long u64;
#define RS (NQ + 1)
extern "C" __global__ void __launch_bounds__(32, MINB)
KNAME(const float* __restrict__ x, float* __restrict__ y, const u32* __restrict__ idx,
      const u32* __restrict__ seg_end, u32 bin, u32 copy_bin) {
  __shared__ __align__(16) float4 slot[32 * RS];
  __shared__ u32 s_row[32];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x;
  const u64 beg = bin ? __ldg(seg_end + bin - 1) : 0u;
  const u64 end = __ldg(seg_end + bin);
  const u64 nb = (end - beg + 31) / 32;
  auto row_id = [&](u64 b) -> u32 {
    const u64 p = beg + b * 32 + lane;
    return b < nb && p < end ? __ldg(idx + p) : 0xffffffffu;
  };
  const u32 slot_s = (u32)__cvta_generic_to_shared(slot);
  u32 id_next = row_id(blockIdx.x);
  for (u64 b = blockIdx.x; b < nb; b += gridDim.x) {
    __syncwarp();
    s_row[lane] = id_next;
    id_next = row_id(b + gridDim.x);
    __syncwarp();
#pragma unroll
    for (int i0 = 0; i0 < 32; i0 += 32 / NQ) {
      const int i = i0 + lane / NQ, q = lane % NQ;
      const u32 row = s_row[i];
      if (row != 0xffffffffu)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(slot_s + (u32)(i * RS + q) * 16u),
                     "l"(x + (size_t)row * N + q * 4) : "memory");
    }
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    float v[N];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const float4 a = slot[lane * RS + q];
      v[4 * q] = a.x; v[4 * q + 1] = a.y; v[4 * q + 2] = a.z; v[4 * q + 3] = a.w;
    }
    if (id_next != 0xffffffffu) {  // the next batch's rows: in L2 by the time this one is done
#if PFMODE == 1
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(x + (size_t)id_next * N), "n"(N * 4) : "memory");
#elif PFMODE == 2
#pragma unroll
      for (int l = 0; l < (N * 4 + 127) / 128; ++l)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(x + (size_t)id_next * N + l * 32) : "memory");
#endif
    }
    {
)CUDA";

const char* kClsEpilogue = R"CUDA(
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) slot[lane * RS + q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    __syncwarp();
#pragma unroll
    for (int i0 = 0; i0 < 32; i0 += 32 / NQ) {
      const int i = i0 + lane / NQ, q = lane % NQ;
      const u32 row = s_row[i];
      if (row != 0xffffffffu) __stcs((float4*)(y + (size_t)row * N) + q, slot[i * RS + q]);
    }
  }
  if (copy_bin) {  // rows with invalid class ids pass through (hygt_bucket flags them)
    const u64 e2 = __ldg(seg_end + bin + 1);
    for (u64 p = end + (u64)blockIdx.x * (32 / NQ) + lane / NQ; p < e2; p += (u64)gridDim.x * (32 / NQ)) {
      const u32 row = __ldg(idx + p);
      ((float4*)(y + (size_t)row * N))[lane % NQ] = ((const float4*)(x + (size_t)row * N))[lane % NQ];
    }
  }
  // complete only after the previous class grid: the last grid's completion implies the chain's
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
#undef KNAME
)CUDA";

const char* kClsProloguePTX = R"CUDA(
typedef unsigned int u32;
typedef unsigned long long u64;
#define RS (NQ + 1)
extern "C" __global__ void __launch_bounds__(32, MINB)
KNAME(const float* __restrict__ x, float* __restrict__ y, const u32* __restrict__ idx,
      const u32* __restrict__ seg_end, u32 bin, u32 copy_bin) {
  __shared__ __align__(16) float4 slot[32 * RS];
  __shared__ u32 s_row[32];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x;
  const u64 beg = bin ? __ldg(seg_end + bin - 1) : 0u;
  const u64 end = __ldg(seg_end + bin);
  const u64 nb = (end - beg + 31) / 32;
  auto row_id = [&](u64 b) -> u32 {
    const u64 p = beg + b * 32 + lane;
    return b < nb && p < end ? __ldg(idx + p) : 0xffffffffu;
  };
  const u32 slot_s = (u32)__cvta_generic_to_shared(slot);
  u32 id_next = row_id(blockIdx.x);
  for (u64 b = blockIdx.x; b < nb; b += gridDim.x) {
    __syncwarp();
    s_row[lane] = id_next;
    id_next = row_id(b + gridDim.x);
    __syncwarp();
#pragma unroll
    for (int i0 = 0; i0 < 32; i0 += 32 / NQ) {
      const int i = i0 + lane / NQ, q = lane % NQ;
      const u32 row = s_row[i];
      if (row != 0xffffffffu)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(slot_s + (u32)(i * RS + q) * 16u),
                     "l"(x + (size_t)row * N + q * 4) : "memory");
    }
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    const u32 rb = slot_s + (u32)lane * (RS * 16u);  // this lane's row: the PTX body reads and rewrites it
    if (id_next != 0xffffffffu) {  // the next batch's rows: in L2 by the time this one is done
#if PFMODE == 1
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(x + (size_t)id_next * N), "n"(N * 4) : "memory");
#elif PFMODE == 2
#pragma unroll
      for (int l = 0; l < (N * 4 + 127) / 128; ++l)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(x + (size_t)id_next * N + l * 32) : "memory");
#endif
    }
    {
)CUDA";

const char* kClsEpiloguePTX = R"CUDA(
    }
    __syncwarp();
#pragma unroll
    for (int i0 = 0; i0 < 32; i0 += 32 / NQ) {
      const int i = i0 + lane / NQ, q = lane % NQ;
      const u32 row = s_row[i];
      if (row != 0xffffffffu) __stcs((float4*)(y + (size_t)row * N) + q, slot[i * RS + q]);
    }
  }
  if (copy_bin) {  // rows with invalid class ids pass through (hygt_bucket flags them)
    const u64 e2 = __ldg(seg_end + bin + 1);
    for (u64 p = end + (u64)blockIdx.x * (32 / NQ) + lane / NQ; p < e2; p += (u64)gridDim.x * (32 / NQ)) {
      const u32 row = __ldg(idx + p);
      ((float4*)(y + (size_t)row * N))[lane % NQ] = ((const float4*)(x + (size_t)row * N))[lane % NQ];
    }
  }
  // complete only after the previous class grid: the last grid's completion implies the chain's
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
#undef KNAME
)CUDA";


// Source of one class's two kernels (hygt_cls_f, hygt_cls_i).
void emit_body_ptx(std::ostringstream& o, const ClassProgram& pr, int n, bool standard);

// ptx: -1 = HYGT_CLS_PTX decides, 0 / 1 = C++ / PTX class bodies
std::string generate_class(int log2n, int minb, bool standard, const ClassProgram& fwd, const ClassProgram& inv,
                           int ptx_mode = -1) {
  const int n = 1 << log2n;
  std::ostringstream o;
  o << "#define N " << n << "\n#define NQ " << n / 4 << "\n#define MINB " << minb << "\n";
  // next-batch L2 prefetch, measured per row length (profiles/r01/cls_experiments.log): the bulk
  // prefetch (a uniform loop of UBLKPF) pays off for 256 B rows, per-lane line prefetches for 128 B
  o << "#define PFMODE " << knob("HYGT_CLS_PF", n >= 64 ? 1 : 2) << "\n";
  // PTX bodies (HYGT_CLS_PTX=1) skip the NVVM pass: 0.7 s instead of 2.5 s per class, but the
  // N = 64 kernels run 15% slower than NVVM's (profiles/r01/cls_experiments.log), so opt-in
  const bool ptx = ptx_mode >= 0 ? ptx_mode == 1 : env_on("HYGT_CLS_PTX");
  for (int d = 0; d < 2; ++d) {
    o << "#define KNAME " << (d == 0 ? "hygt_cls_f" : "hygt_cls_i") << "\n"
      << (ptx ? kClsProloguePTX : kClsPrologue);
    if (ptx)
      emit_body_ptx(o, d == 0 ? fwd : inv, n, standard);
    else
      emit_body(o, d == 0 ? fwd : inv, n, standard);
    o << (ptx ? kClsEpiloguePTX : kClsEpilogue);
  }
  return o.str();
}

// ---- per-class fixed-point kernels (fixed plans, N = 16 / 32 / 64) -------------------------
// Same chain and row movement as above with int64 rows: y_m = (c a + s b + 2^(p-1)) >> p,
// y_n = (c b - s a + 2^(p-1)) >> p (fixedpoint.hpp:170-176) with c, s as IMAD.WIDE immediates
// (the TrigTable lookups and the inverse's code negation done here on the host), permutations
// as register renames. Values are int32 in registers: |input| <= 2^20 is checked per row
// (fixedpoint.hpp:145-150); the plan builds these kernels only when fixed_int32_safe()
// (hygt_capi.cu) proves every rounded butterfly stays below 2^30 for its codes and R * log2N,
// so the 2^46 overflow test cannot fire. A row with an
// out-of-range input is written back unchanged (as int32) and reported through *err as
// (row << 3 | 1); the host turns the minimum into the first failing row.
const char* kFxPrologue = R"CUDA(
typedef unsigned int u32;
typedef unsigned long long u64;
typedef long long i64;
#define RS (NQ + 1)
#define FXS_(v) #v
#define FXS(v) FXS_(v)
// d = (a c + b s + 2^(p-1)) >> p, low word (|d| < 2^30): two IMAD.WIDE with immediates + a funnel shift
#define FX(d, a, c, b, s)                                                                          \
  asm("{.reg .s64 t;.reg .u32 l,h;mad.wide.s32 t,%1," #c "," FXS(RND) ";mad.wide.s32 t,%2," #s   \
      ",t;mov.b64 {l,h},t;shf.r.clamp.b32 %0,l,h," FXS(PREC) ";}"                                  \
      : "=r"(d) : "r"(a), "r"(b))
extern "C" __global__ void __launch_bounds__(32, MINB)
KNAME(const i64* __restrict__ x, i64* __restrict__ y, const u32* __restrict__ idx,
      const u32* __restrict__ seg_end, u32 bin, u64 count, u64* err) {
  __shared__ __align__(16) longlong2 slot[32 * RS];
  __shared__ u32 s_row[32];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x;
  const u64 beg = idx ? (bin ? __ldg(seg_end + bin - 1) : 0u) : 0u;
  const u64 end = idx ? __ldg(seg_end + bin) : count;
  const u64 nb = (end - beg + 31) / 32;
  auto row_id = [&](u64 b) -> u32 {
    const u64 p = beg + b * 32 + lane;
    return b < nb && p < end ? (idx ? __ldg(idx + p) : (u32)p) : 0xffffffffu;
  };
  const u32 slot_s = (u32)__cvta_generic_to_shared(slot);
  u32 id_next = row_id(blockIdx.x);
  for (u64 b = blockIdx.x; b < nb; b += gridDim.x) {
    __syncwarp();
    s_row[lane] = id_next;
    id_next = row_id(b + gridDim.x);
    __syncwarp();
#pragma unroll
    for (int i0 = 0; i0 < 32; i0 += (32 / NQ > 0 ? 32 / NQ : 1)) {
#pragma unroll
      for (int qq = 0; qq < (NQ > 32 ? NQ / 32 : 1); ++qq) {
        const int i = i0 + (NQ >= 32 ? 0 : lane / NQ), q = NQ >= 32 ? lane + 32 * qq : lane % NQ;
        const u32 row = s_row[i];
        if (row != 0xffffffffu)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(slot_s + (u32)(i * RS + q) * 16u),
                       "l"(x + (size_t)row * N + q * 2) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    int v[N];
    bool bad = false;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const longlong2 a = slot[lane * RS + q];
      bad |= a.x > (1 << 20) || a.x < -(1 << 20) || a.y > (1 << 20) || a.y < -(1 << 20);
      v[2 * q] = (int)a.x; v[2 * q + 1] = (int)a.y;
    }
    if (id_next != 0xffffffffu) {  // the next batch's rows: in L2 by the time this one is done
#if PFMODE == 1
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(x + (size_t)id_next * N), "n"(N * 8) : "memory");
#elif PFMODE == 2
#pragma unroll
      for (int l = 0; l < (N * 8 + 127) / 128; ++l)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(x + (size_t)id_next * N + l * 16) : "memory");
#endif
    }
    if (!bad) {
)CUDA";

const char* kFxEpilogue = R"CUDA(
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) slot[lane * RS + q] = make_longlong2(v[2 * q], v[2 * q + 1]);
    if (bad && s_row[lane] != 0xffffffffu) atomicMin(err, ((u64)s_row[lane] << 3) | 1u);
    __syncwarp();
#pragma unroll
    for (int i0 = 0; i0 < 32; i0 += (32 / NQ > 0 ? 32 / NQ : 1)) {
#pragma unroll
      for (int qq = 0; qq < (NQ > 32 ? NQ / 32 : 1); ++qq) {
        const int i = i0 + (NQ >= 32 ? 0 : lane / NQ), q = NQ >= 32 ? lane + 32 * qq : lane % NQ;
        const u32 row = s_row[i];
        if (row != 0xffffffffu) __stcs((longlong2*)(y + (size_t)row * N) + q, slot[i * RS + q]);
      }
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
#undef KNAME
)CUDA";

struct FxOp {
  uint8_t kind;  // 0 butterfly, 1 gather
  uint16_t m, n;
  int32_t c, s;
  uint32_t arg;
};

// Execution-order program of one class and direction, as fixed_row_kernel runs it.
std::vector<FxOp> fixed_program(int log2n, int rounds, const uint16_t* codes_c, const int32_t* ct,
                                const int32_t* sn, uint32_t code_mask, const std::vector<std::vector<int>>& g,
                                bool fwd) {
  const int half = 1 << (log2n - 1);
  std::vector<FxOp> ops;
  auto gather = [&](int k) {
    if (!g[k].empty()) ops.push_back(FxOp{1, 0, 0, 0, 0, (uint32_t)k});
  };
  gather(0);
  for (int k = 0; k < rounds; ++k) {
    const int r = fwd ? k : rounds - 1 - k;
    for (int pp = 0; pp < log2n; ++pp) {
      const int d = fwd ? pp : log2n - 1 - pp;
      const uint32_t kk = 1u << d;
      const size_t base = ((size_t)r * log2n + d) * half;  // model.hpp:77-79
      for (int j = 0; j < half; ++j) {
        const uint32_t m = j + (j & (0u - kk)), n = m + kk;  // hypercube.hpp:73-74
        uint32_t code = codes_c[base + j];
        if (!fwd) code = (0u - code) & code_mask;  // fixedpoint.hpp:170
        ops.push_back(FxOp{0, (uint16_t)m, (uint16_t)n, ct[code], sn[code], 0});
      }
    }
    gather(k + 1);
  }
  return ops;
}

void emit_fixed_body(std::ostringstream& o, const std::vector<FxOp>& ops, const std::vector<std::vector<int>>& g,
                     int n) {
  std::vector<std::string> cur(n);
  for (int i = 0; i < n; ++i) cur[i] = "v[" + std::to_string(i) + "]";
  int k = 0;
  for (const FxOp& op : ops) {
    if (op.kind == 0) {
      const std::string a = cur[op.m], b = cur[op.n];
      const std::string ym = "t" + std::to_string(k++), yn = "t" + std::to_string(k++);
      o << "int " << ym << "," << yn << ";FX(" << ym << "," << a << "," << op.c << "," << b << "," << op.s
        << ");FX(" << yn << "," << b << "," << op.c << "," << a << "," << -(int64_t)op.s << ");\n";
      cur[op.m] = ym;
      cur[op.n] = yn;
    } else {
      const auto& gg = g[op.arg];
      std::vector<std::string> nxt(n);
      for (int i = 0; i < n; ++i) nxt[i] = cur[gg[i]];
      cur.swap(nxt);
    }
  }
  for (int i = 0; i < n; ++i) o << "v[" << i << "]=" << cur[i] << ";";
  o << "\n";
}

std::string hexf(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  char b[16];
  std::snprintf(b, sizeof b, "0f%08X", u);
  return b;
}

// The class body as one PTX block over the lane's row in its slot (operand %0: shared address):
// the front end never sees the straight-line code, so NVRTC time is ptxas time.
void emit_body_ptx(std::ostringstream& o, const ClassProgram& pr, int n, bool standard) {
  std::ostringstream b;
  int nreg = 0;
  auto R = [](int r) { return "%%hv" + std::to_string(r); };
  std::vector<int> cur(n);
  for (int q = 0; q < n / 4; ++q) {
    b << "ld.shared.v4.f32 {" << R(nreg) << "," << R(nreg + 1) << "," << R(nreg + 2) << "," << R(nreg + 3) << "}, [%0+"
      << q * 16 << "];\n";
    for (int t = 0; t < 4; ++t) cur[4 * q + t] = nreg++;
  }
  for (const ProgOp& op : pr.ops) {
    if (op.kind == 0) {
      const int a = cur[op.m], bb = cur[op.n];
      if (!standard) {  // a' = a + t1 b ; b' = b - t2 a   (op.b = -t2)
        b << "fma.rn.f32 " << R(nreg) << ", " << R(bb) << ", " << hexf(op.a) << ", " << R(a) << ";\n"
          << "fma.rn.f32 " << R(nreg + 1) << ", " << R(a) << ", " << hexf(op.b) << ", " << R(bb) << ";\n";
        cur[op.m] = nreg;
        cur[op.n] = nreg + 1;
        nreg += 2;
      } else {  // y_m = c a + s b ; y_n = c b - s a   (givens.hpp:44-47)
        b << "mul.rn.f32 " << R(nreg) << ", " << R(bb) << ", " << hexf(op.b) << ";\n"
          << "fma.rn.f32 " << R(nreg + 1) << ", " << R(a) << ", " << hexf(op.a) << ", " << R(nreg) << ";\n"
          << "mul.rn.f32 " << R(nreg + 2) << ", " << R(a) << ", " << hexf(-op.b) << ";\n"
          << "fma.rn.f32 " << R(nreg + 3) << ", " << R(bb) << ", " << hexf(op.a) << ", " << R(nreg + 2) << ";\n";
        cur[op.m] = nreg + 1;
        cur[op.n] = nreg + 3;
        nreg += 4;
      }
    } else if (op.kind == 1) {
      const auto& g = pr.gathers[op.arg];
      std::vector<int> nxt(n);
      for (int i = 0; i < n; ++i) nxt[i] = cur[g[i]];
      cur.swap(nxt);
    } else {
      for (int i = 0; i < n; ++i) {
        b << "mul.rn.f32 " << R(nreg) << ", " << R(cur[i]) << ", " << hexf(pr.scales[i]) << ";\n";
        cur[i] = nreg++;
      }
    }
  }
  for (int q = 0; q < n / 4; ++q)
    b << "st.shared.v4.f32 [%0+" << q * 16 << "], {" << R(cur[4 * q]) << "," << R(cur[4 * q + 1]) << ","
      << R(cur[4 * q + 2]) << "," << R(cur[4 * q + 3]) << "};\n";
  o << "asm volatile(\"{\\n.reg .f32 %%hv<" << nreg << ">;\\n\"\n";
  std::istringstream lines(b.str());
  std::string ln;
  while (std::getline(lines, ln)) o << "\"" << ln << "\\n\"\n";
  o << "\"}\" :: \"r\"(rb) : \"memory\");\n";
}

std::mutex g_cache_mu;
std::unordered_map<std::string, std::vector<char>> g_cubin_cache;  // source -> cubin

int compile(const std::string& src, std::vector<char>& cubin, std::string& log) {
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cubin_cache.find(src);
    if (it != g_cubin_cache.end()) {
      cubin = it->second;
      return 0;
    }
  }
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "hygt_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
    return 1;
  const char* opts[] = {"--gpu-architecture=sm_100a", "-default-device", "-lineinfo", "--std=c++17",
                        "-DNDEBUG"};
  const nvrtcResult r = nvrtcCompileProgram(prog, (int)(sizeof(opts) / sizeof(opts[0])), opts);
  size_t ls = 0;
  nvrtcGetProgramLogSize(prog, &ls);
  log.resize(ls);
  if (ls) nvrtcGetProgramLog(prog, &log[0]);
  if (r != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    return 1;
  }
  size_t cs = 0;
  nvrtcGetCUBINSize(prog, &cs);
  cubin.resize(cs);
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  if (g_cubin_cache.size() >= 512) g_cubin_cache.clear();  // bound the process's cache (~0.5 MB per class)
  g_cubin_cache.emplace(src, cubin);
  return 0;
}

}  // namespace

int jit_compile_only(int log2n, int rounds, int classes, const double* angles,
                     const uint16_t* perms, uint32_t mask, bool standard, size_t* cubin_bytes,
                     std::string& err) {
  const int warps = log2n >= 6 ? 8 : 16, minb = log2n >= 6 ? 1 : 2;
  *cubin_bytes = 0;
  for (int d = 0; d < 2; ++d) {
    std::vector<ClassProgram> progs;
    if (!build_programs(log2n, rounds, classes, angles, perms, mask, d == 0, standard, progs)) {
      err = "unsafe";
      return 3;
    }
    std::vector<char> cubin;
    std::string log;
    if (compile(generate(log2n, classes, warps, minb, standard, progs), cubin, log)) {
      err = log;
      return 5;
    }
    err += log;
    *cubin_bytes += cubin.size();
  }
  return 0;
}

size_t jit_smem_bytes(int log2n, int classes, int warps, int tile_rows) {
  (void)classes;
  (void)tile_rows;
  return (size_t)warps * 32 * (1u << log2n) * 4;  // per-warp transpose buffers
}

bool jit_supported(int log2n, int classes, int rounds) {
  if (log2n < 2 || log2n > 5) return false;
  // Measured: with many classes the class-bucketed 64-128 B row gathers this path
  // needs cost more than its immediates save; the tile kernel serves those plans.
  if (classes > 4) return false;
  // NVRTC time grows superlinearly with the kernel body: ~16 s for N=16 x 35 classes x 3
  // rounds (both directions), minutes for N=32 x 35 x 3. Bound the total butterflies per kernel.
  const size_t butterflies = (size_t)classes * rounds * log2n * (1u << (log2n - 1));
  return butterflies <= (size_t)35 * 3 * 4 * 8;
}

int jit_build(int log2n, int rounds, int classes, const double* angles, const uint16_t* perms,
              uint32_t mask, bool standard, JitKernels& out, std::string& err) {
  const int warps = log2n >= 6 ? 8 : 16, minb = log2n >= 6 ? 1 : 2;
  out.warps = warps;
  out.tile_rows = 0;
  // generate + compile both directions concurrently (NVRTC is thread safe per program)
  std::vector<char> cubins[2];
  std::string logs[2];
  int status[2] = {0, 0};
  auto work = [&](int d) {
    std::vector<ClassProgram> progs;
    if (!build_programs(log2n, rounds, classes, angles, perms, mask, d == 0, standard, progs)) {
      status[d] = 3;
      logs[d] = "jit: scale-folded program unsafe";
      return;
    }
    if (compile(generate(log2n, classes, warps, minb, standard, progs), cubins[d], logs[d])) {
      status[d] = 5;
      logs[d] = "jit: NVRTC compilation failed: " + logs[d].substr(0, 2000);
    }
  };
  std::thread th(work, 1);
  work(0);
  th.join();
  for (int d = 0; d < 2; ++d) {
    if (status[d]) {
      err = logs[d];
      return status[d];
    }
    const std::vector<char>& cubin = cubins[d];
    if (cudaLibraryLoadData(&out.lib[d], cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess ||
        cudaLibraryGetKernel(&out.fn[d], out.lib[d], "hygt_jit_kernel") != cudaSuccess) {
      err = "jit: cannot load the compiled module";
      return 5;
    }
    out.smem = jit_smem_bytes(log2n, classes, warps, out.tile_rows);
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaKernelSetAttributeForDevice(out.fn[d], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)out.smem, dev) != cudaSuccess) {
      err = "jit: cannot set shared memory size";
      return 5;
    }
  }
  out.ok = true;
  return 0;
}

void jit_release(JitKernels& k) {
  for (int d = 0; d < 2; ++d)
    if (k.lib[d]) cudaLibraryUnload(k.lib[d]);
  k = JitKernels{};
}

int jit_launch(const JitKernels& k, int dir, const float* x, float* y, const uint32_t* idx,
               const uint32_t* seg_end, uint32_t nseg, uint64_t count, int classes, int num_sms,
               cudaStream_t st) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)k.fn[dir], k.warps * 32, k.smem) != cudaSuccess || occ < 1)
    occ = 1;
  cudaGetLastError();
  const uint64_t step = (uint64_t)k.warps * 32;
  uint64_t grid = std::min<uint64_t>((uint64_t)num_sms * occ, (count + step - 1) / step);
  if (grid < 1) grid = 1;
  uint64_t span = (count + grid - 1) / grid;
  span = (span + step - 1) / step * step;
  void* args[] = {(void*)&x, (void*)&y, (void*)&idx, (void*)&seg_end, (void*)&nseg, (void*)&count,
                  (void*)&classes, (void*)&span};
  return cudaLaunchKernel((const void*)k.fn[dir], dim3((unsigned)grid), dim3(k.warps * 32), args, k.smem, st) == cudaSuccess ? 0 : 5;
}

// Compiles one NVRTC program per class (kernels hygt_cls_f / hygt_cls_i) on all host threads
// and loads them; out.grid = one warp-CTA per resident slot on every SM.
int load_class_modules(const std::vector<std::string>& srcs, JitClsKernels& out, std::string& err) {
  const int classes = (int)srcs.size();
  std::vector<std::vector<char>> cubins(classes);
  std::vector<std::string> logs(classes);
  std::vector<int> status(classes, 0);
  std::atomic<int> next{0};
  auto worker = [&]() {
    for (int c; (c = next.fetch_add(1)) < classes;)
      if (compile(srcs[c], cubins[c], logs[c])) status[c] = 5;
  };
  const int nt = std::max(1, std::min<int>(classes, (int)std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(worker);
  worker();
  for (auto& t : pool) t.join();
  out.lib.assign(classes, nullptr);
  out.fn[0].assign(classes, nullptr);
  out.fn[1].assign(classes, nullptr);
  for (int c = 0; c < classes; ++c) {
    if (status[c]) {
      err = "jit: NVRTC compilation failed: " + logs[c].substr(0, 2000);
      return 5;
    }
    if (cudaLibraryLoadData(&out.lib[c], cubins[c].data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess ||
        cudaLibraryGetKernel(&out.fn[0][c], out.lib[c], "hygt_cls_f") != cudaSuccess ||
        cudaLibraryGetKernel(&out.fn[1][c], out.lib[c], "hygt_cls_i") != cudaSuccess) {
      err = "jit: cannot load the compiled module";
      return 5;
    }
  }
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)out.fn[0][0], out.threads, 0) != cudaSuccess || occ < 1)
    occ = 1;
  cudaGetLastError();
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  out.grid = (unsigned)(sms * occ);
  out.ok = true;
  return 0;
}



// One NVRTC module per class: plans with very many classes would spend minutes compiling, so the
// per-class chains are limited to HYGT_CLS_JIT_MAX_CLASSES (default 64) classes.
int max_jit_classes() { return knob("HYGT_CLS_JIT_MAX_CLASSES", 64); }

bool jit_cls_supported(int log2n, int classes, int rounds) {
  if (classes > max_jit_classes()) return false;
  // N = 16 rows (64 B) are half a 128 B line: gathered per class they cost twice the staged
  // kernel's time (profiles/r01/cls_experiments.log), so N = 16 is opt-in (experiments only).
  return log2n >= 4 && log2n <= 6 && classes >= 2 && rounds >= 1 && rounds <= 8 &&
         (log2n >= 5 || env_on("HYGT_CLS_JIT_SHORT"));
}

int jit_cls_build(int log2n, int rounds, int classes, const double* angles, const uint16_t* perms,
                  uint32_t mask, bool standard, JitClsKernels& out, std::string& err) {
  std::vector<ClassProgram> progs[2];
  for (int d = 0; d < 2; ++d)
    if (!build_programs(log2n, rounds, classes, angles, perms, mask, d == 0, standard, progs[d])) {
      err = "jit: scale-folded program unsafe";
      return 3;
    }
  std::vector<std::string> srcs(classes);
  for (int c = 0; c < classes; ++c) srcs[c] = generate_class(log2n, knob("HYGT_CLS_MINB", 16), standard, progs[0][c], progs[1][c]);
  return load_class_modules(srcs, out, err);
}

void jit_cls_release(JitClsKernels& k) {
  for (cudaLibrary_t l : k.lib)
    if (l) cudaLibraryUnload(l);
  k = JitClsKernels{};
}

int jit_cls_launch(const JitClsKernels& k, int dir, const float* x, float* y, const uint32_t* idx,
                   const uint32_t* seg_end, int classes, cudaStream_t st) {
  for (int c = 0; c < classes; ++c) {
    uint32_t bin = (uint32_t)c, copy_bin = c == classes - 1 ? 1u : 0u;
    void* args[] = {(void*)&x, (void*)&y, (void*)&idx, (void*)&seg_end, (void*)&bin, (void*)&copy_bin};
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(k.grid);
    cfg.blockDim = dim3(k.threads);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = c > 0 ? 1 : 0;  // the first grid follows the bucketing normally
    const cudaKernel_t fn = k.fn[dir][c];
    if (cudaLaunchKernelExC(&cfg, (const void*)fn, args) != cudaSuccess) return 5;
  }
  return 0;
}

bool jit_fixed_supported(int log2n, int rounds, int classes) {
  if (classes > max_jit_classes()) return false;
  return log2n >= 4 && log2n <= 6 && rounds >= 1 && rounds * log2n <= 32 && !env_off("HYGT_FIXED_JIT");
}

int jit_fixed_build(int log2n, int rounds, int classes, int angle_bits, int precision_bits,
                    const uint16_t* codes, const int32_t* ct, const int32_t* sn, const uint16_t* perms,
                    uint32_t perm_mask, JitClsKernels& out, std::string& err) {
  const int n = 1 << log2n;
  const size_t a = (size_t)rounds * log2n * n / 2;
  const uint32_t code_mask = (1u << angle_bits) - 1u;
  std::vector<std::string> srcs(classes);
  for (int c = 0; c < classes; ++c) {
    std::ostringstream o;
    o << "#define PFMODE " << knob("HYGT_FIXED_PF", n >= 64 ? 0 : 2) << "\n";
    o << "#define N " << n << "\n#define NQ " << n / 2 << "\n#define MINB 12\n#define PREC " << precision_bits
      << "\n#define RND " << (1ll << (precision_bits - 1)) << "\n";
    for (int d = 0; d < 2; ++d) {
      uint64_t gm = 0;
      const auto g = exec_gathers(log2n, rounds, perms ? perms + (size_t)c * rounds * n : nullptr, perm_mask,
                                  d == 0, &gm);
      const auto ops = fixed_program(log2n, rounds, codes + (size_t)c * a, ct, sn, code_mask, g, d == 0);
      o << "#define KNAME " << (d == 0 ? "hygt_cls_f" : "hygt_cls_i") << "\n" << kFxPrologue;
      emit_fixed_body(o, ops, g, n);
      o << kFxEpilogue;
    }
    srcs[c] = o.str();
  }
  return load_class_modules(srcs, out, err);
}

int jit_fixed_launch(const JitClsKernels& k, int dir, const int64_t* x, int64_t* y, const uint32_t* idx,
                     const uint32_t* seg_end, int classes, uint64_t count, unsigned long long* err,
                     cudaStream_t st) {
  const int launches = idx ? classes : 1;
  for (int c = 0; c < launches; ++c) {
    uint32_t bin = (uint32_t)c;
    void* args[] = {(void*)&x, (void*)&y, (void*)&idx, (void*)&seg_end, (void*)&bin, (void*)&count, (void*)&err};
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(k.grid);
    cfg.blockDim = dim3(32);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = c > 0 ? 1 : 0;
    if (cudaLaunchKernelExC(&cfg, (const void*)k.fn[dir][c], args) != cudaSuccess) return 5;
  }
  return 0;
}

}  // namespace hygt_gpu

// Debug hook (not in the public header; used by the CPU test suite): generates and compiles class
// 0's per-class kernels without touching a GPU and returns the cubin size. kind 0: float
// (N = 32 / 64 C++ bodies, N = 256 PTX warp-pair bodies; ptx != 0 selects PTX bodies for N <= 64),
// kind 1: fixed point (8-bit codes, p = 10). Returns 0 or the failing status.
extern "C" int hygt_debug_jit_compile(int kind, int log2n, int rounds, const double* angles,
                                      const uint16_t* codes, const uint16_t* perms, uint32_t mask, int ptx,
                                      unsigned long long* cubin_bytes) {
  using namespace hygt_gpu;
  std::string src;
  if (kind == 0) {
    std::vector<ClassProgram> progs[2];
    for (int d = 0; d < 2; ++d)
      if (!build_programs(log2n, rounds, 1, angles, perms, mask, d == 0, false, progs[d])) return 3;
    if (log2n > 6) return 1;  // per-class kernels: N = 16 / 32 / 64
    src = generate_class(log2n, 16, false, progs[0][0], progs[1][0], ptx ? 1 : 0);
  } else {
    const int n = 1 << log2n;
    std::vector<int32_t> ct(256), sn(256);
    for (int q = 0; q < 256; ++q) {
      const double ang = 2.0 * 3.14159265358979323846 * q / 256.0;
      ct[q] = (int32_t)std::lround(std::cos(ang) * 1024.0);
      sn[q] = (int32_t)std::lround(std::sin(ang) * 1024.0);
    }
    std::ostringstream o;
    o << "#define PFMODE 1\n#define N " << n << "\n#define NQ " << n / 2 << "\n#define MINB 12\n#define PREC 10\n#define RND 512\n";
    for (int d = 0; d < 2; ++d) {
      uint64_t gm = 0;
      const auto g = exec_gathers(log2n, rounds, perms, mask, d == 0, &gm);
      const auto ops = fixed_program(log2n, rounds, codes, ct.data(), sn.data(), 255u, g, d == 0);
      o << "#define KNAME " << (d == 0 ? "hygt_cls_f" : "hygt_cls_i") << "\n" << kFxPrologue;
      emit_fixed_body(o, ops, g, n);
      o << kFxEpilogue;
    }
    src = o.str();
  }
  std::vector<char> cubin;
  std::string log;
  if (compile(src, cubin, log)) return 5;
  if (cubin_bytes) *cubin_bytes = cubin.size();
  return 0;
}
