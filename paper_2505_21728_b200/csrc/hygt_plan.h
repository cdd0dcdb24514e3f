// hygt_plan.h -- host plan builder interface (see hygt_plan.cpp).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cmath>
#include <vector>

#include "layout.h"

namespace hygt_gpu {

struct Float2 {
  float x, y;
};

// One direction's device tables before upload.
struct DirTables {
  std::vector<Float2> coef;    // [C][TPV][stream_len]
  std::vector<uint16_t> gidx;  // [C][R+1][TPV][E] gather sources (element indices)
  uint64_t gmask = 0;          // bit k: gather step k present
  uint32_t stream_len = 0;     // float2 words per lane stream
  double sigma_min = 1.0;      // scale-folded form: smallest running per-sample scale
};

// Input range of the scale-folded form. Its stored values are true / sigma with sigma the
// running per-sample scale, and |true| <= ||x||_2 <= sqrt(N) max|x| (orthogonal passes), so every
// intermediate stays finite in fp32 while max|x| < 2^127 sigma_min / sqrt(N): the plan's input
// limit (hygt_plan_input_limit). The form is used only when that limit is at least
// 2^FAST_FORM_MIN_INPUT_LOG2 (far above residual data); otherwise the standard rotations.
constexpr int FAST_FORM_MIN_INPUT_LOG2 = 40;
inline double fast_sigma_floor(int log2n) {
  return std::ldexp(1.0, FAST_FORM_MIN_INPUT_LOG2 - 127 + (log2n + 1) / 2);
}
inline double fast_input_limit(int log2n, double sigma_min) {
  return std::ldexp(sigma_min, 127 - (log2n + 1) / 2);
}

// One class's transform as straight-line operations in execution order (for code generation):
//   kind 0: butterfly on (m, n) with coefficients (a, b): scale-folded (t1, -t2) or standard (c, s)
//   kind 1: gather new[i] = old[src[i]] (src in ClassProgram::gathers[arg])
//   kind 2: final per-sample scales (ClassProgram::scales)
struct ProgOp {
  uint8_t kind;
  uint16_t m, n;
  float a, b;
  uint32_t arg;
};
struct ClassProgram {
  std::vector<ProgOp> ops;
  std::vector<std::vector<int>> gathers;
  std::vector<float> scales;
};
bool build_programs(int log2n, int rounds, int classes, const double* angles,
                    const uint16_t* perms, uint32_t mask, bool fwd, bool standard,
                    std::vector<ClassProgram>& out);

// Lane-group width (log2 TPV) used for a dimension unless overridden.
int default_lane_log2(int log2n);

// Execution-order gathers of one class: step 0 runs before round slot 0, step k+1 after slot k.
// Forward: step r+1 = P_r. Inverse: step 0 = P_{R-1}^{-1}, step k+1 = P_{R-2-k}^{-1}.
std::vector<std::vector<int>> exec_gathers(int log2n, int rounds, const uint16_t* perms_c,
                                           uint32_t mask, bool fwd, uint64_t* gmask);

// Builds the coefficient/gather streams of one direction. Returns false when the scale-folded
// form was requested but is numerically unsafe for these angles.
bool build_direction(const Layout& ly, int rounds, int classes, const double* angles,
                     const uint16_t* perms, uint32_t mask, bool fwd, bool standard,
                     DirTables& out);


// The class's whole forward transform as one N x N matrix, fp64: column k = forward(e_k) with the
// reference's pass order and per-butterfly cos/sin (transform.hpp:45-66, the gathers after the
// rounds whose mask bit is set as transform.hpp:75-80; transform.hpp:100-117 builds the same
// matrix). out[i * N + k], so y = out . x.
void compose_operator(int log2n, int rounds, const double* angles_c, const uint16_t* perms_c,
                      uint32_t mask, double* out);

}  // namespace hygt_gpu
