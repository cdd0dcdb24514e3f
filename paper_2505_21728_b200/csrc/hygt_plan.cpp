// hygt_plan.cpp -- host-side plan construction (pure C++, no CUDA).
//
// Turns per-class angle tables (HyGTModel, model.hpp:51-96) into the per-lane coefficient
// streams the kernels consume, in exactly their consumption order (layout.h). For every
// butterfly the rotation (c, s) = (cos t, sin t) is evaluated in fp64 from the same expression the
// reference uses (transform.hpp:57-59: t = +-angle, then std::cos / std::sin), then either
//   * stored as fp32 (c, s)                                   -- the standard form, or
//   * folded with the running per-sample scales sigma (fast Givens): the kernel stores
//       a' = a + t1 b,  b' = b - t2 a,  t1 = s sig_n / (c sig_m),  t2 = s sig_m / (c sig_n),
//     and sig_m, sig_n *= c; the true values are sig * stored, so one FFMA per output replaces
//     an FMUL + FFMA. The remaining sig are applied once after the last pass.
// The fast form is exact algebra; it is used only when every c != 0, all |t| <= 2^100 and the
// scales keep the plan's input limit (hygt_plan.h: 2^127 sigma_min / sqrt(N)) at or above 2^40;
// otherwise the plan falls back to the standard form (hygt_plan_algorithm() reports which).
#include "hygt_plan.h"

#include <algorithm>
#include <vector>

#include <cmath>
#include <cstring>

namespace hygt_gpu {

namespace {

struct Coef {
  double a, b;  // (k1, k2) fast form or (c, s) standard form
};

}  // namespace

int default_lane_log2(int log2n) {
  switch (log2n) {
    case 1: case 2: case 3: case 4: case 5: return 0;
    case 6: return 1;
    case 7: return 2;
    default: return 2;
  }
}

std::vector<std::vector<int>> exec_gathers(int log2n, int rounds, const uint16_t* perms_c,
                                           uint32_t mask, bool fwd, uint64_t* gmask) {
  const int n = 1 << log2n;
  std::vector<std::vector<int>> g(rounds + 1);
  *gmask = 0;
  auto perm = [&](int r) { return perms_c + (size_t)r * n; };
  auto inv_of = [&](int r) {
    std::vector<int> out(n);
    for (int i = 0; i < n; ++i) out[perm(r)[i]] = i;  // scatter x[perm[i]] = y[i]
    return out;
  };
  if (!perms_c) return g;
  if (fwd) {
    for (int r = 0; r < rounds; ++r)
      if ((mask >> r) & 1u) {
        g[r + 1].assign(perm(r), perm(r) + n);
        *gmask |= 1ull << (r + 1);
      }
  } else {
    if ((mask >> (rounds - 1)) & 1u) {
      g[0] = inv_of(rounds - 1);
      *gmask |= 1ull;
    }
    for (int k = 0; k + 1 < rounds; ++k) {
      const int r = rounds - 2 - k;
      if ((mask >> r) & 1u) {
        g[k + 1] = inv_of(r);
        *gmask |= 1ull << (k + 1);
      }
    }
  }
  return g;
}

bool build_direction(const Layout& ly, int rounds, int classes, const double* angles,
                     const uint16_t* perms, uint32_t mask, bool fwd, bool standard,
                     DirTables& out) {
  const int n = ly.n(), log2n = ly.log2n, half = n / 2, tpv = ly.tpv(), e = ly.e();
  const size_t a_count = (size_t)rounds * log2n * half;
  const double sig_floor = fast_sigma_floor(log2n);
  out.sigma_min = 1.0;
  uint32_t len = 0;
  for (int p = 0; p < log2n; ++p) len += ly.words_per_pass(standard, p);
  len *= rounds;
  if (!standard) len += e / 2;
  len = (len + 1) & ~1u;
  out.stream_len = len;
  out.coef.assign((size_t)classes * tpv * len, Float2{0.f, 0.f});
  out.gidx.assign((size_t)classes * (rounds + 1) * tpv * e, 0);
  out.gmask = 0;

  std::vector<double> sig(n);
  std::vector<Coef> pass(half);
  std::vector<size_t> cursor(tpv);
  for (int c = 0; c < classes; ++c) {
    const double* ang = angles + (size_t)c * a_count;
    const uint16_t* pc = perms ? perms + (size_t)c * rounds * n : nullptr;
    uint64_t gm = 0;
    const auto gathers = exec_gathers(log2n, rounds, pc, mask, fwd, &gm);
    out.gmask = gm;
    for (int i = 0; i < n; ++i) sig[i] = 1.0;
    for (int t = 0; t < tpv; ++t) cursor[t] = ((size_t)c * tpv + t) * len;

    auto apply_gather = [&](int step) {
      const auto& gsrc = gathers[step];
      if (gsrc.empty()) return;
      std::vector<double> s2(n);
      for (int i = 0; i < n; ++i) s2[i] = sig[gsrc[i]];
      sig.swap(s2);
      for (int t = 0; t < tpv; ++t)
        for (int s = 0; s < e; ++s)
          out.gidx[(((size_t)c * (rounds + 1) + step) * tpv + t) * e + s] =
              (uint16_t)gsrc[ly.elem(t, s)];
    };
    auto put = [&](int t, double x, double y) {
      out.coef[cursor[t]++] = Float2{(float)x, (float)y};
    };

    apply_gather(0);
    for (int k = 0; k < rounds; ++k) {
      const int r = fwd ? k : rounds - 1 - k;
      for (int pp = 0; pp < log2n; ++pp) {
        const int p = fwd ? pp : log2n - 1 - pp;
        const uint32_t kk = 1u << p;
        const size_t base = ((size_t)r * log2n + p) * half;  // model.hpp:77-79
        for (uint32_t j = 0; j < (uint32_t)half; ++j) {
          const uint32_t m = j + (j & (0u - kk)), nn = m + kk;  // hypercube.hpp:73-74
          const double th = fwd ? ang[base + j] : -ang[base + j];  // transform.hpp:57
          const double cs = std::cos(th), sn = std::sin(th);       // transform.hpp:58-59
          if (standard) {
            pass[j] = {cs, sn};
          } else {
            if (cs == 0.0) return false;
            const double k1 = sn * sig[nn] / (cs * sig[m]);
            const double k2 = sn * sig[m] / (cs * sig[nn]);
            sig[m] *= cs;
            sig[nn] *= cs;
            if (!(std::fabs(k1) <= 0x1p100) || !(std::fabs(k2) <= 0x1p100)) return false;
            if (!(std::fabs(sig[m]) >= sig_floor) || !(std::fabs(sig[nn]) >= sig_floor)) return false;
            out.sigma_min = std::min(out.sigma_min, std::min(std::fabs(sig[m]), std::fabs(sig[nn])));
            pass[j] = {k1, k2};
          }
        }
        // Pack in each lane's consumption order (hygt_kernels.cuh, hygt_pass).
        for (int t = 0; t < tpv; ++t) {
          if (ly.cross(p)) {
            for (int q = 0; q < e / 2; ++q) {
              const int i0 = ly.elem(t, 2 * q), i1 = ly.elem(t, 2 * q + 1);
              const int side = (i0 >> p) & 1;  // identical for every sample of this lane
              const int j0 = pair_index(i0 & ~(1 << p), p), j1 = pair_index(i1 & ~(1 << p), p);
              if (!standard) {
                put(t, side ? -pass[j0].b : pass[j0].a, side ? -pass[j1].b : pass[j1].a);
              } else {
                const double sg = side ? -1.0 : 1.0;
                put(t, pass[j0].a, pass[j1].a);
                put(t, sg * pass[j0].b, sg * pass[j1].b);
              }
            }
          } else if (p == 0) {
            for (int q = 0; q < e / 2; ++q) {
              const int m0 = ly.elem(t, 2 * q);
              const int j = pair_index(m0, 0);
              if (!standard) put(t, pass[j].a, -pass[j].b);
              else put(t, pass[j].a, pass[j].b);
            }
          } else {
            const int so = ly.slot_stride(p) / 2;
            for (int a = 0; a < e / 2; ++a) {
              if (a & so) continue;
              const int m0 = ly.elem(t, 2 * a), m1 = ly.elem(t, 2 * a + 1);
              const int j0 = pair_index(m0, p), j1 = pair_index(m1, p);
              if (!standard) {
                put(t, pass[j0].a, pass[j1].a);
                put(t, -pass[j0].b, -pass[j1].b);
              } else {
                put(t, pass[j0].a, pass[j1].a);
                put(t, pass[j0].b, pass[j1].b);
              }
            }
          }
        }
      }
      apply_gather(k + 1);
    }
    if (!standard)
      for (int t = 0; t < tpv; ++t)
        for (int q = 0; q < e / 2; ++q) put(t, sig[ly.elem(t, 2 * q)], sig[ly.elem(t, 2 * q + 1)]);
  }
  return true;
}

bool build_programs(int log2n, int rounds, int classes, const double* angles,
                    const uint16_t* perms, uint32_t mask, bool fwd, bool standard,
                    std::vector<ClassProgram>& out) {
  const int n = 1 << log2n, half = n / 2;
  const size_t a_count = (size_t)rounds * log2n * half;
  out.assign(classes, ClassProgram{});
  std::vector<double> sig(n);
  for (int c = 0; c < classes; ++c) {
    ClassProgram& pr = out[c];
    const double* ang = angles + (size_t)c * a_count;
    const uint16_t* pc = perms ? perms + (size_t)c * rounds * n : nullptr;
    uint64_t gm = 0;
    const auto gathers = exec_gathers(log2n, rounds, pc, mask, fwd, &gm);
    for (int i = 0; i < n; ++i) sig[i] = 1.0;
    auto gather = [&](int step) {
      if (gathers[step].empty()) return;
      std::vector<double> s2(n);
      for (int i = 0; i < n; ++i) s2[i] = sig[gathers[step][i]];
      sig.swap(s2);
      pr.ops.push_back(ProgOp{1, 0, 0, 0.f, 0.f, (uint32_t)pr.gathers.size()});
      pr.gathers.push_back(gathers[step]);
    };
    gather(0);
    for (int k = 0; k < rounds; ++k) {
      const int r = fwd ? k : rounds - 1 - k;
      for (int pp = 0; pp < log2n; ++pp) {
        const int p = fwd ? pp : log2n - 1 - pp;
        const uint32_t kk = 1u << p;
        const size_t base = ((size_t)r * log2n + p) * half;  // model.hpp:77-79
        for (uint32_t j = 0; j < (uint32_t)half; ++j) {
          const uint32_t m = j + (j & (0u - kk)), nn = m + kk;  // hypercube.hpp:73-74
          const double th = fwd ? ang[base + j] : -ang[base + j];  // transform.hpp:57
          const double cs = std::cos(th), sn = std::sin(th);       // transform.hpp:58-59
          if (standard) {
            pr.ops.push_back(ProgOp{0, (uint16_t)m, (uint16_t)nn, (float)cs, (float)sn, 0});
          } else {
            if (cs == 0.0) return false;
            const double k1 = sn * sig[nn] / (cs * sig[m]);
            const double k2 = sn * sig[m] / (cs * sig[nn]);
            sig[m] *= cs;
            sig[nn] *= cs;
            if (!(std::fabs(k1) <= 0x1p100) || !(std::fabs(k2) <= 0x1p100)) return false;
            if (!(std::fabs(sig[m]) >= fast_sigma_floor(log2n)) || !(std::fabs(sig[nn]) >= fast_sigma_floor(log2n)))
              return false;
            pr.ops.push_back(ProgOp{0, (uint16_t)m, (uint16_t)nn, (float)k1, (float)-k2, 0});
          }
        }
      }
      gather(k + 1);
    }
    if (!standard) {
      pr.scales.resize(n);
      for (int i = 0; i < n; ++i) pr.scales[i] = (float)sig[i];
      pr.ops.push_back(ProgOp{2, 0, 0, 0.f, 0.f, 0});
    }
  }
  return true;
}

}  // namespace hygt_gpu

namespace hygt_gpu {


void compose_operator(int log2n, int rounds, const double* angles_c, const uint16_t* perms_c,
                      uint32_t mask, double* out) {
  const int n = 1 << log2n, half = n / 2;
  // X[i][k] = sample i of the transform of unit vector e_k; the butterflies act on whole rows
  std::vector<double> x((size_t)n * n, 0.0), tmp((size_t)n * n);
  for (int i = 0; i < n; ++i) x[(size_t)i * n + i] = 1.0;
  for (int r = 0; r < rounds; ++r) {
    for (int p = 0; p < log2n; ++p) {
      const uint32_t kk = 1u << p;
      const size_t base = ((size_t)r * log2n + p) * half;  // model.hpp:77-79
      for (int j = 0; j < half; ++j) {
        const uint32_t m = j + (j & (0u - kk)), nn = m + kk;  // transform.hpp:55-56
        const double t = angles_c[base + j], c = std::cos(t), s = std::sin(t);
        double* a = &x[(size_t)m * n];
        double* b = &x[(size_t)nn * n];
        for (int k = 0; k < n; ++k) {
          const double av = a[k], bv = b[k];
          a[k] = c * av + s * bv;  // transform.hpp:60-63
          b[k] = c * bv - s * av;
        }
      }
    }
    if (perms_c && ((mask >> r) & 1u)) {  // gather after round r: out[i] = pre[perm[i]]
      const uint16_t* pr = perms_c + (size_t)r * n;
      for (int i = 0; i < n; ++i) std::copy_n(&x[(size_t)pr[i] * n], n, &tmp[(size_t)i * n]);
      x.swap(tmp);
    }
  }
  std::copy(x.begin(), x.end(), out);
}

}  // namespace hygt_gpu
