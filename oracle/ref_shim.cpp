// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" driver around the UNMODIFIED reference headers, compiled from
// /root/reference/proj/include by oracle/Makefile into oracle/_ref/libhygt_ref.so (git-ignored,
// travels to the GPU box with the snapshot). No reference source is copied: this file only
// #includes the headers where they lie. Uses:
//   * tests/gen_golden.py: golden vectors for tests/golden/ (pins oracle/hygt_oracle.c);
//   * bench.py --impl reference and the cpu_baseline leg: the reference's own hygt::forward /
//     hygt::inverse timed on the host cores (std::thread over contiguous row ranges; models are
//     immutable and shareable, model.hpp:49-50).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <limits>
#include <optional>
#include <thread>
#include <vector>

#include "hygt/fixedpoint.hpp"
#include "hygt/hypercube.hpp"
#include "hygt/matrix.hpp"
#include "hygt/model.hpp"
#include "hygt/optimizer.hpp"
#include "hygt/rng.hpp"
#include "hygt/statistics.hpp"
#include "hygt/transform.hpp"

namespace {

using hygt::HyGTModel;

std::optional<std::vector<std::uint16_t>> perm_of(const std::uint16_t* p, std::size_t n) {
  if (!p) return std::nullopt;
  return std::vector<std::uint16_t>(p, p + n);
}

// The chain of SURVEY.md c2 (inter-round permutations), or the single R-round model when only
// the final permutation (bit rounds-1) or none is present -- the reference as shipped.
struct ClassModels {
  std::vector<HyGTModel> chain;
};

ClassModels build(int log2_n, int rounds, const double* angles, const std::uint16_t* perms,
                  std::uint32_t mask) {
  const std::size_t n = std::size_t{1} << log2_n;
  const std::size_t a1 = n / 2 * static_cast<std::size_t>(log2_n);
  const std::uint32_t inter = rounds > 1 ? (mask & ((1u << (rounds - 1)) - 1u)) : 0u;
  ClassModels cm;
  if (!perms || inter == 0) {
    const std::uint16_t* fin = (perms && ((mask >> (rounds - 1)) & 1u))
                                   ? perms + static_cast<std::size_t>(rounds - 1) * n
                                   : nullptr;
    cm.chain.emplace_back(log2_n, rounds,
                          std::vector<double>(angles, angles + a1 * rounds), perm_of(fin, n));
    return cm;
  }
  for (int r = 0; r < rounds; ++r) {
    const std::uint16_t* p = ((mask >> r) & 1u) ? perms + static_cast<std::size_t>(r) * n : nullptr;
    cm.chain.emplace_back(log2_n, 1, std::vector<double>(angles + a1 * r, angles + a1 * (r + 1)),
                          perm_of(p, n));
  }
  return cm;
}

std::vector<double> run(const ClassModels& cm, std::vector<double> v, bool inverse) {
  if (!inverse) {
    for (const auto& m : cm.chain) v = hygt::forward(m, std::move(v));
  } else {
    for (auto it = cm.chain.rbegin(); it != cm.chain.rend(); ++it) v = hygt::inverse(*it, std::move(v));
  }
  return v;
}

int status_of_current() {
  try {
    throw;
  } catch (const hygt::OverflowError&) {
    return 4;
  } catch (const hygt::NumericalError&) {
    return 3;
  } catch (const hygt::IoError&) {
    return 2;
  } catch (const hygt::ArgumentError&) {
    return 1;
  } catch (...) {
    return 9;
  }
}

}  // namespace

extern "C" {

int ref_hypercube_indices(int log2_n, int pass, std::uint32_t* m, std::uint32_t* n) {
  try {
    const auto idx = hygt::hypercube_indices(log2_n, pass);
    std::copy(idx.m.begin(), idx.m.end(), m);
    std::copy(idx.n.begin(), idx.n.end(), n);
    return 0;
  } catch (...) {
    return status_of_current();
  }
}

// Model-level calls: one vector, fp64 in place.
int ref_apply_one(int log2_n, int rounds, const double* angles, const std::uint16_t* perms,
                  std::uint32_t mask, double* x, int inverse) {
  try {
    const std::size_t n = std::size_t{1} << log2_n;
    const ClassModels cm = build(log2_n, rounds, angles, perms, mask);
    auto y = run(cm, std::vector<double>(x, x + n), inverse != 0);
    std::memcpy(x, y.data(), n * sizeof(double));
    return 0;
  } catch (...) {
    return status_of_current();
  }
}

int ref_to_matrix(int log2_n, int rounds, const double* angles, const std::uint16_t* perm,
                  double* t) {
  try {
    const std::size_t n = std::size_t{1} << log2_n;
    HyGTModel m(log2_n, rounds,
                std::vector<double>(angles, angles + hygt::num_parameters(log2_n, rounds)),
                perm_of(perm, n));
    const hygt::Matrix mt = hygt::to_matrix(m);
    std::memcpy(t, mt.data().data(), n * n * sizeof(double));
    return 0;
  } catch (...) {
    return status_of_current();
  }
}

// Batched apply over fp32 rows (the run_apply loop, hygt_main.cpp:143-149), multi-threaded.
// y may be float (out_f32) or double (out_f64); either may be null.
int ref_apply_batch(int log2_n, int rounds, int classes, const double* angles,
                    const std::uint16_t* perms, std::uint32_t mask, const float* x,
                    const std::uint16_t* cls, std::uint64_t count, int inverse, float* out_f32,
                    double* out_f64, int threads) {
  try {
    const std::size_t n = std::size_t{1} << log2_n;
    const std::size_t a = hygt::num_parameters(log2_n, rounds);
    std::vector<ClassModels> cache;
    for (int c = 0; c < classes; ++c)
      cache.push_back(build(log2_n, rounds, angles + a * c,
                            perms ? perms + static_cast<std::size_t>(c) * rounds * n : nullptr,
                            mask));
    if (threads < 1) threads = 1;
    std::vector<std::thread> pool;
    std::vector<int> bad(threads, 0);
    for (int t = 0; t < threads; ++t) {
      pool.emplace_back([&, t] {
        const std::uint64_t b = count * t / threads, e = count * (t + 1) / threads;
        for (std::uint64_t row = b; row < e; ++row) {
          const unsigned c = cls ? cls[row] : 0u;
          if (static_cast<int>(c) >= classes) {
            bad[t] = 1;
            continue;
          }
          std::vector<double> v(n);
          for (std::size_t i = 0; i < n; ++i) v[i] = static_cast<double>(x[row * n + i]);
          v = run(cache[c], std::move(v), inverse != 0);
          if (out_f32)
            for (std::size_t i = 0; i < n; ++i) out_f32[row * n + i] = static_cast<float>(v[i]);
          if (out_f64) std::memcpy(out_f64 + row * n, v.data(), n * sizeof(double));
        }
      });
    }
    for (auto& th : pool) th.join();
    for (int b : bad)
      if (b) return 1;
    return 0;
  } catch (...) {
    return status_of_current();
  }
}

int ref_trig_table(int angle_bits, int precision_bits, std::int32_t* c, std::int32_t* s) {
  try {
    const hygt::TrigTable t(angle_bits, precision_bits);
    for (std::size_t q = 0; q < t.size(); ++q) {
      c[q] = t.cos_entry(q);
      s[q] = t.sin_entry(q);
    }
    return 0;
  } catch (...) {
    return status_of_current();
  }
}

int ref_quantize(int log2_n, int rounds, const double* angles, int angle_bits,
                 std::uint16_t* codes) {
  try {
    const HyGTModel m(log2_n, rounds,
                      std::vector<double>(angles, angles + hygt::num_parameters(log2_n, rounds)));
    const auto q = hygt::quantize_model(m, angle_bits);
    std::copy(q.codes().begin(), q.codes().end(), codes);
    return 0;
  } catch (...) {
    return status_of_current();
  }
}

// forward_fixed / inverse_fixed on one vector (final permutation only, as the reference).
int ref_fixed_one(int log2_n, int rounds, int angle_bits, int precision_bits,
                  const std::uint16_t* codes, const std::uint16_t* perm, std::int64_t* x,
                  int inverse) {
  try {
    const std::size_t n = std::size_t{1} << log2_n;
    const hygt::QuantizedHyGTModel m(
        log2_n, rounds, angle_bits,
        std::vector<std::uint16_t>(codes, codes + hygt::num_parameters(log2_n, rounds)),
        perm_of(perm, n));
    const hygt::TrigTable t(angle_bits, precision_bits);
    std::vector<std::int64_t> v(x, x + n);
    v = inverse ? hygt::inverse_fixed(m, t, std::move(v)) : hygt::forward_fixed(m, t, std::move(v));
    std::memcpy(x, v.data(), n * sizeof(std::int64_t));
    return 0;
  } catch (...) {
    return status_of_current();
  }
}

std::size_t ref_memory_footprint(int klt, int log2_n, int rounds, int num) {
  return hygt::memory_footprint(klt ? hygt::TransformKind::klt : hygt::TransformKind::hygt,
                                log2_n, rounds, num);
}

// klt_forward (statistics.hpp:222-224) on one vector; inverse via transposed (matrix.hpp:82).
int ref_klt_one(int n, const double* k, const double* x, double* y, int inverse) {
  try {
    hygt::Matrix m(static_cast<std::size_t>(n));
    std::memcpy(m.data().data(), k, static_cast<std::size_t>(n) * n * sizeof(double));
    hygt::KLTResult klt{inverse ? hygt::transposed(m) : m, {}};
    const auto v = hygt::klt_forward(klt, std::span<const double>(x, static_cast<std::size_t>(n)));
    std::memcpy(y, v.data(), static_cast<std::size_t>(n) * sizeof(double));
    return 0;
  } catch (...) {
    return status_of_current();
  }
}

// Diagonal of the per-class CorrelationAccumulator sums over forward outputs (the energy
// oracle of config 5 via the reference accumulator itself: E[c][i] = count_c * Phi_c(i,i)).
int ref_class_energy(int log2_n, int rounds, int classes, const double* angles,
                     const std::uint16_t* perms, std::uint32_t mask, const float* x,
                     const std::uint16_t* cls, std::uint64_t count, double* energy) {
  try {
    const std::size_t n = std::size_t{1} << log2_n;
    const std::size_t a = hygt::num_parameters(log2_n, rounds);
    std::vector<hygt::CorrelationAccumulator> acc;
    std::vector<ClassModels> cache;
    for (int c = 0; c < classes; ++c) {
      acc.emplace_back(n);
      cache.push_back(build(log2_n, rounds, angles + a * c,
                            perms ? perms + static_cast<std::size_t>(c) * rounds * n : nullptr,
                            mask));
    }
    for (std::uint64_t row = 0; row < count; ++row) {
      const unsigned c = cls ? cls[row] : 0u;
      std::vector<double> v(n);
      for (std::size_t i = 0; i < n; ++i) v[i] = static_cast<double>(x[row * n + i]);
      acc[c].add(run(cache[c], std::move(v), false));
    }
    for (int c = 0; c < classes; ++c) {
      if (acc[c].count() == 0) {
        for (std::size_t i = 0; i < n; ++i) energy[c * n + i] = 0.0;
        continue;
      }
      const auto phi = acc[c].finalize();
      for (std::size_t i = 0; i < n; ++i)
        energy[c * n + i] = phi.values()(i, i) * static_cast<double>(acc[c].count());
    }
    return 0;
  } catch (...) {
    return status_of_current();
  }
}

// Reference Rng streams, for pinning the oracle's mt19937_64 restatement.
// kind 0 = uniform01, 1 = gaussian, 2 = below(bound), 3 = raw derive_seed(seed, i).
int ref_rng_stream(std::uint64_t seed, int kind, std::uint64_t bound, std::uint64_t count,
                   double* out_d, std::uint64_t* out_u) {
  hygt::Rng rng(seed);
  for (std::uint64_t i = 0; i < count; ++i) {
    switch (kind) {
      case 0: out_d[i] = rng.uniform01(); break;
      case 1: out_d[i] = rng.gaussian(); break;
      case 2: out_u[i] = rng.below(bound); break;
      default: out_u[i] = hygt::derive_seed(seed, i); break;
    }
  }
  return 0;
}

// Per-class CorrelationAccumulator (statistics.hpp:63-99): phi[c] = finalize() over the rows of
// class c (fp64 values of the fp32 samples), counts[c] = count().
int ref_correlation(int log2_n, int classes, const float* x, const std::uint16_t* cls,
                    std::uint64_t count, double* phi, std::uint64_t* counts) {
  try {
    const std::size_t n = std::size_t{1} << log2_n;
    std::vector<hygt::CorrelationAccumulator> acc;
    for (int c = 0; c < classes; ++c) acc.emplace_back(n);
    std::vector<double> r(n);
    for (std::uint64_t k = 0; k < count; ++k) {
      for (std::size_t i = 0; i < n; ++i) r[i] = static_cast<double>(x[k * n + i]);
      acc.at(cls ? cls[k] : 0).add(r);
    }
    for (int c = 0; c < classes; ++c) {
      counts[c] = acc[c].count();
      if (!acc[c].count()) continue;
      const auto m = acc[c].finalize();
      std::memcpy(phi + (std::size_t)c * n * n, m.values().data().data(), n * n * sizeof(double));
    }
    return 0;
  } catch (...) {
    return status_of_current();
  }
}

int ref_ar1_covariance_2d(int block_size, double rho, double* out) {
  try {
    const auto phi = hygt::ar1_covariance_2d(block_size, rho);
    std::memcpy(out, phi.values().data().data(), phi.n() * phi.n() * sizeof(double));
    return 0;
  } catch (...) {
    return status_of_current();
  }
}

// optimizer.hpp:311-371 through the reference's own optimize(); trajectories are NaN padded
// to max_sweeps + 1 entries per restart.
int ref_optimize(const double* phi, int log2_n, int rounds, int restarts, int max_sweeps,
                 double tol, std::uint64_t seed, int init_mode, double* angles, double* gains,
                 int* best, double* klt_gain, double* traj, int* traj_len) {
  try {
    const std::size_t n = std::size_t{1} << log2_n;
    hygt::Matrix m(n);
    std::memcpy(m.data().data(), phi, n * n * sizeof(double));
    const hygt::CorrelationMatrix cm(std::move(m), 0);
    hygt::OptimizerConfig cfg;
    cfg.restarts = restarts;
    cfg.max_sweeps = max_sweeps;
    cfg.gain_tolerance_db = tol;
    cfg.seed = seed;
    cfg.init_mode = static_cast<hygt::InitMode>(init_mode);
    auto [model, rep] = hygt::optimize(cm, log2_n, rounds, cfg);
    std::memcpy(angles, model.angles().data(), model.angles().size() * sizeof(double));
    for (int r = 0; r < restarts; ++r) {
      gains[r] = rep.restart_gains_db[r];
      traj_len[r] = static_cast<int>(rep.trajectories[r].size());
      for (int k = 0; k <= max_sweeps; ++k)
        traj[(std::size_t)r * (max_sweeps + 1) + k] =
            k < traj_len[r] ? rep.trajectories[r][k] : std::numeric_limits<double>::quiet_NaN();
    }
    *best = static_cast<int>(rep.best_restart);
    *klt_gain = rep.klt_gain_db;
    return 0;
  } catch (...) {
    return status_of_current();
  }
}

// optimizer.hpp:378-390 (variance_permutation) and the propagated diagonal it sorts.
int ref_variance_permutation(const double* phi, int log2_n, int rounds, const double* angles,
                             std::uint16_t* perm, double* var) {
  try {
    const std::size_t n = std::size_t{1} << log2_n;
    hygt::Matrix m(n);
    std::memcpy(m.data().data(), phi, n * n * sizeof(double));
    const hygt::CorrelationMatrix cm(std::move(m), 0);
    const hygt::HyGTModel model(log2_n, rounds,
                                std::vector<double>(angles, angles + hygt::num_parameters(log2_n, rounds)));
    const auto prop = hygt::propagate_covariance(model, cm);
    for (std::size_t i = 0; i < n; ++i) var[i] = prop.values()(i, i);
    const auto sorted = hygt::variance_permutation(model, cm);
    std::memcpy(perm, sorted.permutation()->data(), n * sizeof(std::uint16_t));
    return 0;
  } catch (...) {
    return status_of_current();
  }
}

}  // extern "C"
