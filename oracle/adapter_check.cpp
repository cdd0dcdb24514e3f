// adapter_check.cpp -- TEST PROGRAM: drives include/hygt_gpu_adapter.hpp with the reference's
// own types (built against the unmodified /root/reference headers by oracle/Makefile into
// oracle/_ref/adapter_check) and compares every result with the reference's own functions.
// Run on a GPU box by tests/test_gpu_parity.py::test_reference_adapter. Exit 0 = all checks ok.
#include <cmath>
#include <cstdio>
#include <vector>

#include "hygt/bundle.hpp"
#include "hygt/dataset.hpp"
#include "hygt/fixedpoint.hpp"
#include "hygt/rng.hpp"
#include "hygt/transform.hpp"
#include "hygt_gpu_adapter.hpp"

static int failures = 0;
#define EXPECT(cond, ...)             \
  do {                                \
    if (!(cond)) {                    \
      std::printf("FAIL: " __VA_ARGS__); \
      std::printf("\n");              \
      ++failures;                     \
    }                                 \
  } while (0)

int main() {
  hygt::Rng rng(2505);
  // --- one-vector drop-ins vs hygt::forward / hygt::inverse (transform.hpp:72-96)
  for (int log2n : {1, 2, 4, 6, 8}) {
    const std::size_t n = std::size_t{1} << log2n;
    std::vector<double> ang(hygt::num_parameters(log2n, 3));
    for (double& a : ang) a = rng.uniform(-3.14159, 3.14159);
    std::vector<std::uint16_t> perm(n);  // a reversal as the final sorting permutation
    for (std::size_t i = 0; i < n; ++i) perm[i] = static_cast<std::uint16_t>(n - 1 - i);
    const hygt::HyGTModel m(log2n, 3, ang, perm);
    std::vector<double> x(n);
    for (double& v : x) v = 16 * rng.gaussian();
    for (auto& v : x) v = static_cast<float>(v);
    const auto yr = hygt::forward(m, x), yg = hygt::gpu::forward(m, x);
    const auto xr = hygt::inverse(m, x), xg = hygt::gpu::inverse(m, x);
    double e1 = 0, e2 = 0, s = 0;
    for (std::size_t i = 0; i < n; ++i) {
      e1 = std::max(e1, std::abs(yr[i] - yg[i]));
      e2 = std::max(e2, std::abs(xr[i] - xg[i]));
      s = std::max(s, std::abs(x[i]));
    }
    EXPECT(e1 <= 1e-5 * s && e2 <= 1e-5 * s, "gpu::forward/inverse log2n=%d err %.3g %.3g", log2n, e1, e2);
  }
  // --- errors rethrown as the reference's classes
  bool threw = false;
  try {
    hygt::gpu::forward(hygt::HyGTModel::zeros(2, 1), {1.0, 2.0});
  } catch (const hygt::ArgumentError&) {
    threw = true;
  }
  EXPECT(threw, "dimension mismatch did not throw ArgumentError");
  // --- the `hygt apply` data path on a ResidualDataset (hygt_main.cpp:130-172), float and fixed
  for (int log2n : {4, 6}) {
    const std::size_t n = std::size_t{1} << log2n;
    const int classes = 5, rounds = 2;
    std::vector<hygt::HyGTModel> models;
    std::vector<hygt::QuantizedHyGTModel> qmodels;
    for (int c = 0; c < classes; ++c) {
      std::vector<double> ang(hygt::num_parameters(log2n, rounds));
      for (double& a : ang) a = rng.uniform(0, 6.28318);
      models.emplace_back(log2n, rounds, ang);
      qmodels.push_back(hygt::quantize_model(models.back(), 8));
    }
    std::vector<hygt::ResidualBlock> blocks(3000);
    for (auto& b : blocks) {
      b.class_id = static_cast<std::uint16_t>(rng.below(classes));
      b.values.resize(n);
      for (double& v : b.values) v = std::round(64 * rng.gaussian());
    }
    const hygt::ResidualDataset ds(log2n, classes, blocks);
    const hygt::ModelBundle fb(models), qb(qmodels);
    const auto yf = hygt::gpu::apply(fb, ds, true, false);
    const auto yq = hygt::gpu::apply(qb, ds, true, true);
    const hygt::TrigTable table(8, 10);
    double ef = 0, sc = 0;
    long long mism = 0;
    for (std::size_t r = 0; r < blocks.size(); ++r) {
      const auto& b = blocks[r];
      const auto ref = hygt::forward(models[b.class_id], b.values);
      std::vector<std::int64_t> xi(b.values.begin(), b.values.end());
      const auto refi = hygt::forward_fixed(qmodels[b.class_id], table, xi);
      for (std::size_t i = 0; i < n; ++i) {
        ef = std::max(ef, std::abs(ref[i] - yf.blocks()[r].values[i]));
        sc = std::max(sc, std::abs(b.values[i]));
        mism += static_cast<double>(refi[i]) != yq.blocks()[r].values[i];
      }
      EXPECT(yf.blocks()[r].class_id == b.class_id, "class id not carried");
    }
    EXPECT(ef <= 1e-5 * sc, "gpu::apply float log2n=%d max err %.3g", log2n, ef);
    EXPECT(mism == 0, "gpu::apply fixed log2n=%d: %lld mismatches (must be bit-exact)", log2n, mism);
  }
  // --- hygt::gpu::optimize vs hygt::optimize (optimizer.hpp:311-371), acceptance case N=16 R=2
  {
    const hygt::CorrelationMatrix phi = hygt::ar1_covariance_2d(4, 0.95);
    hygt::OptimizerConfig cfg;
    cfg.restarts = 2;
    cfg.seed = 1;
    cfg.max_sweeps = 5;
    const auto [mr, rr] = hygt::optimize(phi, 4, 2, cfg);
    const auto [mg, rg] = hygt::gpu::optimize(phi, 4, 2, cfg);
    for (std::size_t k = 0; k < rr.restart_gains_db.size(); ++k)
      EXPECT(std::abs(rr.restart_gains_db[k] - rg.restart_gains_db[k]) < 1e-5, "gpu::optimize restart %zu gain %.9f vs %.9f", k,
             rg.restart_gains_db[k], rr.restart_gains_db[k]);
    EXPECT(std::abs(rr.klt_gain_db - rg.klt_gain_db) < 1e-9, "gpu::optimize klt gain");
    EXPECT(rr.best_restart == rg.best_restart, "gpu::optimize best restart");
    bool threw = false;
    try {
      hygt::Matrix bad(2);
      bad(0, 0) = 1.0;
      bad(1, 1) = -1.0;
      hygt::gpu::optimize(hygt::CorrelationMatrix(std::move(bad), 0), 1, 1, hygt::OptimizerConfig{});
    } catch (const hygt::ArgumentError&) {
      threw = true;
    }
    EXPECT(threw, "gpu::optimize must throw ArgumentError on an indefinite covariance");
  }
  // --- hygt::gpu::klt_forward / KLTPlan vs klt_forward and its transpose (statistics.hpp:222-224)
  for (int log2n : {2, 4, 6}) {
    const std::size_t n = std::size_t{1} << log2n;
    const int classes = 3;
    std::vector<hygt::KLTResult> klts;
    for (int c = 0; c < classes; ++c)
      klts.push_back(hygt::jacobi_eigen(hygt::ar1_covariance_2d(1 << (log2n / 2), 0.6 + 0.1 * c)));
    std::vector<double> x(n);
    for (double& v : x) v = static_cast<float>(16 * rng.gaussian());
    const auto yr = hygt::klt_forward(klts[1], x), yg = hygt::gpu::klt_forward(klts[1], x);
    double e = 0, sc = 0;
    for (std::size_t i = 0; i < n; ++i) {
      e = std::max(e, std::abs(yr[i] - yg[i]));
      sc = std::max(sc, std::abs(x[i]));
    }
    EXPECT(e <= 1e-5 * sc, "gpu::klt_forward log2n=%d err %.3g", log2n, e);
    const std::size_t rows = 1000;
    std::vector<float> h(rows * n), hy(rows * n), hb(rows * n);
    std::vector<std::uint16_t> cls(rows);
    for (std::size_t r = 0; r < rows; ++r) {
      cls[r] = static_cast<std::uint16_t>(rng.below(classes));
      for (std::size_t i = 0; i < n; ++i) h[r * n + i] = static_cast<float>(16 * rng.gaussian());
    }
    hygt::gpu::DeviceBuffer<float> dx(rows * n), dy(rows * n), db(rows * n);
    hygt::gpu::DeviceBuffer<std::uint16_t> dc(rows);
    cudaMemcpy(dx.p, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dc.p, cls.data(), rows * 2, cudaMemcpyHostToDevice);
    hygt::gpu::KLTPlan plan(klts);
    plan.bucket(dc.p, rows);
    plan.forward(dx.p, dy.p, dc.p, rows, nullptr, true);
    plan.inverse(dy.p, db.p, dc.p, rows, nullptr, true);
    cudaMemcpy(hy.data(), dy.p, hy.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(hb.data(), db.p, hb.size() * 4, cudaMemcpyDeviceToHost);
    double ef = 0, eb = 0;
    for (std::size_t r = 0; r < rows; ++r) {
      const std::vector<double> xr(h.begin() + r * n, h.begin() + (r + 1) * n);
      const auto ref = hygt::klt_forward(klts[cls[r]], xr);
      for (std::size_t i = 0; i < n; ++i) {
        ef = std::max(ef, std::abs(ref[i] - hy[r * n + i]));
        eb = std::max(eb, std::abs(xr[i] - hb[r * n + i]));
      }
    }
    EXPECT(ef <= 1e-5 * 80 && eb <= 1e-5 * 80, "gpu::KLTPlan log2n=%d fwd err %.3g roundtrip %.3g", log2n, ef, eb);
  }
  // --- hygt::gpu::class_correlations vs the CorrelationAccumulator loop of hygt train
  //     (hygt_main.cpp:85-87, statistics.hpp:63-99)
  for (int log2n : {4, 6, 7}) {
    const std::size_t n = std::size_t{1} << log2n;
    const int classes = 4;  // class 3 stays empty
    std::vector<hygt::ResidualBlock> blocks(2500);
    for (auto& b : blocks) {
      b.class_id = static_cast<std::uint16_t>(rng.below(3));
      b.values.resize(n);
      for (double& v : b.values) v = static_cast<float>(16 * rng.gaussian());
    }
    const hygt::ResidualDataset ds(log2n, classes, blocks);
    const auto got = hygt::gpu::class_correlations(ds);
    for (int c = 0; c < classes; ++c) {
      hygt::CorrelationAccumulator acc(n);
      for (const auto& b : ds.blocks())
        if (b.class_id == c) acc.add(b.values);
      if (!acc.count()) {
        EXPECT(!got[c].has_value(), "class_correlations: empty class %d must be nullopt", c);
        continue;
      }
      EXPECT(got[c].has_value() && got[c]->sample_count() == acc.count(), "class_correlations: count of class %d", c);
      if (!got[c]) continue;
      const auto ref = acc.finalize();
      double e = 0, m = 0;
      for (std::size_t i = 0; i < n * n; ++i) {
        e = std::max(e, std::abs(ref.values().data()[i] - got[c]->values().data()[i]));
        m = std::max(m, std::abs(ref.values().data()[i]));
      }
      EXPECT(e <= 1e-12 * m, "class_correlations log2n=%d class %d err %.3g of %.3g", log2n, c, e, m);
    }
  }
  // --- hygt::gpu::train vs the loop of run_train (hygt_main.cpp:74-120): same per-class gains
  {
    const int log2n = 4, rounds = 2, classes = 3;  // class 2 gets too few samples -> identity
    const std::size_t n = 16;
    std::vector<hygt::ResidualBlock> blocks;
    const auto cov = hygt::ar1_covariance_2d(4, 0.9);
    hygt::Rng srng(77);
    for (int c = 0; c < classes; ++c) {
      const std::size_t m = c == 2 ? 5 : 600;
      for (std::size_t k = 0; k < m; ++k) {
        hygt::ResidualBlock b;
        b.class_id = static_cast<std::uint16_t>(c);
        b.values.resize(n);
        double prev = 0.0;
        for (std::size_t i = 0; i < n; ++i) {  // an AR(1) line with a class-dependent rho
          const double rho = 0.5 + 0.2 * c;
          prev = i ? rho * prev + std::sqrt(1 - rho * rho) * srng.gaussian() : srng.gaussian();
          b.values[i] = static_cast<float>(16 * prev);
        }
        blocks.push_back(std::move(b));
      }
    }
    const hygt::ResidualDataset ds(log2n, classes, blocks);
    std::vector<hygt::TrainingReport> reps;
    const hygt::ModelBundle bundle = hygt::gpu::train(ds, rounds, 2, 9, 0, &reps);
    EXPECT(bundle.class_count() == static_cast<std::size_t>(classes), "gpu::train class count");
    for (std::uint16_t c = 0; c < classes; ++c) {
      hygt::CorrelationAccumulator acc(n);
      for (const auto& b : ds.blocks())
        if (b.class_id == c) acc.add(b.values);
      const hygt::HyGTModel got = bundle.dequantized(c);
      if (acc.count() < n) {
        bool zero = !got.permutation();
        for (double a : got.angles()) zero = zero && a == 0.0;
        EXPECT(zero, "gpu::train: class %d must keep the identity model", c);
        continue;
      }
      const auto phi = acc.finalize();
      hygt::OptimizerConfig cfg;
      cfg.restarts = 2;
      cfg.seed = hygt::derive_seed(9, c);
      auto [mr, rr] = hygt::optimize(phi, log2n, rounds, cfg);
      EXPECT(std::abs(rr.restart_gains_db[rr.best_restart] - reps[c].restart_gains_db[reps[c].best_restart]) < 1e-5,
             "gpu::train class %d gain %.9f vs %.9f", c, reps[c].restart_gains_db[reps[c].best_restart],
             rr.restart_gains_db[rr.best_restart]);
      EXPECT(got.permutation().has_value(), "gpu::train: class %d has no variance permutation", c);
    }
    (void)cov;
  }
  std::printf("adapter_check: %s (%d failures)\n", failures ? "FAILED" : "ok", failures);
  return failures ? 1 : 0;
}
