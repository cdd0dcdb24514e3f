// hygt_gpu_adapter.hpp -- header-only C++ adapter from the reference's types to the C ABI.
//
// Include it next to the reference headers (/root/reference/proj/include) and link
// libhygt_gpu.so + cudart. It replaces, for batches:
//   * the per-class model cache + per-block loop of run_apply (tools/hygt_main.cpp:143-149)
//     -> hygt::gpu::Plan(std::vector<HyGTModel>) + Plan::forward/inverse on device buffers;
//   * hygt::forward / hygt::inverse (transform.hpp:72-96) on one vector -> hygt::gpu::forward /
//     hygt::gpu::inverse (same signatures, fp32 device arithmetic);
//   * forward_fixed / inverse_fixed (fixedpoint.hpp:191-224) -> hygt::gpu::FixedPlan;
//   * the whole `hygt apply` data path on a ResidualDataset (hygt_main.cpp:130-172)
//     -> hygt::gpu::apply(bundle, dataset, forward, fixed);
//   * klt_forward (statistics.hpp:222-224) and its transpose -> hygt::gpu::KLTPlan (batches, one
//     KLTResult per class) and hygt::gpu::klt_forward (one vector, same signature);
//   * the per-class CorrelationAccumulator loop of `hygt train` (hygt_main.cpp:85-87,
//     statistics.hpp:63-99) -> hygt::gpu::class_correlations(dataset);
//   * hygt::optimize (optimizer.hpp:311-371) -> hygt::gpu::optimize;
//   * the training loop of `hygt train` (run_train, hygt_main.cpp:74-120) -> hygt::gpu::train(dataset, rounds, ...).
// Non-zero C-ABI statuses are rethrown as the reference's exception classes (errors.hpp:23-45).
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <optional>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "hygt/bundle.hpp"
#include "hygt/dataset.hpp"
#include "hygt/errors.hpp"
#include "hygt/fixedpoint.hpp"
#include "hygt/model.hpp"
#include "hygt/optimizer.hpp"
#include "hygt/statistics.hpp"
#include <algorithm>

#include "hygt_gpu.h"

namespace hygt::gpu {

inline void check(int status) {
  if (status == HYGT_OK) return;
  char msg[512];
  hygt_last_error(msg, sizeof msg);
  switch (status) {
    case HYGT_ERR_ARGUMENT: throw ArgumentError(msg);
    case HYGT_ERR_IO: throw IoError(msg);
    case HYGT_ERR_OVERFLOW: throw OverflowError(msg);
    case HYGT_ERR_NUMERICAL: throw NumericalError(msg);
    default: throw std::runtime_error(std::string("hygt_gpu: ") + msg);
  }
}

inline void cuda_check(cudaError_t e) {
  if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
}

// Device buffer (RAII).
template <class T>
struct DeviceBuffer {
  T* p = nullptr;
  std::size_t n = 0;
  explicit DeviceBuffer(std::size_t count = 0) { resize(count); }
  ~DeviceBuffer() { cudaFree(p); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  // Grows the buffer. New storage is zeroed: the transforms only ever OR error bits into a
  // workspace's first word (hygt_workspace_bytes), so a recycled allocation must not carry
  // stale bits. A pending error word of the old buffer is carried over.
  void resize(std::size_t count) {
    if (count <= n) return;
    T* q = nullptr;
    if (count) {
      cuda_check(cudaMalloc(reinterpret_cast<void**>(&q), count * sizeof(T)));
      cuda_check(cudaMemset(q, 0, count * sizeof(T)));
      if (p) cuda_check(cudaMemcpy(q, p, std::min<std::size_t>(n * sizeof(T), 16), cudaMemcpyDeviceToDevice));
    }
    cudaFree(p);
    p = q;
    n = count;
  }
};

// Per-class float plan. inter_round_perms (optional, BASELINE extension): [C][R-1] gathers
// applied after rounds 0..R-2; each model's own permutation is the final sorting gather.
class Plan {
 public:
  explicit Plan(const std::vector<HyGTModel>& models,
                const std::vector<std::vector<std::vector<std::uint16_t>>>* inter_round_perms = nullptr,
                std::uint32_t flags = 0) {
    if (models.empty()) throw ArgumentError("gpu::Plan: need at least one class");
    const int log2n = models.front().log2_n(), rounds = models.front().rounds();
    const std::size_t n = models.front().dimension();
    std::vector<double> angles;
    std::vector<std::uint16_t> perms(models.size() * rounds * n);
    std::uint32_t mask = 0;
    for (std::size_t c = 0; c < models.size(); ++c) {
      const auto& m = models[c];
      if (m.log2_n() != log2n || m.rounds() != rounds)
        throw ArgumentError("gpu::Plan: all classes must share log2_n and rounds");
      angles.insert(angles.end(), m.angles().begin(), m.angles().end());
      for (int r = 0; r < rounds; ++r)
        for (std::size_t i = 0; i < n; ++i) perms[(c * rounds + r) * n + i] = static_cast<std::uint16_t>(i);
      if (m.permutation()) {
        mask |= 1u << (rounds - 1);
        for (std::size_t i = 0; i < n; ++i) perms[(c * rounds + rounds - 1) * n + i] = (*m.permutation())[i];
      }
      if (inter_round_perms) {
        mask |= (1u << (rounds - 1)) - 1u;
        for (int r = 0; r + 1 < rounds; ++r)
          for (std::size_t i = 0; i < n; ++i) perms[(c * rounds + r) * n + i] = (*inter_round_perms)[c][r][i];
      }
    }
    check(hygt_plan_create(log2n, rounds, static_cast<int>(models.size()), angles.data(),
                           mask ? perms.data() : nullptr, mask, flags, &plan_));
    n_ = n;
  }
  explicit Plan(const ModelBundle& bundle) : Plan(dequantized_models(bundle)) {}
  ~Plan() { hygt_plan_destroy(plan_); }
  Plan(const Plan&) = delete;
  Plan& operator=(const Plan&) = delete;

  std::size_t dimension() const { return n_; }
  const hygt_plan* handle() const { return plan_; }

  // Device rows in/out (stream-ordered, asynchronous). d_cls may be null (all class 0).
  void forward(const float* d_x, float* d_y, const std::uint16_t* d_cls, std::size_t count,
               cudaStream_t stream = nullptr) {
    run(true, d_x, d_y, d_cls, count, stream);
  }
  void inverse(const float* d_y, float* d_x, const std::uint16_t* d_cls, std::size_t count,
               cudaStream_t stream = nullptr) {
    run(false, d_y, d_x, d_cls, count, stream);
  }
  // Throws ArgumentError if a previous call saw a class id >= class_count.
  void sync(cudaStream_t stream = nullptr) { check(hygt_sync_status(plan_, ws_.p, stream)); }

 private:
  static std::vector<HyGTModel> dequantized_models(const ModelBundle& b) {
    std::vector<HyGTModel> out;
    for (std::size_t c = 0; c < b.class_count(); ++c) out.push_back(b.dequantized(c));
    return out;
  }
  void run(bool fwd, const float* in, float* out, const std::uint16_t* cls, std::size_t count,
           cudaStream_t stream) {
    ws_.resize(hygt_workspace_bytes(plan_, count));
    check((fwd ? hygt_forward_f32 : hygt_inverse_f32)(plan_, in, out, cls, count, ws_.p, ws_.n, 0, stream));
  }
  hygt_plan* plan_ = nullptr;
  std::size_t n_ = 0;
  DeviceBuffer<unsigned char> ws_{256};
};

// Integer plan over quantized per-class models (bit-exact with forward_fixed/inverse_fixed).
class FixedPlan {
 public:
  FixedPlan(const std::vector<QuantizedHyGTModel>& models, const TrigTable& table) {
    if (models.empty()) throw ArgumentError("gpu::FixedPlan: need at least one class");
    const auto& m0 = models.front();
    const std::size_t n = m0.dimension();
    std::vector<std::uint16_t> codes, perms(models.size() * m0.rounds() * n);
    std::uint32_t mask = 0;
    for (std::size_t c = 0; c < models.size(); ++c) {
      const auto& m = models[c];
      if (m.angle_bits() != table.angle_bits())
        throw ArgumentError("forward_fixed: table/model angle_bits mismatch");
      codes.insert(codes.end(), m.codes().begin(), m.codes().end());
      for (int r = 0; r < m0.rounds(); ++r)
        for (std::size_t i = 0; i < n; ++i) perms[(c * m0.rounds() + r) * n + i] = static_cast<std::uint16_t>(i);
      if (m.permutation()) {
        mask |= 1u << (m0.rounds() - 1);
        for (std::size_t i = 0; i < n; ++i) perms[(c * m0.rounds() + m0.rounds() - 1) * n + i] = (*m.permutation())[i];
      }
    }
    check(hygt_fixed_plan_create(m0.log2_n(), m0.rounds(), static_cast<int>(models.size()),
                                 table.angle_bits(), table.precision_bits(), codes.data(),
                                 mask ? perms.data() : nullptr, mask, &plan_));
  }
  ~FixedPlan() { hygt_plan_destroy(plan_); }
  FixedPlan(const FixedPlan&) = delete;
  FixedPlan& operator=(const FixedPlan&) = delete;
  // Synchronous; throws like the reference for the first failing row (in row order).
  std::uint64_t forward(const std::int64_t* d_x, std::int64_t* d_y, const std::uint16_t* d_cls,
                        std::size_t count, cudaStream_t stream = nullptr) {
    std::uint64_t bad = 0;
    check(hygt_forward_i64(plan_, d_x, d_y, d_cls, count, &bad, stream));
    return bad;
  }
  std::uint64_t inverse(const std::int64_t* d_y, std::int64_t* d_x, const std::uint16_t* d_cls,
                        std::size_t count, cudaStream_t stream = nullptr) {
    std::uint64_t bad = 0;
    check(hygt_inverse_i64(plan_, d_y, d_x, d_cls, count, &bad, stream));
    return bad;
  }

 private:
  hygt_plan* plan_ = nullptr;
};

// One-vector drop-ins with the signatures of hygt::forward / hygt::inverse (transform.hpp:72,86).
inline std::vector<double> forward(const HyGTModel& model, std::vector<double> x) {
  if (x.size() != model.dimension()) throw ArgumentError("forward: dimension mismatch");
  Plan plan({model});
  std::vector<float> h(x.begin(), x.end());
  DeviceBuffer<float> d(h.size());
  cuda_check(cudaMemcpy(d.p, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
  plan.forward(d.p, d.p, nullptr, 1);
  cuda_check(cudaMemcpy(h.data(), d.p, h.size() * 4, cudaMemcpyDeviceToHost));
  return std::vector<double>(h.begin(), h.end());
}
inline std::vector<double> inverse(const HyGTModel& model, std::vector<double> y) {
  if (y.size() != model.dimension()) throw ArgumentError("inverse: dimension mismatch");
  Plan plan({model});
  std::vector<float> h(y.begin(), y.end());
  DeviceBuffer<float> d(h.size());
  cuda_check(cudaMemcpy(d.p, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
  plan.inverse(d.p, d.p, nullptr, 1);
  cuda_check(cudaMemcpy(h.data(), d.p, h.size() * 4, cudaMemcpyDeviceToHost));
  return std::vector<double>(h.begin(), h.end());
}

// The data path of `hygt apply` (hygt_main.cpp:130-172) on an in-memory dataset: float
// arithmetic through Plan, or fixed arithmetic (llround inputs, :157) through FixedPlan.
inline ResidualDataset apply(const ModelBundle& bundle, const ResidualDataset& ds, bool fwd,
                             bool fixed) {
  if (ds.log2_n() != bundle.log2_n()) throw ArgumentError("apply: model/data dimension mismatch");
  if (ds.class_count() != bundle.class_count())
    throw ArgumentError("apply: model/data class count mismatch");
  const std::size_t n = ds.dimension(), rows = ds.blocks().size();
  std::vector<std::uint16_t> cls(rows);
  for (std::size_t r = 0; r < rows; ++r) cls[r] = ds.blocks()[r].class_id;
  DeviceBuffer<std::uint16_t> dc(rows);
  if (rows) cuda_check(cudaMemcpy(dc.p, cls.data(), rows * 2, cudaMemcpyHostToDevice));
  std::vector<ResidualBlock> out(rows);
  if (!fixed) {
    std::vector<float> x(rows * n);
    for (std::size_t r = 0; r < rows; ++r)
      for (std::size_t i = 0; i < n; ++i) x[r * n + i] = static_cast<float>(ds.blocks()[r].values[i]);
    DeviceBuffer<float> d(rows * n);
    if (rows) cuda_check(cudaMemcpy(d.p, x.data(), x.size() * 4, cudaMemcpyHostToDevice));
    Plan plan(bundle);
    if (fwd) plan.forward(d.p, d.p, dc.p, rows);
    else plan.inverse(d.p, d.p, dc.p, rows);
    plan.sync();
    if (rows) cuda_check(cudaMemcpy(x.data(), d.p, x.size() * 4, cudaMemcpyDeviceToHost));
    for (std::size_t r = 0; r < rows; ++r)
      out[r] = {cls[r], std::vector<double>(x.begin() + r * n, x.begin() + (r + 1) * n)};
  } else {
    if (!bundle.quantized())
      throw ArgumentError("apply: fixed arithmetic needs a quantized bundle (train with --angle-bits 8)");
    std::vector<std::int64_t> x(rows * n);
    for (std::size_t r = 0; r < rows; ++r)
      for (std::size_t i = 0; i < n; ++i) x[r * n + i] = std::llround(ds.blocks()[r].values[i]);
    DeviceBuffer<std::int64_t> d(rows * n);
    if (rows) cuda_check(cudaMemcpy(d.p, x.data(), x.size() * 8, cudaMemcpyHostToDevice));
    std::vector<QuantizedHyGTModel> qm;
    for (std::size_t c = 0; c < bundle.class_count(); ++c) qm.push_back(bundle.quantized_model(c));
    FixedPlan plan(qm, TrigTable(bundle.angle_bits(), bundle.precision_bits()));
    if (fwd) plan.forward(d.p, d.p, dc.p, rows);
    else plan.inverse(d.p, d.p, dc.p, rows);
    if (rows) cuda_check(cudaMemcpy(x.data(), d.p, x.size() * 8, cudaMemcpyDeviceToHost));
    for (std::size_t r = 0; r < rows; ++r)
      out[r] = {cls[r], std::vector<double>(x.begin() + r * n, x.begin() + (r + 1) * n)};
  }
  return ResidualDataset(ds.log2_n(), ds.class_count(), std::move(out));
}

// Per-class dense KLT: y = K_c r (klt_forward, statistics.hpp:222-224 -> multiply,
// matrix.hpp:70-80) and x = K_c^T y (transposed, matrix.hpp:82-88), rows of KLTResult::basis =
// basis vectors. Device rows in/out, stream-ordered; n a power of two in [2, 256].
class KLTPlan {
 public:
  explicit KLTPlan(const std::vector<KLTResult>& klts) {
    if (klts.empty()) throw ArgumentError("gpu::KLTPlan: need at least one class");
    n_ = klts.front().basis.n();
    std::vector<double> k;
    for (const auto& r : klts) {
      if (r.basis.n() != n_) throw ArgumentError("matrix dimension mismatch");
      k.insert(k.end(), r.basis.data().begin(), r.basis.data().end());
    }
    check(hygt_klt_plan_create(static_cast<int>(n_), static_cast<int>(klts.size()), k.data(), 0, &plan_));
  }
  ~KLTPlan() { hygt_klt_plan_destroy(plan_); }
  KLTPlan(const KLTPlan&) = delete;
  KLTPlan& operator=(const KLTPlan&) = delete;
  std::size_t dimension() const { return n_; }

  // Groups the rows by class once; forward / inverse with reuse = true then run on that grouping.
  void bucket(const std::uint16_t* d_cls, std::size_t count, cudaStream_t stream = nullptr) {
    ws_.resize(hygt_klt_workspace_bytes(plan_, count));
    check(hygt_klt_bucket(plan_, d_cls, count, ws_.p, ws_.n, stream));
  }
  void forward(const float* d_x, float* d_y, const std::uint16_t* d_cls, std::size_t count,
               cudaStream_t stream = nullptr, bool reuse = false) {
    ws_.resize(hygt_klt_workspace_bytes(plan_, count));
    check(hygt_klt_forward_f32_ex(plan_, d_x, d_y, d_cls, count, ws_.p, ws_.n, reuse ? HYGT_REUSE_BUCKETS : 0u, stream));
  }
  void inverse(const float* d_y, float* d_x, const std::uint16_t* d_cls, std::size_t count,
               cudaStream_t stream = nullptr, bool reuse = false) {
    ws_.resize(hygt_klt_workspace_bytes(plan_, count));
    check(hygt_klt_inverse_f32_ex(plan_, d_y, d_x, d_cls, count, ws_.p, ws_.n, reuse ? HYGT_REUSE_BUCKETS : 0u, stream));
  }

 private:
  hygt_klt_plan* plan_ = nullptr;
  std::size_t n_ = 0;
  DeviceBuffer<unsigned char> ws_;
};

// One-vector drop-in with the signature of klt_forward (statistics.hpp:222).
inline std::vector<double> klt_forward(const KLTResult& klt, std::span<const double> r) {
  if (r.size() != klt.basis.n()) throw ArgumentError("matrix/vector dimension mismatch");
  KLTPlan plan({klt});
  std::vector<float> h(r.begin(), r.end());
  DeviceBuffer<float> d(h.size()), o(h.size());
  cuda_check(cudaMemcpy(d.p, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
  plan.forward(d.p, o.p, nullptr, 1);
  cuda_check(cudaMemcpy(h.data(), o.p, h.size() * 4, cudaMemcpyDeviceToHost));
  return std::vector<double>(h.begin(), h.end());
}

// The per-class CorrelationAccumulator loop of `hygt train` (hygt_main.cpp:85-87): for every
// class, finalize() of the accumulator over its blocks (statistics.hpp:63-99), or nullopt for a
// class without samples (finalize would throw). Samples are taken as fp32, as RBLK stores them
// (dataset.hpp:68-70): every product is exact in fp64, as in the reference.
inline std::vector<std::optional<CorrelationMatrix>> class_correlations(const ResidualDataset& ds) {
  const std::size_t n = ds.dimension(), rows = ds.blocks().size(), classes = ds.class_count();
  if (ds.log2_n() < 2 || ds.log2_n() > 8) throw ArgumentError("gpu::class_correlations: log2_n must be in [2, 8]");
  std::vector<float> x(rows * n);
  std::vector<std::uint16_t> cls(rows);
  for (std::size_t r = 0; r < rows; ++r) {
    cls[r] = ds.blocks()[r].class_id;
    for (std::size_t i = 0; i < n; ++i) x[r * n + i] = static_cast<float>(ds.blocks()[r].values[i]);
  }
  DeviceBuffer<float> dx(x.size());
  DeviceBuffer<std::uint16_t> dc(rows);
  DeviceBuffer<double> dsum(classes * n * n);
  DeviceBuffer<unsigned long long> dcnt(classes);
  DeviceBuffer<unsigned char> ws(std::max<std::size_t>(256, hygt_correlation_workspace_bytes(static_cast<int>(classes), rows)));
  if (rows) {
    cuda_check(cudaMemcpy(dx.p, x.data(), x.size() * 4, cudaMemcpyHostToDevice));
    cuda_check(cudaMemcpy(dc.p, cls.data(), rows * 2, cudaMemcpyHostToDevice));
    check(hygt_correlation_f64(ds.log2_n(), static_cast<int>(classes), dx.p, dc.p, rows, dsum.p, dcnt.p,
                               ws.p, ws.n, nullptr));
    check(hygt_sync_status(nullptr, ws.p, nullptr));
  }
  std::vector<double> sum(classes * n * n);
  std::vector<unsigned long long> cnt(classes);
  cuda_check(cudaMemcpy(sum.data(), dsum.p, sum.size() * 8, cudaMemcpyDeviceToHost));
  cuda_check(cudaMemcpy(cnt.data(), dcnt.p, cnt.size() * 8, cudaMemcpyDeviceToHost));
  std::vector<std::optional<CorrelationMatrix>> out(classes);
  for (std::size_t c = 0; c < classes; ++c) {
    if (!cnt[c]) continue;
    Matrix phi(n);
    const double inv = 1.0 / static_cast<double>(cnt[c]);  // finalize(), statistics.hpp:81-94
    for (std::size_t i = 0; i < n; ++i)
      for (std::size_t j = i; j < n; ++j) {
        const double v = sum[(c * n + i) * n + j] * inv;
        phi(i, j) = v;
        phi(j, i) = v;
      }
    out[c].emplace(std::move(phi), static_cast<std::size_t>(cnt[c]));
  }
  return out;
}

// hygt::optimize (optimizer.hpp:311-371) with the reference's types, searched on the GPU
// (hygt_optimize_f64). Gains agree with the reference to rounding; a near-tie in the search may
// pick an equivalent angle.
inline std::pair<HyGTModel, TrainingReport> optimize(const CorrelationMatrix& phi, int log2_n, int rounds,
                                                     const OptimizerConfig& config) {
  if (log2_n < 1 || log2_n > kMaxLog2N) throw ArgumentError("optimize: log2_n out of range [1, 16]");
  if (phi.n() != (std::size_t{1} << log2_n)) throw ArgumentError("optimize: dimension mismatch");
  const hygt_optimize_config c{config.restarts, config.max_sweeps, config.gain_tolerance_db, config.seed,
                               static_cast<int>(config.init_mode)};
  const std::size_t r = config.restarts > 0 ? static_cast<std::size_t>(config.restarts) : 1;
  const std::size_t s = config.max_sweeps > 0 ? static_cast<std::size_t>(config.max_sweeps) : 0;
  std::vector<double> angles(num_parameters(log2_n, rounds)), gains(r), traj(r * (s + 1));
  std::vector<int> tlen(r);
  int best = 0;
  double klt = 0.0;
  check(hygt_optimize_f64(log2_n, rounds, 1, phi.values().data().data(), &c, nullptr, angles.data(),
                          gains.data(), &best, &klt, traj.data(), tlen.data(), nullptr, nullptr));
  TrainingReport rep;
  rep.restart_gains_db = gains;
  rep.best_restart = static_cast<std::size_t>(best);
  for (std::size_t k = 0; k < r; ++k)
    rep.trajectories.emplace_back(traj.begin() + k * (s + 1), traj.begin() + k * (s + 1) + tlen[k]);
  rep.klt_gain_db = klt;
  rep.gain_ratio = klt > 1e-15 ? gains[best] / klt : 1.0;
  return {HyGTModel(log2_n, rounds, std::move(angles)), std::move(rep)};
}

// The training loop of `hygt train` (run_train, tools/hygt_main.cpp:74-120) on an in-memory
// dataset: per-class correlation on the GPU (class_correlations), the identity model for classes
// with fewer than N samples (:89-96), hygt::gpu::optimize with seed derive_seed(seed, c) (:96),
// variance_permutation (:100), and the optional angle quantisation (:110-115). `reports`, if
// given, receives one TrainingReport per class (default-constructed for identity classes).
inline ModelBundle train(const ResidualDataset& ds, int rounds, int restarts = 4, std::uint64_t seed = 0,
                         int angle_bits = 0, std::vector<TrainingReport>* reports = nullptr) {
  if (rounds < 1 || rounds > 255) throw ArgumentError("train: rounds out of range [1, 255]");
  if (angle_bits != 0 && (angle_bits < 1 || angle_bits > 8))
    throw ArgumentError("train: angle-bits must be 0 (float) or in [1, 8]");
  const std::size_t n = ds.dimension();
  const auto phis = class_correlations(ds);
  std::vector<HyGTModel> models;
  if (reports) reports->assign(ds.class_count(), TrainingReport{});
  for (std::uint16_t c = 0; c < ds.class_count(); ++c) {
    if (!phis[c] || phis[c]->sample_count() < n) {
      models.push_back(HyGTModel::zeros(ds.log2_n(), rounds));
      continue;
    }
    OptimizerConfig config;
    config.restarts = restarts;
    config.seed = derive_seed(seed, c);
    auto [model, report] = gpu::optimize(*phis[c], ds.log2_n(), rounds, config);
    models.push_back(variance_permutation(model, *phis[c]));
    if (reports) (*reports)[c] = std::move(report);
  }
  if (angle_bits > 0) {
    std::vector<QuantizedHyGTModel> quantized;
    quantized.reserve(models.size());
    for (const auto& m : models) quantized.push_back(quantize_model(m, angle_bits));
    return ModelBundle(std::move(quantized));
  }
  return ModelBundle(std::move(models));
}

}  // namespace hygt::gpu
