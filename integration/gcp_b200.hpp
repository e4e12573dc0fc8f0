// gcp_b200.hpp -- the reference-side binding of the B200 engine.
//
// What a maintainer adds to the reference (/root/reference/proj) to run its
// hot path on a B200: a header over the C-ABI (include/gcpb.h) that speaks the
// reference's own types (Shape, SparseTensor, DenseTensor, TensorView,
// KruskalModel, LossFunction, SamplerKind, EstimatorSamples, FitConfig,
// FitResult, RngStream) and rethrows its exception classes.  Compile with
//   -I<reference>/include -I<repo>/include  and link  -lgcpb.
// tests/cpp/ref_binding_check.cpp compiles it against the reference headers
// and checks gcp::b200::fit_gcp_adam against the reference's own
// gcp::fit_gcp_adam (src/optimizer.cpp:68-158) for all six losses.
#pragma once

#include <chrono>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "gcp/kernels.hpp"
#include "gcp/kruskal.hpp"
#include "gcp/loss.hpp"
#include "gcp/optimizer.hpp"
#include "gcp/rng.hpp"
#include "gcp/samplers.hpp"
#include "gcp/tensor.hpp"
#include "gcpb.h"

namespace gcp::b200 {

// Status codes -> the reference's exception classes.
inline void check(int rc, const gcpb_ctx* c) {
  if (rc == GCPB_OK) return;
  const std::string msg = gcpb_last_error(c);
  switch (rc) {
    case GCPB_ERR_USAGE: throw std::invalid_argument(msg);
    case GCPB_ERR_DOMAIN: throw std::domain_error(msg);
    case GCPB_ERR_RANGE: throw std::out_of_range(msg);
    case GCPB_ERR_LOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

// LossFunction (loss.hpp:20-56) -> gcpb_loss.  The reference keeps the Huber
// half-width private (loss.hpp:55); for |x - m| > delta its derivative is
// -2 delta sign(x - m) (loss.cpp:103-106), so deriv(0, 1e300) = 2 delta
// exactly and delta is recovered without rounding.
inline gcpb_loss to_c(const LossFunction& loss) {
  gcpb_loss l{static_cast<int32_t>(loss.kind()), 0.0};
  if (loss.kind() == LossKind::kHuber) l.delta = loss.deriv(0.0, 1e300) / 2.0;
  return l;
}

// SamplerKind (samplers.hpp:31-51) -> gcpb_sampler (same enum order).
inline gcpb_sampler to_c(const SamplerKind& s) {
  return gcpb_sampler{static_cast<int32_t>(s.strategy), s.num_samples, s.nonzero_samples,
                      s.zero_samples, s.oversample};
}

// The state of an RngStream as the device's RefStream mode takes it.  The
// reference draws u = mix64(key + phi * ++counter) (rng.cpp:43-45); mix64 is
// the invertible SplitMix64 finalizer, so one draw of a COPY gives
// key + phi * (counter + 1), i.e. the stream's base key + phi * counter,
// without touching the caller's stream.  RefStream draw j of a call is then
// mix64(base + phi * (device_counter + j + 1)) with device_counter = 0.
inline std::uint64_t unmix64(std::uint64_t z) {
  z = z ^ (z >> 31) ^ (z >> 62);
  z *= 0x319642b2d24d8ec3ull;  // inverse of 0x94d049bb133111eb mod 2^64
  z = z ^ (z >> 27) ^ (z >> 54);
  z *= 0x96de1b173f119089ull;  // inverse of 0xbf58476d1ce4e5b9 mod 2^64
  z = z ^ (z >> 30) ^ (z >> 60);
  return z;
}
inline std::uint64_t stream_base(RngStream copy) {
  return unmix64(copy.next_u64()) - 0x9e3779b97f4a7c15ull;
}

// One problem on one GPU: the tensor, the model's factors, the gradient, the
// Adam moments and the estimator set, all device-resident (include/gcpb.h).
class Engine {
 public:
  Engine(const Shape& shape, std::int64_t rank, int dtype = GCPB_F64, int device = 0)
      : shape_(shape), rank_(rank) {
    check(gcpb_create(device, dtype, shape.ndims(), shape.dims().data(), rank, &c_), nullptr);
  }
  ~Engine() { gcpb_destroy(c_); }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  gcpb_ctx* get() const { return c_; }

  // SparseTensor: the reference's normalised order (tensor.cpp:10-41) is kept,
  // so nonzero ordinal e names the same entry on both sides.
  void set_tensor(const SparseTensor& x) {
    std::vector<std::int64_t> coords;
    coords.reserve(static_cast<std::size_t>(x.nnz() * x.ndims()));
    for (std::int64_t e = 0; e < x.nnz(); ++e)
      for (std::int64_t i : x.index(e)) coords.push_back(i);
    check(gcpb_set_sparse(c_, x.nnz(), coords.data(), x.values().data()), c_);
  }
  void set_tensor(const DenseTensor& x) {  // first-mode-fastest values
    check(gcpb_set_dense(c_, x.values().data(), GCPB_STORE_F64), c_);
  }
  // TensorView has no dense accessor: a dense view is read entry by entry
  // (the reference caps dense tensors at 1e8 entries, tensor.hpp:54).
  void set_tensor(const TensorView& x) {
    if (x.is_sparse()) return set_tensor(*x.as_sparse());
    const Shape& s = x.shape();
    std::vector<double> v(static_cast<std::size_t>(s.total()));
    std::vector<std::int64_t> idx(static_cast<std::size_t>(s.ndims()), 0);
    for (double& out : v) {
      out = x.value_at(idx);
      for (int k = 0; k < s.ndims(); ++k) {
        if (++idx[static_cast<std::size_t>(k)] < s.dim(k)) break;
        idx[static_cast<std::size_t>(k)] = 0;
      }
    }
    check(gcpb_set_dense(c_, v.data(), GCPB_STORE_F64), c_);
  }

  void set_model(const KruskalModel& m) {  // row-major n_k x r (kruskal.hpp:15)
    for (int k = 0; k < m.ndims(); ++k) check(gcpb_set_factors(c_, k, m.factor(k).data()), c_);
  }
  KruskalModel model() const {
    std::vector<Matrix> f;
    for (int k = 0; k < shape_.ndims(); ++k) {
      f.emplace_back(shape_.dim(k), rank_);
      check(gcpb_get_factors(c_, k, f.back().data()), c_);
    }
    return KruskalModel(std::move(f));
  }
  void moments(std::vector<Matrix>& first, std::vector<Matrix>& second) const {
    first.clear();
    second.clear();
    for (int k = 0; k < shape_.ndims(); ++k) {
      first.emplace_back(shape_.dim(k), rank_);
      second.emplace_back(shape_.dim(k), rank_);
      check(gcpb_get_moment(c_, 0, k, first.back().data()), c_);
      check(gcpb_get_moment(c_, 1, k, second.back().data()), c_);
    }
  }

  // EstimatorSamples (samplers.hpp:257-351): the reference's own fixed draws.
  void set_estimator(const EstimatorSamples& est) {
    const std::int64_t n = est.size(), d = shape_.ndims();
    std::vector<std::int64_t> idx(static_cast<std::size_t>(n * d));
    std::vector<double> x(static_cast<std::size_t>(n)), w(static_cast<std::size_t>(n));
    for (std::int64_t e = 0; e < n; ++e) {
      const auto ix = est.index(e);
      for (std::int64_t k = 0; k < d; ++k) idx[static_cast<std::size_t>(e * d + k)] = ix[k];
      x[static_cast<std::size_t>(e)] = est.data_value(e);
      w[static_cast<std::size_t>(e)] = est.weight(e);
    }
    check(gcpb_estimator_set(c_, n, idx.data(), x.data(), w.data()), c_);
  }
  double estimate(const LossFunction& loss) {  // EstimatorSamples::estimate
    const gcpb_loss l = to_c(loss);
    double f = 0.0;
    check(gcpb_estimate(c_, &l, &f), c_);
    return f;
  }

  // Draws continue the reference stream `rng` (RefStream mode).
  void follow(const RngStream& rng) {
    key_ = stream_base(rng);
    check(gcpb_set_draw_stream(c_, 1, 0), c_);
  }
  // draw_gradient_samples + mttkrp_sampled_all + adam_step, n times
  // (optimizer.cpp:116-119), replayed on the device as one CUDA graph.
  void iterate(const SamplerKind& sk, const LossFunction& loss, const gcpb_adam& adam,
               std::int64_t n) {
    const gcpb_sampler s = to_c(sk);
    const gcpb_loss l = to_c(loss);
    check(gcpb_run_steps(c_, &s, &l, key_, 0, n, &adam), c_);
    check(gcpb_synchronize(c_), c_);
  }
  void snapshot_save() { check(gcpb_snapshot_save(c_), c_); }
  void snapshot_restore() { check(gcpb_snapshot_restore(c_), c_); }
  std::int64_t iterations() const {
    std::int64_t t = 0;
    check(gcpb_get_iterations(c_, &t), c_);
    return t;
  }

 private:
  gcpb_ctx* c_ = nullptr;
  Shape shape_;
  std::int64_t rank_;
  std::uint64_t key_ = 0;
};

// fit_gcp_adam (optimizer.cpp:68-153) with the epoch loop's iterations on the
// device: the reference's own init (init split, random_uniform,
// scale_norm_to), its own estimator draws (estimator split), its own gradient
// stream (gradients split) reproduced by the device's RefStream mode, and
// its accept / roll back / decay logic on the host.  The result matches
// gcp::fit_gcp_adam(x, loss, cfg, rng) up to floating-point summation order
// (dtype GCPB_F64); GCPB_F32 is the fast path.
inline FitResult fit_gcp_adam(const TensorView& x, const LossFunction& loss, const FitConfig& cfg,
                              RngStream& rng, int dtype = GCPB_F64, int device = 0) {
  cfg.validate();
  const auto start = std::chrono::steady_clock::now();
  auto since = [](std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };
  FitConfig effective = cfg;
  if (!effective.lower_bound.has_value()) effective.lower_bound = loss.default_lower_bound();
  RngStream init_rng = rng.split("init");
  RngStream estimator_rng = rng.split("estimator");
  RngStream gradient_rng = rng.split("gradients");
  KruskalModel model = KruskalModel::random_uniform(x.shape(), cfg.rank, init_rng);
  const double data_norm = x.norm();
  if (data_norm > 0.0) model.scale_norm_to(data_norm);

  Engine eng(x.shape(), cfg.rank, dtype, device);
  eng.set_tensor(x);
  eng.set_model(model);
  const bool custom = static_cast<bool>(cfg.estimate_override);
  if (!custom) {
    const EstimatorSamples::Kind kind = cfg.estimator_kind.value_or(
        x.is_sparse() ? EstimatorSamples::Kind::kStratified : EstimatorSamples::Kind::kUniform);
    eng.set_estimator(draw_estimator_samples(x, kind, cfg.estimator_samples, estimator_rng));
  }
  auto estimate = [&]() {
    return custom ? cfg.estimate_override(eng.model()) : eng.estimate(loss);
  };
  eng.follow(gradient_rng);
  check(gcpb_adam_reset(eng.get()), eng.get());
  double learning_rate = cfg.learning_rate;
  std::int64_t bad_epochs = 0;
  gcpb_adam ad{learning_rate, cfg.beta1, cfg.beta2, cfg.epsilon,
               effective.lower_bound.has_value() ? 1 : 0, effective.lower_bound.value_or(0.0)};

  double best_estimate = estimate();
  if (!std::isfinite(best_estimate))
    throw std::runtime_error("fit: initial loss estimate is not finite (" +
                             std::to_string(best_estimate) + ")");
  eng.snapshot_save();  // factors, moments, iteration counter
  FitResult result;
  result.trace.records.push_back({0, best_estimate, learning_rate, since(start), true});
  if (cfg.on_epoch) cfg.on_epoch(result.trace.records.back());
  for (std::int64_t epoch = 1; epoch <= cfg.max_epochs; ++epoch) {
    const auto epoch_start = std::chrono::steady_clock::now();
    const double alpha_used = learning_rate;
    ad.learning_rate = learning_rate;
    eng.iterate(cfg.sampler, loss, ad, cfg.epoch_iters);
    const double new_estimate = estimate();
    if (!std::isfinite(new_estimate))
      throw std::runtime_error("fit: loss estimate became non-finite at epoch " +
                               std::to_string(epoch));
    const double secs = since(epoch_start);
    if (new_estimate <= best_estimate) {
      best_estimate = new_estimate;
      eng.snapshot_save();
      result.trace.records.push_back({epoch, new_estimate, alpha_used, secs, true});
      if (cfg.on_epoch) cfg.on_epoch(result.trace.records.back());
    } else {
      eng.snapshot_restore();  // the gradient stream is not rewound (optimizer.cpp:129-140)
      learning_rate *= cfg.decay;
      ++bad_epochs;
      result.trace.records.push_back({epoch, new_estimate, alpha_used, secs, false});
      if (cfg.on_epoch) cfg.on_epoch(result.trace.records.back());
      if (bad_epochs > cfg.max_bad_epochs) break;
    }
  }
  result.model = eng.model();
  result.final_loss_estimate = best_estimate;
  eng.moments(result.final_state.first_moment, result.final_state.second_moment);
  result.final_state.iterations = eng.iterations();
  result.final_state.learning_rate = learning_rate;
  result.final_state.bad_epochs = bad_epochs;
  return result;
}

inline FitResult fit_gcp_adam(const TensorView& x, const LossFunction& loss, const FitConfig& cfg,
                              int dtype = GCPB_F64, int device = 0) {
  RngStream rng(cfg.seed);
  return fit_gcp_adam(x, loss, cfg, rng, dtype, device);
}

}  // namespace gcp::b200
