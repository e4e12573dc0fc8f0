// gcpb.hpp — C++ host API over the C-ABI (include/gcpb.h), mirroring the
// reference's names and error behaviour (/root/reference/proj/include/gcp):
// LossFunction, SamplerKind, RejectionStats, FitConfig, FitTraceRecord,
// fit_gcp_adam, and an Engine owning one device problem (the tensor, the
// Kruskal model's factors, the gradient and the Adam state).  Status codes
// are rethrown as the reference's exception classes.  Header-only; link with
// -lgcpb (paper_1906_01687_b200/libgcpb.so).
#pragma once

#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gcpb.h"

namespace gcpb {

inline void check(int rc, const gcpb_ctx* ctx = nullptr) {
  if (rc == GCPB_OK) return;
  const std::string msg = gcpb_last_error(ctx);
  switch (rc) {
    case GCPB_ERR_USAGE: throw std::invalid_argument(msg);
    case GCPB_ERR_DOMAIN: throw std::domain_error(msg);
    case GCPB_ERR_RANGE: throw std::out_of_range(msg);
    case GCPB_ERR_LOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

// LossFunction (include/gcp/loss.hpp:20-56).
class LossFunction {
 public:
  static LossFunction gaussian() { return LossFunction(GCPB_LOSS_GAUSSIAN); }
  static LossFunction poisson() { return LossFunction(GCPB_LOSS_POISSON); }
  static LossFunction bernoulli_odds() { return LossFunction(GCPB_LOSS_BERNOULLI_ODDS); }
  static LossFunction gamma() { return LossFunction(GCPB_LOSS_GAMMA); }
  static LossFunction beta_half() { return LossFunction(GCPB_LOSS_BETA_HALF); }
  static LossFunction huber(double delta) {
    if (!(delta > 0.0)) throw std::invalid_argument("huber: delta must be > 0");
    return LossFunction(GCPB_LOSS_HUBER, delta);
  }
  static LossFunction parse(const std::string& token) {  // loss.cpp:21-40
    if (token == "gaussian") return gaussian();
    if (token == "poisson") return poisson();
    if (token == "bernoulli-odds") return bernoulli_odds();
    if (token == "gamma") return gamma();
    if (token == "beta-half") return beta_half();
    if (token.rfind("huber:", 0) == 0) {
      const std::string arg = token.substr(6);
      std::size_t pos = 0;
      double delta = 0.0;
      try {
        delta = std::stod(arg, &pos);
      } catch (const std::exception&) {
        throw std::invalid_argument("huber: bad delta '" + arg + "'");
      }
      if (pos != arg.size()) throw std::invalid_argument("huber: bad delta '" + arg + "'");
      return huber(delta);
    }
    throw std::invalid_argument("unknown loss '" + token + "'");
  }
  int kind() const { return c_.kind; }
  double delta() const { return c_.delta; }
  double value(double x, double m) const { return gcpb_loss_value(&c_, x, m); }
  double deriv(double x, double m) const { return gcpb_loss_deriv(&c_, x, m); }
  std::optional<double> default_lower_bound() const {  // loss.cpp:112-124
    if (c_.kind == GCPB_LOSS_GAUSSIAN || c_.kind == GCPB_LOSS_HUBER) return std::nullopt;
    return 0.0;
  }
  const gcpb_loss* c() const { return &c_; }

 private:
  explicit LossFunction(int kind, double delta = 0.0) : c_{kind, delta} {}
  gcpb_loss c_;
};

// SamplerKind (include/gcp/samplers.hpp:31-51).
struct SamplerKind {
  gcpb_sampler c{GCPB_UNIFORM, 0, 0, 0, 1.1};
  static SamplerKind uniform(int64_t s) {
    SamplerKind k;
    k.c = {GCPB_UNIFORM, s, 0, 0, 1.1};
    k.validate();
    return k;
  }
  static SamplerKind stratified(int64_t p, int64_t q, double rho = 1.1) {
    SamplerKind k;
    k.c = {GCPB_STRATIFIED, 0, p, q, rho};
    k.validate();
    return k;
  }
  static SamplerKind semi_stratified(int64_t p, int64_t q) {
    SamplerKind k;
    k.c = {GCPB_SEMI_STRATIFIED, 0, p, q, 1.1};
    k.validate();
    return k;
  }
  static SamplerKind from_token(const std::string& token, int64_t total) {  // samplers.cpp:37-45
    if (token == "uniform") return uniform(total);
    if (token == "stratified") return stratified(total / 2, total - total / 2);
    if (token == "semi-stratified") return semi_stratified(total / 2, total - total / 2);
    throw std::invalid_argument("unknown sampler '" + token +
                                "' (expected uniform, stratified, or semi-stratified)");
  }
  void validate() const {  // samplers.cpp:56-67
    if (c.strategy == GCPB_UNIFORM) {
      if (c.num_samples < 1) throw std::invalid_argument("uniform sampler: s must be >= 1");
      return;
    }
    if (c.nonzero_samples < 0 || c.zero_samples < 0 || c.nonzero_samples + c.zero_samples < 1)
      throw std::invalid_argument("sampler: need p, q >= 0 and p + q >= 1");
    if (c.strategy == GCPB_STRATIFIED && !(c.oversample > 1.0))
      throw std::invalid_argument("stratified sampler: oversample rate must be > 1");
  }
};

using RejectionStats = gcpb_stats;  // tested, accepted, rejected

struct FitConfig {  // include/gcp/optimizer.hpp:42-65
  int64_t rank = 2;
  SamplerKind sampler = SamplerKind::uniform(1);
  double learning_rate = 0.01;
  double beta1 = 0.9, beta2 = 0.999, epsilon = 1e-8;
  int64_t epoch_iters = 1000;
  int64_t max_bad_epochs = 1;
  double decay = 0.1;
  std::optional<double> lower_bound;  // empty: the loss's default bound
  int64_t estimator_samples = 100000;
  int estimator_kind = -1;            // -1: by tensor kind
  int64_t max_epochs = 100;
  uint64_t seed = 0;
  bool keep_factors = false;
  bool reference_stream = false;      // RefStream: the reference's own draws
};

struct FitTraceRecord {
  int64_t epoch;
  double loss_estimate;
  double learning_rate;
  double seconds;
  bool accepted;
};

// RngStream (include/gcp/rng.hpp:15-47) as the state the device generators
// consume and advance.
class RngStream {
 public:
  explicit RngStream(uint64_t seed) { check(gcpb_rng_seed(seed, &s_)); }
  RngStream split(uint64_t label) const {
    RngStream c(0);
    check(gcpb_rng_split(&s_, label, &c.s_));
    return c;
  }
  gcpb_rng* c() { return &s_; }
  uint64_t key() const { return s_.key; }
  uint64_t counter() const { return s_.counter; }

 private:
  gcpb_rng s_{};
};

// BinaryProblemSpec (include/gcp/synthetic.hpp:22-31); shape and rank are the engine's.
struct BinaryProblemSpec {
  double delta = 0.15;
  double p_high = 0.9;
  double p_low = 0.0025;
};

struct BiasVariance {  // samplers.hpp BiasVariance
  double bias = 0.0;
  double variance = 0.0;
};

// A coordinate list read from / written to a file (io.hpp).
struct CooTensor {
  std::vector<int64_t> dims;
  std::vector<int64_t> coords;  // nnz x d, 0-based
  std::vector<double> values;
};

inline CooTensor take_coo(gcpb_coo& c) {
  CooTensor t;
  t.dims.assign(c.dims, c.dims + c.d);
  t.coords.assign(c.coords, c.coords + c.nnz * c.d);
  t.values.assign(c.values, c.values + c.nnz);
  gcpb_coo_free(&c);
  return t;
}

inline gcpb_coo view_coo(const CooTensor& t) {
  gcpb_coo c{};
  c.d = static_cast<int>(t.dims.size());
  for (int k = 0; k < c.d && k < 16; ++k) c.dims[k] = t.dims[k];
  c.nnz = static_cast<int64_t>(t.values.size());
  c.coords = const_cast<int64_t*>(t.coords.data());
  c.values = const_cast<double*>(t.values.data());
  return c;
}

// read_tns / write_tns (io.cpp:75-151): entries in file order; Engine::set_sparse
// normalises them like the SparseTensor constructor.
inline CooTensor read_tns(const std::string& path, int threads = 0) {
  gcpb_coo c{};
  check(gcpb_tns_read(path.c_str(), threads, &c));
  return take_coo(c);
}
inline void write_tns(const CooTensor& t, const std::string& path) {
  const gcpb_coo c = view_coo(t);
  check(gcpb_tns_write(path.c_str(), &c));
}
inline CooTensor read_coo(const std::string& path, int threads = 0) {
  gcpb_coo c{};
  check(gcpb_coo_read(path.c_str(), threads, &c));
  return take_coo(c);
}
inline void write_coo(const CooTensor& t, const std::string& path) {
  const gcpb_coo c = view_coo(t);
  check(gcpb_coo_write(path.c_str(), &c));
}

// read_model / write_model (io.cpp:153-193): factors as n_k x r row-major.
inline std::vector<std::vector<double>> read_model(const std::string& path,
                                                   std::vector<int64_t>* dims_out = nullptr) {
  int d = 0;
  int64_t dims[16] = {};
  int64_t r = 0;
  check(gcpb_model_read_header(path.c_str(), &d, dims, &r));
  size_t n = 0;
  for (int k = 0; k < d; ++k) n += static_cast<size_t>(dims[k] * r);
  std::vector<double> flat(n);
  check(gcpb_model_read(path.c_str(), flat.data()));
  std::vector<std::vector<double>> out(static_cast<size_t>(d));
  size_t at = 0;
  for (int k = 0; k < d; ++k) {
    out[k].assign(flat.begin() + at, flat.begin() + at + dims[k] * r);
    at += static_cast<size_t>(dims[k] * r);
  }
  if (dims_out) dims_out->assign(dims, dims + d);
  return out;
}
inline void write_model(const std::vector<std::vector<double>>& factors,
                        const std::vector<int64_t>& dims, int64_t rank, const std::string& path) {
  std::vector<double> flat;
  for (const auto& f : factors) flat.insert(flat.end(), f.begin(), f.end());
  check(gcpb_model_write(path.c_str(), static_cast<int>(dims.size()), dims.data(), rank,
                         flat.data()));
}

// One stochastic-GCP problem on one GPU.
class Engine {
 public:
  Engine(const std::vector<int64_t>& dims, int64_t rank, int dtype = GCPB_F64, int device = 0)
      : dims_(dims), rank_(rank) {
    check(gcpb_create(device, dtype, static_cast<int>(dims.size()), dims.data(), rank, &ctx_));
  }
  ~Engine() { gcpb_destroy(ctx_); }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  Engine(Engine&& o) noexcept : ctx_(std::exchange(o.ctx_, nullptr)), dims_(o.dims_), rank_(o.rank_) {}

  gcpb_ctx* handle() const { return ctx_; }
  int ndims() const { return static_cast<int>(dims_.size()); }
  int64_t rank() const { return rank_; }

  // SparseTensor(shape, indices, values): coords nnz x d row-major.
  void set_sparse(const std::vector<int64_t>& coords, const std::vector<double>& values) {
    if (coords.size() != values.size() * dims_.size())
      throw std::invalid_argument("sparse tensor: index/value count mismatch");
    check(gcpb_set_sparse(ctx_, static_cast<int64_t>(values.size()), coords.data(), values.data()),
          ctx_);
  }
  void set_dense(const std::vector<double>& values, int storage = GCPB_STORE_F64) {
    check(gcpb_set_dense(ctx_, values.data(), storage), ctx_);
  }
  double tensor_norm() const {
    double v = 0.0;
    check(gcpb_tensor_norm(ctx_, &v), ctx_);
    return v;
  }

  // Factors / gradient as one n_k x r row-major matrix per mode.
  void set_factors(const std::vector<std::vector<double>>& f) {
    for (int k = 0; k < ndims(); ++k) check(gcpb_set_factors(ctx_, k, f.at(k).data()), ctx_);
  }
  std::vector<std::vector<double>> factors() const { return get(gcpb_get_factors); }
  std::vector<std::vector<double>> gradient() const { return get(gcpb_get_grad); }

  // draw_gradient_samples + mttkrp_sampled_all, fused on the device.
  RejectionStats stoch_grad(const SamplerKind& s, const LossFunction& loss, uint64_t seed,
                            uint64_t iter) {
    RejectionStats st{0, 0, 0};
    check(gcpb_stoch_grad(ctx_, &s.c, loss.c(), seed, iter, &st), ctx_);
    return st;
  }
  void adam_step(double lr, double beta1 = 0.9, double beta2 = 0.999, double eps = 1e-8,
                 std::optional<double> lb = std::nullopt) {
    const gcpb_adam a{lr, beta1, beta2, eps, lb.has_value() ? 1 : 0, lb.value_or(0.0)};
    check(gcpb_adam_step(ctx_, &a), ctx_);
  }
  void step(const SamplerKind& s, const LossFunction& loss, uint64_t seed, uint64_t iter, double lr,
            std::optional<double> lb = std::nullopt) {
    const gcpb_adam a{lr, 0.9, 0.999, 1e-8, lb.has_value() ? 1 : 0, lb.value_or(0.0)};
    check(gcpb_step(ctx_, &s.c, loss.c(), seed, iter, &a), ctx_);
  }

  // Exact gradients (kernels.cpp:170-235) -> gradient().
  void gradient_full(const LossFunction& loss) { check(gcpb_gradient_full(ctx_, loss.c()), ctx_); }
  void gradient_poisson_implicit(const LossFunction& loss) {
    check(gcpb_gradient_poisson_implicit(ctx_, loss.c()), ctx_);
  }
  // empirical_bias_variance (samplers.cpp:134-168); exact empty -> gradient_full.
  BiasVariance bias_variance(const SamplerKind& s, const LossFunction& loss, int64_t trials,
                             uint64_t seed, const std::vector<double>& exact = {}) {
    BiasVariance bv;
    check(gcpb_bias_variance(ctx_, &s.c, loss.c(), trials, seed,
                             exact.empty() ? nullptr : exact.data(), &bv.bias, &bv.variance),
          ctx_);
    return bv;
  }
  // Synthetic problems (synthetic.cpp), generated in HBM; returns the truth.
  std::vector<double> gen_gamma_problem(RngStream& rng, int storage = GCPB_STORE_F64) {
    std::vector<double> truth(truth_size());
    check(gcpb_gen_gamma_problem(ctx_, rng.c(), storage, truth.data()), ctx_);
    return truth;
  }
  std::vector<double> gen_binary_problem(const BinaryProblemSpec& spec, RngStream& rng) {
    std::vector<double> truth(truth_size());
    const gcpb_binary_spec cs{spec.delta, spec.p_high, spec.p_low};
    check(gcpb_gen_binary_problem(ctx_, &cs, rng.c(), truth.data()), ctx_);
    return truth;
  }
  void set_sparse(const CooTensor& t) { set_sparse(t.coords, t.values); }
  int64_t nnz() const { return gcpb_nnz(ctx_); }

 private:
  template <typename F>
  std::vector<std::vector<double>> get(F fn) const {
    std::vector<std::vector<double>> out(dims_.size());
    for (int k = 0; k < ndims(); ++k) {
      out[k].resize(static_cast<size_t>(dims_[k] * rank_));
      check(fn(ctx_, k, out[k].data()), ctx_);
    }
    return out;
  }
  size_t truth_size() const {
    size_t n = 0;
    for (int64_t d : dims_) n += static_cast<size_t>(d * rank_);
    return n;
  }
  gcpb_ctx* ctx_ = nullptr;
  std::vector<int64_t> dims_;
  int64_t rank_;
};

struct FitResult {
  std::vector<std::vector<double>> model;
  std::vector<FitTraceRecord> trace;
  double final_loss_estimate = 0.0;
};

// write_trace_csv (io.cpp:252-260).
inline void write_trace_csv(const std::vector<FitTraceRecord>& trace, const std::string& path) {
  std::vector<gcpb_trace_record> recs;
  for (const auto& t : trace)
    recs.push_back({t.epoch, t.loss_estimate, t.learning_rate, t.seconds, t.accepted ? 1 : 0});
  check(gcpb_trace_write_csv(path.c_str(), recs.data(), static_cast<int64_t>(recs.size())));
}

// fit_gcp_adam (src/optimizer.cpp:68-158), device-resident epochs.
inline FitResult fit_gcp_adam(Engine& e, const LossFunction& loss, const FitConfig& cfg) {
  if (cfg.rank != e.rank()) throw std::invalid_argument("fit: rank must match the engine");
  gcpb_fit_config c{};
  c.sampler = cfg.sampler.c;
  c.learning_rate = cfg.learning_rate;
  c.beta1 = cfg.beta1;
  c.beta2 = cfg.beta2;
  c.epsilon = cfg.epsilon;
  c.epoch_iters = cfg.epoch_iters;
  c.max_bad_epochs = cfg.max_bad_epochs;
  c.decay = cfg.decay;
  c.lower_bound_mode = cfg.lower_bound.has_value() ? 1 : 0;
  c.lower_bound = cfg.lower_bound.value_or(0.0);
  c.estimator_samples = cfg.estimator_samples;
  c.estimator_kind = cfg.estimator_kind;
  c.max_epochs = cfg.max_epochs;
  c.seed = cfg.seed;
  c.keep_factors = cfg.keep_factors ? 1 : 0;
  c.draw_stream = cfg.reference_stream ? 1 : 0;
  std::vector<gcpb_trace_record> tr(static_cast<size_t>(cfg.max_epochs + 1));
  int64_t n = 0;
  double fin = 0.0;
  check(gcpb_fit_gcp_adam(e.handle(), loss.c(), &c, tr.data(), static_cast<int64_t>(tr.size()), &n,
                          &fin),
        e.handle());
  FitResult r;
  for (int64_t i = 0; i < n && i < static_cast<int64_t>(tr.size()); ++i)
    r.trace.push_back({tr[i].epoch, tr[i].loss_estimate, tr[i].learning_rate, tr[i].seconds,
                       tr[i].accepted != 0});
  r.model = e.factors();
  r.final_loss_estimate = fin;
  return r;
}

}  // namespace gcpb
