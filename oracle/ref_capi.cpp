// ref_capi.cpp — TEST INFRASTRUCTURE ONLY (never shipped, never on the product
// path).  A thin extern "C" wrapper over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile against
// oracle/eigen_shim) so pytest can call the reference's own code through ctypes:
//   * golden vectors (RngStream known answers, loss values),
//   * the reference samplers driven by a scripted draw sequence
//     (tests/oracles.hpp:23-31 ScriptedRng semantics: script[at++] % n),
//   * mttkrp_sampled_all / adam_step / EstimatorSamples::estimate / fit_gcp_adam,
//   * the CPU baseline timings used by bench.py --impl reference.
// Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
// legs may load the resulting oracle/_ref/libgcpref.so.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <iostream>  // static libstdc++ in the .so: pull in the stream/locale init
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "gcp/io.hpp"
#include "gcp/kernels.hpp"
#include "gcp/kruskal.hpp"
#include "gcp/loss.hpp"
#include "gcp/optimizer.hpp"
#include "gcp/rng.hpp"
#include "gcp/samplers.hpp"
#include "gcp/shape.hpp"
#include "gcp/scoring.hpp"
#include "gcp/synthetic.hpp"
#include "oracles.hpp"  // the reference's own test fixtures (tests/oracles.hpp)
#include "gcp/tensor.hpp"

namespace {

thread_local std::string g_err;

int fail(int code, const char* what) {
  g_err = what;
  return code;
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(2, e.what());
  } catch (const std::domain_error& e) {
    return fail(3, e.what());
  } catch (const std::out_of_range& e) {
    return fail(4, e.what());
  } catch (const std::logic_error& e) {
    return fail(5, e.what());
  } catch (const std::exception& e) {
    return fail(1, e.what());
  }
}

struct ScriptedRng {  // same contract as tests/oracles.hpp:23-31
  const std::uint64_t* script = nullptr;
  std::int64_t len = 0;
  std::int64_t at = 0;
  std::uint64_t next_below(std::uint64_t n) {
    if (at >= len) throw std::logic_error("ScriptedRng: script exhausted");
    return script[at++] % n;
  }
};

gcp::Shape make_shape(int d, const std::int64_t* dims) {
  return gcp::Shape(std::vector<std::int64_t>(dims, dims + d));
}

gcp::KruskalModel make_model(int d, const std::int64_t* dims, std::int64_t r, const double* flat) {
  gcp::KruskalModel model(make_shape(d, dims), r);
  std::int64_t at = 0;
  for (int k = 0; k < d; ++k) {
    gcp::Matrix& f = model.factor(k);
    for (Eigen::Index i = 0; i < f.rows(); ++i)
      for (Eigen::Index j = 0; j < f.cols(); ++j) f(i, j) = flat[at++];
  }
  return model;
}

void flatten_model(const gcp::KruskalModel& model, double* out) {
  std::int64_t at = 0;
  for (int k = 0; k < model.ndims(); ++k) {
    const gcp::Matrix& f = model.factor(k);
    for (Eigen::Index i = 0; i < f.rows(); ++i)
      for (Eigen::Index j = 0; j < f.cols(); ++j) out[at++] = f(i, j);
  }
}

void flatten_mats(const std::vector<gcp::Matrix>& mats, double* out) {
  std::int64_t at = 0;
  for (const gcp::Matrix& f : mats)
    for (Eigen::Index i = 0; i < f.rows(); ++i)
      for (Eigen::Index j = 0; j < f.cols(); ++j) out[at++] = f(i, j);
}

void unflatten_mats(std::vector<gcp::Matrix>& mats, const double* in) {
  std::int64_t at = 0;
  for (gcp::Matrix& f : mats)
    for (Eigen::Index i = 0; i < f.rows(); ++i)
      for (Eigen::Index j = 0; j < f.cols(); ++j) f(i, j) = in[at++];
}

gcp::LossFunction make_loss(int kind, double delta) {
  switch (kind) {
    case 0: return gcp::LossFunction::gaussian();
    case 1: return gcp::LossFunction::poisson();
    case 2: return gcp::LossFunction::bernoulli_odds();
    case 3: return gcp::LossFunction::gamma();
    case 4: return gcp::LossFunction::beta_half();
    case 5: return gcp::LossFunction::huber(delta);
  }
  throw std::invalid_argument("ref_capi: unknown loss kind");
}

gcp::SamplerKind make_kind(int strategy, std::int64_t s, std::int64_t p, std::int64_t q, double rho) {
  gcp::SamplerKind kind;
  kind.strategy = static_cast<gcp::SamplerKind::Strategy>(strategy);
  kind.num_samples = s;
  kind.nonzero_samples = p;
  kind.zero_samples = q;
  kind.oversample = rho;
  return kind;
}

// A tensor handle is either sparse or dense.
struct TensorH {
  std::unique_ptr<gcp::SparseTensor> sparse;
  std::unique_ptr<gcp::DenseTensor> dense;
  gcp::TensorView view() const {
    if (sparse) return gcp::TensorView(*sparse);
    return gcp::TensorView(*dense);
  }
};

void copy_samples(const gcp::GradientSamples& gs, std::int64_t cap, std::int64_t* idx_out,
                  double* y_out, std::int64_t* n_out) {
  const std::int64_t n = gs.size();
  *n_out = n;
  if (n > cap) throw std::length_error("ref_capi: output capacity too small");
  const int d = gs.ndims();
  for (std::int64_t e = 0; e < n; ++e) {
    const auto idx = gs.index(e);
    for (int k = 0; k < d; ++k) idx_out[e * d + k] = idx[static_cast<std::size_t>(k)];
    y_out[e] = gs.value(e);
  }
}

double secs(std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- RngStream (rng.hpp:15-47) ----------------------------------------------
void* ref_rng_new(std::uint64_t seed) { return new gcp::RngStream(seed); }
void ref_rng_free(void* h) { delete static_cast<gcp::RngStream*>(h); }
void* ref_rng_split_label(void* h, const char* label) {
  return new gcp::RngStream(static_cast<gcp::RngStream*>(h)->split(std::string_view(label)));
}
void* ref_rng_split_u64(void* h, std::uint64_t label) {
  return new gcp::RngStream(static_cast<gcp::RngStream*>(h)->split(label));
}
std::uint64_t ref_rng_next_u64(void* h) { return static_cast<gcp::RngStream*>(h)->next_u64(); }
double ref_rng_next_double(void* h) { return static_cast<gcp::RngStream*>(h)->next_double(); }
int ref_rng_next_below(void* h, std::uint64_t n, std::uint64_t* out) {
  return guard([&] { *out = static_cast<gcp::RngStream*>(h)->next_below(n); });
}

// ---- LossFunction (loss.cpp:64-124) -------------------------------------------
int ref_loss_value(int kind, double delta, double x, double m, double* out) {
  return guard([&] { *out = make_loss(kind, delta).value(x, m); });
}
int ref_loss_deriv(int kind, double delta, double x, double m, double* out) {
  return guard([&] { *out = make_loss(kind, delta).deriv(x, m); });
}
int ref_loss_parse(const char* token, int* kind, double* has_bound, double* bound) {
  return guard([&] {
    const gcp::LossFunction l = gcp::LossFunction::parse(token);
    *kind = static_cast<int>(l.kind());
    const auto b = l.default_lower_bound();
    *has_bound = b.has_value() ? 1.0 : 0.0;
    *bound = b.value_or(0.0);
  });
}

// ---- tensors --------------------------------------------------------------------
int ref_sparse_new(int d, const std::int64_t* dims, std::int64_t n, const std::int64_t* coords,
                   const double* values, void** out) {
  return guard([&] {
    std::vector<gcp::MultiIndex> idx;
    idx.reserve(static_cast<std::size_t>(n));
    std::vector<double> vals(values, values + n);
    for (std::int64_t e = 0; e < n; ++e) {
      idx.emplace_back(std::span<const std::int64_t>(coords + e * d, static_cast<std::size_t>(d)));
    }
    auto h = std::make_unique<TensorH>();
    h->sparse = std::make_unique<gcp::SparseTensor>(make_shape(d, dims), idx, vals);
    *out = h.release();
  });
}
int ref_dense_new(int d, const std::int64_t* dims, const double* values, void** out) {
  return guard([&] {
    auto h = std::make_unique<TensorH>();
    h->dense = std::make_unique<gcp::DenseTensor>(make_shape(d, dims));
    auto v = h->dense->values();
    std::memcpy(v.data(), values, v.size() * sizeof(double));
    *out = h.release();
  });
}
void ref_tensor_free(void* h) { delete static_cast<TensorH*>(h); }
std::int64_t ref_sparse_nnz(void* h) { return static_cast<TensorH*>(h)->sparse->nnz(); }
// Normalized COO (tensor.cpp:10-41): sorted coords, summed values.
int ref_sparse_export(void* h, std::int64_t* coords_out, double* values_out) {
  return guard([&] {
    const gcp::SparseTensor& x = *static_cast<TensorH*>(h)->sparse;
    const int d = x.ndims();
    for (std::int64_t e = 0; e < x.nnz(); ++e) {
      const auto idx = x.index(e);
      for (int k = 0; k < d; ++k) coords_out[e * d + k] = idx[static_cast<std::size_t>(k)];
      values_out[e] = x.value(e);
    }
  });
}
int ref_tensor_value_at(void* h, const std::int64_t* idx, double* out) {
  return guard([&] {
    const TensorH* t = static_cast<TensorH*>(h);
    const int d = t->view().shape().ndims();
    *out = t->view().value_at(std::span<const std::int64_t>(idx, static_cast<std::size_t>(d)));
  });
}
double ref_tensor_norm(void* h) { return static_cast<TensorH*>(h)->view().norm(); }

// ---- synthetic problems (synthetic.cpp) ------------------------------------------------
// The generators run on RngStream(seed); *next_draw = the stream's next u64
// afterwards (pins how many draws were consumed).
int ref_gen_gamma(int d, const std::int64_t* dims, std::int64_t r, std::uint64_t seed, void** out,
                  double* truth, std::uint64_t* next_draw) {
  return guard([&] {
    gcp::RngStream rng(seed);
    auto [data, model] = gcp::gen_gamma_problem(make_shape(d, dims), r, rng);
    auto h = std::make_unique<TensorH>();
    h->dense = std::make_unique<gcp::DenseTensor>(std::move(data));
    flatten_model(model, truth);
    *next_draw = rng.next_u64();
    *out = h.release();
  });
}
int ref_gen_binary(int d, const std::int64_t* dims, std::int64_t r, double delta, double p_high,
                   double p_low, std::uint64_t seed, void** out, double* truth,
                   std::uint64_t* next_draw) {
  return guard([&] {
    gcp::RngStream rng(seed);
    gcp::BinaryProblemSpec spec{make_shape(d, dims), r, delta, p_high, p_low};
    auto [data, model] = gcp::gen_binary_problem(spec, rng);
    auto h = std::make_unique<TensorH>();
    h->sparse = std::make_unique<gcp::SparseTensor>(std::move(data));
    flatten_model(model, truth);
    *next_draw = rng.next_u64();
    *out = h.release();
  });
}

// The seeded instances of acceptance.cpp criteria 4 (:166-213) and 10
// (:432-461), built by the reference's own fixtures: the sparse tensor and
// the model (flattened).
int ref_acceptance_instance(int criterion, void** tensor_out, double* model_out) {
  return guard([&] {
    auto h = std::make_unique<TensorH>();
    if (criterion == 4) {
      const gcp::Shape shape({6, 5, 4});
      gcp::RngStream rng(1004);
      const gcp::KruskalModel model = oracles::random_model(shape, 2, rng, 0.1, 1.0);
      h->sparse = std::make_unique<gcp::SparseTensor>(oracles::random_sparse(
          shape, 0.25, [](gcp::RngStream& r) { return 1.0 + r.next_double(); }, rng));
      flatten_model(model, model_out);
    } else if (criterion == 10) {
      const gcp::Shape shape({10, 8, 6});
      gcp::RngStream rng(1010);
      h->sparse = std::make_unique<gcp::SparseTensor>(oracles::random_sparse(
          shape, 0.25, [](gcp::RngStream& r) { return 0.5 + r.next_double(); }, rng));
      const gcp::KruskalModel model = oracles::random_model(shape, 2, rng, 0.1, 1.0);
      flatten_model(model, model_out);
    } else {
      throw std::invalid_argument("ref_acceptance_instance: criterion 4 or 10");
    }
    *tensor_out = h.release();
  });
}

// cosine_similarity_score (scoring.cpp:23-60) of an estimate against a truth.
int ref_similarity(int d, const std::int64_t* dims, std::int64_t r_est, const double* est,
                   std::int64_t r_true, const double* truth, double* out) {
  return guard([&] {
    *out = gcp::cosine_similarity_score(make_model(d, dims, r_est, est),
                                        make_model(d, dims, r_true, truth));
  });
}

// acceptance.cpp:215-250 (criterion 5, variance ordering), restated through
// the public API: the instance, the scaled model it evaluates, and the three
// empirical variances (uniform, stratified, semi-stratified).
int ref_variance_ordering(double* model_out, double* var_out) {
  return guard([&] {
    gcp::BinaryProblemSpec spec;
    spec.shape = gcp::Shape({40, 30, 20});
    spec.rank = 3;
    spec.delta = 0.15;
    spec.p_high = 0.9;
    spec.p_low = 0.0025;
    gcp::RngStream rng(1005);
    const auto [x, truth] = gcp::gen_binary_problem(spec, rng);
    gcp::KruskalModel model = gcp::KruskalModel::random_uniform(spec.shape, 3, rng);
    if (x.norm() > 0.0) model.scale_norm_to(0.5 * x.norm());
    flatten_model(model, model_out);
    const gcp::LossFunction loss = gcp::LossFunction::bernoulli_odds();
    const char* tokens[3] = {"uniform", "stratified", "semi-stratified"};
    for (int i = 0; i < 3; ++i) {
      gcp::RngStream r = rng.split(tokens[i]);
      var_out[i] = gcp::empirical_bias_variance(gcp::SamplerKind::from_token(tokens[i], 90),
                                                gcp::TensorView(x), model, loss, 1000, r)
                       .variance;
    }
  });
}

// ---- tensor files (io.cpp) ------------------------------------------------------------
namespace {
void shape_out(const gcp::Shape& s, int* d, std::int64_t* dims) {
  *d = s.ndims();
  for (int k = 0; k < s.ndims(); ++k) dims[k] = s.dim(k);
}
}  // namespace
int ref_read_tns(const char* path, void** out, int* d, std::int64_t* dims) {
  return guard([&] {
    auto h = std::make_unique<TensorH>();
    h->sparse = std::make_unique<gcp::SparseTensor>(gcp::read_tns(path));
    shape_out(h->sparse->shape(), d, dims);
    *out = h.release();
  });
}
int ref_write_tns(void* h, const char* path) {
  return guard([&] { gcp::write_tns(*static_cast<TensorH*>(h)->sparse, path); });
}
int ref_read_dense(const char* path, void** out, int* d, std::int64_t* dims) {
  return guard([&] {
    auto h = std::make_unique<TensorH>();
    h->dense = std::make_unique<gcp::DenseTensor>(gcp::read_dense(path));
    shape_out(h->dense->shape(), d, dims);
    *out = h.release();
  });
}
int ref_write_dense(void* h, const char* path) {
  return guard([&] { gcp::write_dense(*static_cast<TensorH*>(h)->dense, path); });
}
int ref_write_model(int d, const std::int64_t* dims, std::int64_t r, const double* factors,
                    const char* path) {
  return guard([&] { gcp::write_model(make_model(d, dims, r, factors), path); });
}
int ref_read_model(const char* path, int* d, std::int64_t* dims, std::int64_t* r,
                   double* factors, std::int64_t cap) {
  return guard([&] {
    const gcp::KruskalModel m = gcp::read_model(path);
    *d = m.ndims();
    *r = m.rank();
    std::int64_t n = 0;
    for (int k = 0; k < m.ndims(); ++k) {
      dims[k] = m.shape().dim(k);
      n += dims[k] * m.rank();
    }
    if (n > cap) throw std::length_error("ref_read_model: capacity");
    flatten_model(m, factors);
  });
}
int ref_write_trace(const char* path, std::int64_t n, const std::int64_t* epoch,
                    const double* loss, const double* lr, const double* secs,
                    const int* accepted) {
  return guard([&] {
    gcp::FitTrace t;
    for (std::int64_t i = 0; i < n; ++i)
      t.records.push_back({epoch[i], loss[i], lr[i], secs[i], accepted[i] != 0});
    gcp::write_trace_csv(t, path);
  });
}
int ref_dense_export(void* h, double* out) {
  return guard([&] {
    const auto v = static_cast<TensorH*>(h)->dense->values();
    std::memcpy(out, v.data(), v.size() * sizeof(double));
  });
}

// ---- model evaluation -------------------------------------------------------------
int ref_model_entry(int d, const std::int64_t* dims, std::int64_t r, const double* factors,
                    std::int64_t n, const std::int64_t* idx, double* out) {
  return guard([&] {
    const gcp::KruskalModel model = make_model(d, dims, r, factors);
    for (std::int64_t e = 0; e < n; ++e)
      out[e] = model.entry(std::span<const std::int64_t>(idx + e * d, static_cast<std::size_t>(d)));
  });
}

// ---- samplers driven by a script (samplers.hpp:75-245) --------------------------------
int ref_draw_gradient_samples_scripted(void* tensor, int d, const std::int64_t* dims,
                                       std::int64_t r, const double* factors, int loss_kind,
                                       double delta, int strategy, std::int64_t s,
                                       std::int64_t p, std::int64_t q, double rho,
                                       const std::uint64_t* script, std::int64_t script_len,
                                       std::int64_t cap, std::int64_t* idx_out, double* y_out,
                                       std::int64_t* n_out, std::int64_t* consumed,
                                       std::int64_t* stats /*tested,accepted,rejected*/) {
  return guard([&] {
    const TensorH* t = static_cast<TensorH*>(tensor);
    const gcp::KruskalModel model = make_model(d, dims, r, factors);
    const gcp::LossFunction loss = make_loss(loss_kind, delta);
    ScriptedRng rng{script, script_len, 0};
    gcp::RejectionStats st;
    const gcp::GradientSamples gs = gcp::draw_gradient_samples(
        t->view(), model, loss, make_kind(strategy, s, p, q, rho), rng, &st);
    copy_samples(gs, cap, idx_out, y_out, n_out);
    *consumed = rng.at;
    stats[0] = st.tested;
    stats[1] = st.accepted;
    stats[2] = st.rejected;
  });
}

// Same, with the reference's own RngStream (seeded), for statistical checks and
// the CPU baseline.
int ref_draw_gradient_samples_seeded(void* tensor, int d, const std::int64_t* dims, std::int64_t r,
                                     const double* factors, int loss_kind, double delta,
                                     int strategy, std::int64_t s, std::int64_t p, std::int64_t q,
                                     double rho, std::uint64_t seed, std::int64_t cap,
                                     std::int64_t* idx_out, double* y_out, std::int64_t* n_out) {
  return guard([&] {
    const TensorH* t = static_cast<TensorH*>(tensor);
    const gcp::KruskalModel model = make_model(d, dims, r, factors);
    const gcp::LossFunction loss = make_loss(loss_kind, delta);
    gcp::RngStream rng(seed);
    const gcp::GradientSamples gs = gcp::draw_gradient_samples(
        t->view(), model, loss, make_kind(strategy, s, p, q, rho), rng);
    copy_samples(gs, cap, idx_out, y_out, n_out);
  });
}

// GradientSamples built from builder-supplied (index, x, weight) exactly as the
// uniform sampler body does (samplers.hpp:90-91): y = w * deriv(x, entry(i)).
// subtract_zero=1 mirrors the semi-stratified nonzero term (samplers.hpp:206).
int ref_weighted_derivs(int d, const std::int64_t* dims, std::int64_t r, const double* factors,
                        int loss_kind, double delta, std::int64_t n, const std::int64_t* idx,
                        const double* x, const double* w, int subtract_zero, double* y_out) {
  return guard([&] {
    const gcp::KruskalModel model = make_model(d, dims, r, factors);
    const gcp::LossFunction loss = make_loss(loss_kind, delta);
    for (std::int64_t e = 0; e < n; ++e) {
      const std::span<const std::int64_t> span(idx + e * d, static_cast<std::size_t>(d));
      const double m = model.entry(span);
      y_out[e] = subtract_zero ? w[e] * (loss.deriv(x[e], m) - loss.deriv(0.0, m))
                               : w[e] * loss.deriv(x[e], m);
    }
  });
}

// ---- mttkrp_sampled_all (kernels.cpp:137-168) ---------------------------------------
int ref_mttkrp_sampled_all(int d, const std::int64_t* dims, std::int64_t r, const double* factors,
                           std::int64_t n, const std::int64_t* idx, const double* y, int threads,
                           double* grad_out) {
  return guard([&] {
    const gcp::KruskalModel model = make_model(d, dims, r, factors);
    gcp::GradientSamples gs(model.shape());
    gs.reserve(n);
    for (std::int64_t e = 0; e < n; ++e)
      gs.append(std::span<const std::int64_t>(idx + e * d, static_cast<std::size_t>(d)), y[e]);
    const gcp::GradientSet g = gcp::mttkrp_sampled_all(gs, model, threads);
    flatten_mats(g.modes, grad_out);
  });
}

int ref_gradient_full(void* tensor, int d, const std::int64_t* dims, std::int64_t r,
                      const double* factors, int loss_kind, double delta, double* grad_out) {
  return guard([&] {
    const TensorH* t = static_cast<TensorH*>(tensor);
    const gcp::KruskalModel model = make_model(d, dims, r, factors);
    const gcp::GradientSet g = gcp::gradient_full(t->view(), model, make_loss(loss_kind, delta));
    flatten_mats(g.modes, grad_out);
  });
}

int ref_gradient_poisson_implicit(void* tensor, int d, const std::int64_t* dims, std::int64_t r,
                                  const double* factors, double* grad_out) {
  return guard([&] {
    const TensorH* t = static_cast<TensorH*>(tensor);
    const gcp::KruskalModel model = make_model(d, dims, r, factors);
    const gcp::GradientSet g =
        gcp::gradient_poisson_implicit(*t->sparse, model, gcp::LossFunction::poisson());
    flatten_mats(g.modes, grad_out);
  });
}

// empirical_bias_variance(kind, x, model, loss, trials, RngStream(seed))
// (samplers.cpp:157-168).
int ref_empirical_bias_variance(void* tensor, int d, const std::int64_t* dims, std::int64_t r,
                                const double* factors, int loss_kind, double delta, int strategy,
                                std::int64_t s, std::int64_t p, std::int64_t q, double rho,
                                std::int64_t trials, std::uint64_t seed, double* bias,
                                double* variance) {
  return guard([&] {
    const TensorH* t = static_cast<TensorH*>(tensor);
    const gcp::KruskalModel model = make_model(d, dims, r, factors);
    gcp::RngStream rng(seed);
    const gcp::BiasVariance bv = gcp::empirical_bias_variance(
        make_kind(strategy, s, p, q, rho), t->view(), model, make_loss(loss_kind, delta), trials,
        rng);
    *bias = bv.bias;
    *variance = bv.variance;
  });
}

// ---- adam_step (optimizer.cpp:47-66) -----------------------------------------------
int ref_adam_step(int d, const std::int64_t* dims, std::int64_t r, double* factors, double* first,
                  double* second, std::int64_t* iterations, double learning_rate,
                  const double* grads, double beta1, double beta2, double epsilon, int has_lb,
                  double lb) {
  return guard([&] {
    gcp::KruskalModel model = make_model(d, dims, r, factors);
    gcp::AdamState st = gcp::AdamState::init(model, learning_rate);
    unflatten_mats(st.first_moment, first);
    unflatten_mats(st.second_moment, second);
    st.iterations = *iterations;
    gcp::GradientSet g = gcp::GradientSet::zeros_like(model);
    unflatten_mats(g.modes, grads);
    gcp::FitConfig cfg;
    cfg.beta1 = beta1;
    cfg.beta2 = beta2;
    cfg.epsilon = epsilon;
    if (has_lb) cfg.lower_bound = lb;
    gcp::adam_step(model, st, g, cfg);
    flatten_model(model, factors);
    flatten_mats(st.first_moment, first);
    flatten_mats(st.second_moment, second);
    *iterations = st.iterations;
  });
}

// ---- EstimatorSamples (samplers.hpp:257-351; samplers.cpp:114-124) ------------------------
// Draws the estimator set from a script; exports (idx, x, w) and the estimate.
int ref_estimator_scripted(void* tensor, int kind, std::int64_t count, double rho,
                           const std::uint64_t* script, std::int64_t script_len, int d,
                           const std::int64_t* dims, std::int64_t r, const double* factors,
                           int loss_kind, double delta, std::int64_t cap, std::int64_t* idx_out,
                           double* x_out, double* w_out, std::int64_t* n_out, double* estimate) {
  return guard([&] {
    const TensorH* t = static_cast<TensorH*>(tensor);
    ScriptedRng rng{script, script_len, 0};
    const gcp::EstimatorSamples est = gcp::draw_estimator_samples(
        t->view(), static_cast<gcp::EstimatorSamples::Kind>(kind), count, rng, rho);
    const std::int64_t n = est.size();
    *n_out = n;
    if (n > cap) throw std::length_error("ref_capi: output capacity too small");
    for (std::int64_t e = 0; e < n; ++e) {
      const auto idx = est.index(e);
      for (int k = 0; k < d; ++k) idx_out[e * d + k] = idx[static_cast<std::size_t>(k)];
      x_out[e] = est.data_value(e);
      w_out[e] = est.weight(e);
    }
    const gcp::KruskalModel model = make_model(d, dims, r, factors);
    *estimate = est.estimate(model, make_loss(loss_kind, delta));
  });
}

// Sequential weighted loss sum over builder-supplied (idx, x, w), the body of
// EstimatorSamples::estimate (samplers.cpp:118-123).
int ref_estimate_given(int d, const std::int64_t* dims, std::int64_t r, const double* factors,
                       int loss_kind, double delta, std::int64_t n, const std::int64_t* idx,
                       const double* x, const double* w, double* out) {
  return guard([&] {
    const gcp::KruskalModel model = make_model(d, dims, r, factors);
    const gcp::LossFunction loss = make_loss(loss_kind, delta);
    double sum = 0.0;
    for (std::int64_t e = 0; e < n; ++e) {
      const double m =
          model.entry(std::span<const std::int64_t>(idx + e * d, static_cast<std::size_t>(d)));
      sum += w[e] * loss.value(x[e], m);
    }
    *out = sum;
  });
}

// ---- fit_gcp_adam (optimizer.cpp:68-158), reference trajectory ----------------------------
int ref_fit_gcp_adam(void* tensor, int loss_kind, double delta, std::int64_t rank, int strategy,
                     std::int64_t s, std::int64_t p, std::int64_t q, double rho,
                     double learning_rate, double beta1, double beta2, double epsilon,
                     std::int64_t epoch_iters, std::int64_t max_bad_epochs, double decay,
                     int has_lb, double lb, std::int64_t estimator_samples, int estimator_kind,
                     std::int64_t max_epochs, std::uint64_t seed, int threads,
                     std::int64_t trace_cap, double* trace_out /*rows: epoch,F,lr,sec,acc*/,
                     std::int64_t* n_trace, double* factors_out, double* final_estimate) {
  return guard([&] {
    const TensorH* t = static_cast<TensorH*>(tensor);
    gcp::FitConfig cfg;
    cfg.rank = rank;
    cfg.sampler = make_kind(strategy, s, p, q, rho);
    cfg.learning_rate = learning_rate;
    cfg.beta1 = beta1;
    cfg.beta2 = beta2;
    cfg.epsilon = epsilon;
    cfg.epoch_iters = epoch_iters;
    cfg.max_bad_epochs = max_bad_epochs;
    cfg.decay = decay;
    if (has_lb) cfg.lower_bound = lb;
    cfg.estimator_samples = estimator_samples;
    if (estimator_kind >= 0)
      cfg.estimator_kind = static_cast<gcp::EstimatorSamples::Kind>(estimator_kind);
    cfg.max_epochs = max_epochs;
    cfg.seed = seed;
    cfg.threads = threads;
    const gcp::FitResult res = gcp::fit_gcp_adam(t->view(), make_loss(loss_kind, delta), cfg);
    const auto& recs = res.trace.records;
    *n_trace = static_cast<std::int64_t>(recs.size());
    for (std::size_t i = 0; i < recs.size() && static_cast<std::int64_t>(i) < trace_cap; ++i) {
      trace_out[i * 5 + 0] = static_cast<double>(recs[i].epoch);
      trace_out[i * 5 + 1] = recs[i].loss_estimate;
      trace_out[i * 5 + 2] = recs[i].learning_rate;
      trace_out[i * 5 + 3] = recs[i].seconds;
      trace_out[i * 5 + 4] = recs[i].accepted ? 1.0 : 0.0;
    }
    flatten_model(res.model, factors_out);
    *final_estimate = res.final_loss_estimate;
  });
}

// ---- CPU baseline timings ---------------------------------------------------
// One reference "step" on builder-supplied (index, x, weight): the per-sample
// entry + deriv + weight + append loop (samplers.hpp:87-93), then
// mttkrp_sampled_all(threads) (kernels.cpp:137-168), then adam_step
// (optimizer.cpp:47-66).  The model is updated in place across calls.
struct BenchModel {
  gcp::KruskalModel model;
  gcp::AdamState state;
};
int ref_bench_model_new(int d, const std::int64_t* dims, std::int64_t r, const double* factors,
                        void** out) {
  return guard([&] {
    auto b = std::make_unique<BenchModel>();
    b->model = make_model(d, dims, r, factors);
    b->state = gcp::AdamState::init(b->model, 1e-3);
    *out = b.release();
  });
}
void ref_bench_model_free(void* h) { delete static_cast<BenchModel*>(h); }

// The reference step's tail: mttkrp_sampled_all(threads) and, when do_adam,
// adam_step (times[1], times[2]; times[2] = 0 when skipped).
static void bench_tail(BenchModel& b, const gcp::GradientSamples& gs, int threads,
                       double learning_rate, int has_lb, double lb, int do_adam, double* times) {
  const auto t1 = std::chrono::steady_clock::now();
  const gcp::GradientSet g = gcp::mttkrp_sampled_all(gs, b.model, threads);
  const auto t2 = std::chrono::steady_clock::now();
  times[1] = secs(t1, t2);
  times[2] = 0.0;
  if (!do_adam) return;
  gcp::FitConfig cfg;
  if (has_lb) cfg.lower_bound = lb;
  b.state.learning_rate = learning_rate;
  gcp::adam_step(b.model, b.state, g, cfg);
  times[2] = secs(t2, std::chrono::steady_clock::now());
}

// Semi-stratified step on builder-supplied draws (C5, whose COO the reference
// cannot hold): the loop body of sample_semi_stratified (samplers.hpp:199-216)
// on p pre-drawn nonzero picks (index, value) and q pre-drawn unrestricted
// indices (x = 0: the COO lookup of value_at is excluded), then the tail.
int ref_bench_step_semi_given(void* bm, int loss_kind, double delta, std::int64_t p,
                              const std::int64_t* idx_p, const double* x_p, std::int64_t q,
                              const std::int64_t* idx_q, std::int64_t eta, double total,
                              int threads, double learning_rate, int has_lb, double lb,
                              int do_adam, double* times /*3*/) {
  return guard([&] {
    BenchModel& b = *static_cast<BenchModel*>(bm);
    const gcp::LossFunction loss = make_loss(loss_kind, delta);
    const int d = b.model.ndims();
    const auto t0 = std::chrono::steady_clock::now();
    gcp::GradientSamples gs(b.model.shape());
    gs.reserve(p + q);
    const double eta_over_p = p > 0 ? static_cast<double>(eta) / static_cast<double>(p) : 0.0;
    for (std::int64_t t = 0; t < p; ++t) {
      const std::span<const std::int64_t> span(idx_p + t * d, static_cast<std::size_t>(d));
      const double m = b.model.entry(span);
      gs.append(span, eta_over_p * (loss.deriv(x_p[t], m) - loss.deriv(0.0, m)));
    }
    const double weight = total / static_cast<double>(q > 0 ? q : 1);
    for (std::int64_t t = 0; t < q; ++t) {
      const std::span<const std::int64_t> span(idx_q + t * d, static_cast<std::size_t>(d));
      const double m = b.model.entry(span);
      gs.append(span, weight * loss.deriv(0.0, m));
    }
    times[0] = secs(t0, std::chrono::steady_clock::now());
    bench_tail(b, gs, threads, learning_rate, has_lb, lb, do_adam, times);
  });
}

int ref_bench_step_given(void* bm, int loss_kind, double delta, std::int64_t n,
                         const std::int64_t* idx, const double* x, double weight, int threads,
                         double learning_rate, int has_lb, double lb, int do_adam,
                         double* times /*3*/) {
  return guard([&] {
    BenchModel& b = *static_cast<BenchModel*>(bm);
    const gcp::LossFunction loss = make_loss(loss_kind, delta);
    const int d = b.model.ndims();
    const auto t0 = std::chrono::steady_clock::now();
    gcp::GradientSamples gs(b.model.shape());
    gs.reserve(n);
    for (std::int64_t e = 0; e < n; ++e) {
      const std::span<const std::int64_t> span(idx + e * d, static_cast<std::size_t>(d));
      const double m = b.model.entry(span);
      gs.append(span, weight * loss.deriv(x[e], m));
    }
    times[0] = secs(t0, std::chrono::steady_clock::now());
    bench_tail(b, gs, threads, learning_rate, has_lb, lb, do_adam, times);
  });
}

// One reference step with its own sampler + RngStream (C1, C3, C4 per BASELINE.md §2).
int ref_bench_step_sampler(void* bm, void* tensor, int loss_kind, double delta, int strategy,
                           std::int64_t s, std::int64_t p, std::int64_t q, double rho,
                           std::uint64_t seed, int threads, double learning_rate, int has_lb,
                           double lb, int do_adam, double* times /*3*/, std::int64_t* n_samples) {
  return guard([&] {
    BenchModel& b = *static_cast<BenchModel*>(bm);
    const TensorH* t = static_cast<TensorH*>(tensor);
    const gcp::LossFunction loss = make_loss(loss_kind, delta);
    gcp::RngStream rng(seed);
    const auto t0 = std::chrono::steady_clock::now();
    const gcp::GradientSamples gs = gcp::draw_gradient_samples(
        t->view(), b.model, loss, make_kind(strategy, s, p, q, rho), rng);
    times[0] = secs(t0, std::chrono::steady_clock::now());
    bench_tail(b, gs, threads, learning_rate, has_lb, lb, do_adam, times);
    *n_samples = gs.size();
  });
}

}  // extern "C"
