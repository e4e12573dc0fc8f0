// ref_binding_check.cpp -- TEST INFRASTRUCTURE.  Compiles the reference-side
// binding (integration/gcp_b200.hpp) against the reference's own headers and
// objects (oracle/_ref, built from /root/reference by oracle/Makefile) and
// checks, for all six losses on the reference's own containers,
//   gcp::b200::fit_gcp_adam(x, loss, cfg)   (epoch loop on the B200)
// against
//   gcp::fit_gcp_adam(x, loss, cfg)         (src/optimizer.cpp:68-158)
// epoch by epoch: same accept/rollback decisions, loss estimates within 1e-9
// relative, final model within 1e-8 (tests/oracles.hpp:174-182 rel_error).
// Also checks the Huber half-width crossing the boundary (to_c) and the
// exception mapping.  Prints "ok" and exits 0 on success.
//   ref_binding_check            all checks (needs a GPU)
//   ref_binding_check --no-gpu   host-side checks only
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "gcp_b200.hpp"

using namespace gcp;

namespace {

int failures = 0;
void expect(bool ok, const std::string& what) {
  if (!ok) {
    std::fprintf(stderr, "FAIL: %s\n", what.c_str());
    ++failures;
  }
}

double rel_error(const KruskalModel& a, const KruskalModel& b) {
  double num = 0.0, den = 0.0;
  for (int k = 0; k < a.ndims(); ++k)
    for (Eigen::Index i = 0; i < a.factor(k).rows(); ++i)
      for (Eigen::Index j = 0; j < a.factor(k).cols(); ++j) {
        const double d = a.factor(k)(i, j) - b.factor(k)(i, j);
        num += d * d;
        den += b.factor(k)(i, j) * b.factor(k)(i, j);
      }
  return den > 0.0 ? std::sqrt(num / den) : std::sqrt(num);
}

DenseTensor dense_problem(const Shape& s, std::uint64_t seed, int kind) {
  RngStream rng(seed);
  DenseTensor x(s);
  for (double& v : x.values()) {
    const double u = rng.next_double();
    v = kind == 0 ? 2.0 * u - 1.0 : 0.05 + u;  // real (gaussian, huber) / positive
  }
  return x;
}

SparseTensor sparse_problem(const Shape& s, std::uint64_t seed, bool binary) {
  RngStream rng(seed);
  std::vector<MultiIndex> idx;
  std::vector<double> vals;
  std::vector<std::int64_t> c(static_cast<std::size_t>(s.ndims()));
  for (int t = 0; t < 400; ++t) {
    for (int k = 0; k < s.ndims(); ++k)
      c[static_cast<std::size_t>(k)] = static_cast<std::int64_t>(
          rng.next_below(static_cast<std::uint64_t>(s.dim(k))));
    idx.emplace_back(std::span<const std::int64_t>(c));
    vals.push_back(binary ? 1.0 : 1.0 + static_cast<double>(rng.next_below(4)));
  }
  if (binary)  // duplicates sum: keep binary data binary
    for (double& v : vals) v = 1.0;
  SparseTensor x(s, idx, vals);
  if (!binary) return x;
  std::vector<MultiIndex> idx2;
  std::vector<double> v2;
  for (std::int64_t e = 0; e < x.nnz(); ++e) {
    idx2.push_back(x.multi_index_at(e));
    v2.push_back(1.0);
  }
  return SparseTensor(s, idx2, v2);
}

void compare_fit(const char* name, const TensorView& x, const LossFunction& loss,
                 const FitConfig& cfg) {
  const FitResult want = gcp::fit_gcp_adam(x, loss, cfg);
  const FitResult got = gcp::b200::fit_gcp_adam(x, loss, cfg);
  const std::string n = name;
  expect(got.trace.records.size() == want.trace.records.size(), n + ": trace length");
  const std::size_t m = std::min(got.trace.records.size(), want.trace.records.size());
  for (std::size_t i = 0; i < m; ++i) {
    const auto& g = got.trace.records[i];
    const auto& w = want.trace.records[i];
    expect(g.epoch == w.epoch && g.accepted == w.accepted, n + ": epoch decision " +
                                                               std::to_string(i));
    expect(std::fabs(g.loss_estimate - w.loss_estimate) <= 1e-9 * std::fabs(w.loss_estimate),
           n + ": loss estimate at epoch " + std::to_string(i));
    expect(g.learning_rate == w.learning_rate, n + ": learning rate " + std::to_string(i));
  }
  expect(std::fabs(got.final_loss_estimate - want.final_loss_estimate) <=
             1e-9 * std::fabs(want.final_loss_estimate),
         n + ": final estimate");
  expect(rel_error(got.model, want.model) <= 1e-8, n + ": final model");
  expect(got.final_state.iterations == want.final_state.iterations, n + ": iterations");
}

}  // namespace

int main(int argc, char** argv) {
  const bool gpu = !(argc > 1 && std::strcmp(argv[1], "--no-gpu") == 0);
  // host side: the Huber half-width survives the boundary exactly
  for (double delta : {0.25, 0.5, 1.0 / 3.0, 7.0, 1e-3}) {
    const gcpb_loss l = b200::to_c(LossFunction::huber(delta));
    expect(l.kind == GCPB_LOSS_HUBER && l.delta == delta, "huber delta " + std::to_string(delta));
  }
  expect(b200::to_c(LossFunction::parse("huber:0.75")).delta == 0.75, "parsed huber delta");
  expect(b200::to_c(LossFunction::gamma()).kind == GCPB_LOSS_GAMMA, "loss kind order");
  const gcpb_sampler sk = b200::to_c(SamplerKind::stratified(7, 9, 1.5));
  expect(sk.strategy == GCPB_STRATIFIED && sk.nonzero_samples == 7 && sk.zero_samples == 9 &&
             sk.oversample == 1.5,
         "sampler fields");
  // the stream base recovered from a copy equals the device RefStream key
  {
    RngStream r(1234);
    RngStream g = r.split("gradients");
    gcpb_rng seeded, split;
    gcpb_rng_seed(1234, &seeded);
    std::uint64_t h = 0xcbf29ce484222325ull;  // FNV-1a of the label (rng.cpp:22-29)
    for (char ch : std::string("gradients")) {
      h ^= static_cast<unsigned char>(ch);
      h *= 0x100000001b3ull;
    }
    gcpb_rng_split(&seeded, h, &split);
    expect(b200::stream_base(g) == split.key, "stream base of a fresh split");
    const std::uint64_t base0 = b200::stream_base(g);
    g.next_u64();
    expect(b200::stream_base(g) == base0 + 0x9e3779b97f4a7c15ull, "stream base after one draw");
  }
  if (gpu) {
    // exception mapping across the boundary
    try {
      b200::Engine bad(Shape{3, 4}, 0);
      expect(false, "rank 0 must throw");
    } catch (const std::invalid_argument&) {
    }
    const Shape sd{12, 10, 8}, ss{14, 12, 10, 8};
    FitConfig cfg;
    cfg.rank = 3;
    cfg.epoch_iters = 60;
    cfg.estimator_samples = 500;
    cfg.max_epochs = 5;
    cfg.learning_rate = 2e-2;
    cfg.seed = 11;
    cfg.sampler = SamplerKind::uniform(40);
    compare_fit("gaussian/dense/uniform", dense_problem(sd, 1, 0), LossFunction::gaussian(), cfg);
    compare_fit("huber/dense/uniform", dense_problem(sd, 2, 0), LossFunction::huber(0.3), cfg);
    compare_fit("gamma/dense/uniform", dense_problem(sd, 3, 1), LossFunction::gamma(), cfg);
    compare_fit("beta-half/dense/uniform", dense_problem(sd, 4, 1), LossFunction::beta_half(),
                cfg);
    cfg.sampler = SamplerKind::semi_stratified(20, 30);
    compare_fit("poisson/sparse/semi", sparse_problem(ss, 5, false), LossFunction::poisson(), cfg);
    cfg.sampler = SamplerKind::stratified(20, 30);
    compare_fit("bernoulli-odds/sparse/stratified", sparse_problem(ss, 6, true),
                LossFunction::bernoulli_odds(), cfg);
    cfg.sampler = SamplerKind::uniform(50);
    compare_fit("poisson/sparse/uniform", sparse_problem(ss, 7, false), LossFunction::poisson(),
                cfg);
  }
  if (failures) {
    std::fprintf(stderr, "%d failure(s)\n", failures);
    return 1;
  }
  std::printf("ok\n");
  return 0;
}
