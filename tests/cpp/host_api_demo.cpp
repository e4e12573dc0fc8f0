// C++ host API check (include/gcpb.hpp): the reference-named wrappers drive
// the device engine and rethrow the reference's exception classes.  Built by
// tests/test_cpp_api.py; run on the GPU box.  Prints "ok" on success.
#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>

#include "gcpb.hpp"

#define EXPECT(c)                                                  \
  do {                                                             \
    if (!(c)) {                                                    \
      std::fprintf(stderr, "FAILED %s (line %d)\n", #c, __LINE__); \
      return 1;                                                    \
    }                                                              \
  } while (0)

int main() {
  std::mt19937_64 gen(7);
  std::uniform_real_distribution<double> u(0.1, 1.0);
  const std::vector<int64_t> dims{20, 15, 10};
  const int64_t r = 4;
  gcpb::Engine e(dims, r, GCPB_F64);
  std::vector<int64_t> coords;
  std::vector<double> vals;
  for (int64_t i = 0; i < 20; ++i)
    for (int64_t j = 0; j < 15; ++j)
      for (int64_t k = 0; k < 10; ++k)
        if (u(gen) < 0.15) {
          coords.insert(coords.end(), {i, j, k});
          vals.push_back(1.0);
        }
  e.set_sparse(coords, vals);
  std::vector<std::vector<double>> F(3);
  for (int k = 0; k < 3; ++k) {
    F[k].resize(dims[k] * r);
    for (auto& v : F[k]) v = u(gen);
  }
  e.set_factors(F);
  const auto st = e.stoch_grad(gcpb::SamplerKind::stratified(100, 200), gcpb::LossFunction::bernoulli_odds(), 3, 0);
  EXPECT(st.tested >= 200 && st.accepted + st.rejected == st.tested);
  double gn = 0.0;
  for (const auto& g : e.gradient())
    for (double v : g) gn += v * v;
  EXPECT(std::isfinite(gn) && gn > 0.0);
  // reference exception classes
  bool range = false, usage = false, domain = false;
  try {
    e.set_sparse({0, 0, 10}, {1.0});
  } catch (const std::out_of_range&) {
    range = true;
  }
  try {
    gcpb::SamplerKind::stratified(1, 1, 1.0);
  } catch (const std::invalid_argument&) {
    usage = true;
  }
  e.set_sparse({0, 0, 0}, {3.0});
  try {
    e.stoch_grad(gcpb::SamplerKind::semi_stratified(1, 1), gcpb::LossFunction::bernoulli_odds(), 1, 0);
  } catch (const std::domain_error&) {
    domain = true;
  }
  EXPECT(range && usage && domain);
  // device fit
  e.set_sparse(coords, vals);
  gcpb::FitConfig cfg;
  cfg.rank = r;
  cfg.sampler = gcpb::SamplerKind::stratified(150, 150);
  cfg.epoch_iters = 50;
  cfg.max_epochs = 4;
  cfg.estimator_samples = 2000;
  cfg.seed = 11;
  const auto res = gcpb::fit_gcp_adam(e, gcpb::LossFunction::bernoulli_odds(), cfg);
  EXPECT(!res.trace.empty() && res.trace.front().epoch == 0);
  EXPECT(res.final_loss_estimate <= res.trace.front().loss_estimate);
  gcpb::write_trace_csv(res.trace, "/tmp/gcpb_demo_trace.csv");
  gcpb::write_model(res.model, dims, r, "/tmp/gcpb_demo.model");
  std::vector<int64_t> mdims;
  EXPECT(gcpb::read_model("/tmp/gcpb_demo.model", &mdims) == res.model && mdims == dims);
  // .tns round trip through the native reader/writer
  gcpb::CooTensor t{dims, coords, vals};
  gcpb::write_tns(t, "/tmp/gcpb_demo.tns");
  const gcpb::CooTensor back = gcpb::read_tns("/tmp/gcpb_demo.tns");
  EXPECT(back.dims == dims && back.coords == coords && back.values == vals);
  bool io_err = false;
  try {
    gcpb::read_tns("/tmp/gcpb_demo_missing.tns");
  } catch (const std::runtime_error&) {
    io_err = true;
  }
  EXPECT(io_err);
  // exact gradients: the implicit Poisson form equals the full walk
  e.set_sparse(back);
  e.set_factors(F);
  e.gradient_full(gcpb::LossFunction::poisson());
  const auto gf = e.gradient();
  e.gradient_poisson_implicit(gcpb::LossFunction::poisson());
  const auto gi = e.gradient();
  double num = 0.0, den = 0.0;
  for (int k = 0; k < 3; ++k)
    for (size_t i = 0; i < gf[k].size(); ++i) {
      num += (gf[k][i] - gi[k][i]) * (gf[k][i] - gi[k][i]);
      den += gf[k][i] * gf[k][i];
    }
  EXPECT(std::sqrt(num / den) < 1e-12);
  const auto bv = e.bias_variance(gcpb::SamplerKind::stratified(200, 200),
                                  gcpb::LossFunction::bernoulli_odds(), 64, 5);
  EXPECT(bv.variance > 0.0 && bv.bias * bv.bias < 4.0 * bv.variance / 64);
  // device generators
  gcpb::RngStream rng(3);
  gcpb::Engine b({30, 20, 10}, 3, GCPB_F32);
  const auto truth = b.gen_binary_problem(gcpb::BinaryProblemSpec{}, rng);
  EXPECT(truth.size() == 60 * 3 && b.nnz() > 0 && rng.counter() > 0);
  std::printf("ok\n");
  return 0;
}
