/* gcp_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's stochastic-GCP hot path
 * (/root/reference/proj), used by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg as the CHECKER — never by the product path.
 * Every function cites the reference file:line it restates.  It is pinned
 * against the reference itself (oracle/_ref, built from the unmodified
 * sources) and against the golden fixtures under tests/golden/.
 *
 * It also holds the host replica of the product's Philox4x32-10 draw stream
 * (DESIGN.md §3), so sampler indices can be checked bit-exactly.
 */
#ifndef GCP_ORACLE_H
#define GCP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- RngStream restatement (rng.cpp:12-61) ---- */
typedef struct {
  uint64_t key;
  uint64_t counter;
} or_rng;

uint64_t or_mix64(uint64_t z);
void or_rng_init(or_rng* r, uint64_t seed);
void or_rng_split_label(const or_rng* r, const char* label, or_rng* out);
void or_rng_split_u64(const or_rng* r, uint64_t label, or_rng* out);
uint64_t or_rng_next_u64(or_rng* r);
double or_rng_next_double(or_rng* r);
uint64_t or_rng_next_below(or_rng* r, uint64_t n);

/* ---- product Philox stream replica ---- */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* Bounded draw in [0, n) for (seed, tag, iter, t, slot k).  Returns n on
 * attempt exhaustion (never observed). */
uint64_t or_draw_bounded(uint64_t seed, uint32_t tag, uint64_t iter, uint64_t t, int k,
                         uint64_t n);

enum {
  OR_TAG_GRAD_UNIFORM = 1,
  OR_TAG_GRAD_NZ_PICK = 2,
  OR_TAG_GRAD_ZERO_CAND = 3,
  OR_TAG_GRAD_SEMI_Q = 4,
  OR_TAG_EST_UNIFORM = 5,
  OR_TAG_EST_NZ_PICK = 6,
  OR_TAG_EST_ZERO_CAND = 7
};

/* ---- loss (loss.cpp:42-124) ---- */
double or_loss_value(int kind, double delta, double x, double m);
double or_loss_deriv(int kind, double delta, double x, double m);
int or_loss_check_domain(int kind, double x); /* 0 ok, 3 domain error */

/* ---- model (kruskal.cpp:47-58); factors flattened mode-major, row-major ---- */
double or_entry(int d, const int64_t* dims, int64_t r, const double* factors, const int64_t* idx);

/* ---- mttkrp_sampled_all, serial (kernels.cpp:12-57,137-146) ---- */
void or_mttkrp_sampled_all(int d, const int64_t* dims, int64_t r, const double* factors,
                           int64_t n, const int64_t* idx, const double* y, double* grad_out);

/* ---- adam_step (optimizer.cpp:47-66) ---- */
void or_adam_step(int d, const int64_t* dims, int64_t r, double* factors, double* first,
                  double* second, int64_t* iterations, double learning_rate,
                  const double* grads, double beta1, double beta2, double epsilon, int has_lb,
                  double lb);

/* ---- SparseTensor normalisation (tensor.cpp:10-41): returns nnz or -4 on a
 * bad index (out_of_range), -2 on N >= 2^64 (unsupported by u64 keys). ---- */
int64_t or_sparse_normalize(int d, const int64_t* dims, int64_t n, const int64_t* coords_in,
                            const double* values_in, int64_t* coords_out, double* values_out,
                            uint64_t* keys_out);

/* ---- samplers (samplers.hpp:62-245) with a pluggable draw source ---- */
typedef struct {
  int mode; /* 0 = script (ScriptedRng: script[at++] % n), 1 = product Philox, 2 = RngStream */
  const uint64_t* script;
  int64_t len;
  int64_t at;
  uint64_t seed;
  uint64_t iter;
  uint32_t tag_uniform, tag_pick, tag_zero; /* philox tags per phase */
  int strategy;                             /* layout of the sequential consumption */
  int64_t p;                                /* effective nonzero budget (set by the sampler) */
  int d;
  or_rng rng;
  int exhausted;
} or_src;

typedef struct {
  int d;
  const int64_t* dims;
  int is_sparse;
  int64_t nnz;
  const int64_t* coords;  /* normalised (sorted) COO, nnz x d */
  const double* values;
  const uint64_t* keys;   /* strictly increasing linear keys */
  const double* dense;    /* first-mode-fastest, when !is_sparse */
} or_tensor;

typedef struct {
  int strategy; /* 0 uniform, 1 stratified, 2 semi-stratified */
  int64_t s, p, q;
  double rho;
} or_sampler;

/* Returns 0 ok, 2 usage (invalid_argument), 3 domain, 5 script exhausted.
 * Outputs per sample: index (n x d), data value x, weight w, flag (1 for the
 * semi-stratified nonzero term y = w*(g(x,m)-g(0,m))), final value y. */
int or_draw_gradient_samples(const or_tensor* x, int64_t r, const double* factors, int loss_kind,
                             double delta, const or_sampler* kind, or_src* src, int64_t cap,
                             int64_t* idx_out, double* x_out, double* w_out, int* flag_out,
                             double* y_out, int64_t* n_out, int64_t* stats /*3*/);

/* EstimatorSamples::draw_uniform / draw_stratified (samplers.hpp:263-315). */
int or_estimator_draw(const or_tensor* x, int kind, int64_t count, double rho, or_src* src,
                      int64_t cap, int64_t* idx_out, double* x_out, double* w_out,
                      int64_t* n_out);
/* EstimatorSamples::estimate (samplers.cpp:114-124), sequential fp64. */
double or_estimate(int d, const int64_t* dims, int64_t r, const double* factors, int loss_kind,
                   double delta, int64_t n, const int64_t* idx, const double* x,
                   const double* w);

/* Batch size of one zero-rejection round (samplers.hpp:118-122). */
int64_t or_zero_batch_size(double total, double zeta, double rho, int64_t shortfall);

#ifdef __cplusplus
}
#endif
#endif
