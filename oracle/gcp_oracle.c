/* gcp_oracle.c — TEST INFRASTRUCTURE ONLY (see gcp_oracle.h).
 *
 * CPU restatement of the reference hot path.  Operation order follows the
 * reference so results agree to the last few ulps (the reference's own pins
 * are 1e-12 relational).  Pinned against oracle/_ref (the unmodified reference
 * compiled here) by tests/test_oracle_pin.py and against tests/golden/.
 */
#include "gcp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------------ */
/* RngStream (rng.cpp:12-61)                                                 */
/* ------------------------------------------------------------------------ */
static const uint64_t kGolden = 0x9e3779b97f4a7c15ull; /* rng.cpp:14 */

uint64_t or_mix64(uint64_t z) { /* rng.cpp:15-19 */
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

static uint64_t fnv1a(const char* s) { /* rng.cpp:22-29 */
  uint64_t h = 0xcbf29ce484222325ull;
  for (; *s; ++s) {
    h ^= (unsigned char)*s;
    h *= 0x100000001b3ull;
  }
  return h;
}

void or_rng_init(or_rng* r, uint64_t seed) { /* rng.cpp:33 */
  r->key = or_mix64(seed + kGolden);
  r->counter = 0;
}

void or_rng_split_u64(const or_rng* r, uint64_t label, or_rng* out) { /* rng.cpp:35-37 */
  out->key = or_mix64(r->key ^ or_mix64(label + kGolden));
  out->counter = 0;
}

void or_rng_split_label(const or_rng* r, const char* label, or_rng* out) { /* rng.cpp:39-41 */
  or_rng_split_u64(r, fnv1a(label), out);
}

uint64_t or_rng_next_u64(or_rng* r) { /* rng.cpp:43-45 */
  return or_mix64(r->key + kGolden * ++r->counter);
}

double or_rng_next_double(or_rng* r) { /* rng.cpp:47-49 */
  return (double)(or_rng_next_u64(r) >> 11) * 0x1.0p-53;
}

uint64_t or_rng_next_below(or_rng* r, uint64_t n) { /* rng.cpp:51-61 */
  const uint64_t threshold = (0 - n) % n;
  for (;;) {
    const uint64_t v = or_rng_next_u64(r);
    if (v >= threshold) return v % n;
  }
}

/* ------------------------------------------------------------------------ */
/* Product Philox4x32-10 stream replica.  Independent code    */
/* from the device implementation in paper_1906_01687_b200/csrc/philox.cuh.  */
/* ------------------------------------------------------------------------ */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ c1 ^ k0;
    const uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

static void philox_block(uint64_t seed, uint32_t tag, uint32_t group, uint32_t attempt,
                         uint64_t iter, uint64_t t, uint32_t out[4]) {
  uint32_t ctr[4], key[2];
  ctr[0] = (uint32_t)t;
  ctr[1] = (uint32_t)((t >> 32) & 0xFFFFu) | (attempt << 16);
  ctr[2] = (uint32_t)iter;
  ctr[3] = (tag << 24) | ((group & 0xFFu) << 16) | (uint32_t)((iter >> 32) & 0xFFFFu);
  key[0] = (uint32_t)seed;
  key[1] = (uint32_t)(seed >> 32);
  or_philox4x32_10(ctr, key, out);
}

uint64_t or_draw_bounded(uint64_t seed, uint32_t tag, uint64_t iter, uint64_t t, int k,
                         uint64_t n) {
  uint32_t b[4];
  if (n <= ((uint64_t)1 << 32)) {
    /* 32-bit Lemire multiply-shift with rejection; four slots share a block. */
    const uint64_t thr = (((uint64_t)1 << 32) - n) % n;
    for (uint32_t a = 0; a < 65536u; ++a) {
      philox_block(seed, tag, (uint32_t)k >> 2, a, iter, t, b);
      const uint64_t prod = (uint64_t)b[k & 3] * n;
      if ((uint32_t)prod >= thr) return prod >> 32;
    }
    return n;
  }
  {
    const uint64_t thr = (0 - n) % n;
    for (uint32_t a = 0; a < 65536u; ++a) {
      philox_block(seed, tag, 0x80u | (uint32_t)k, a, iter, t, b);
      const uint64_t v = (uint64_t)b[0] | ((uint64_t)b[1] << 32);
      const u128 prod = (u128)v * n;
      if ((uint64_t)prod >= thr) return (uint64_t)(prod >> 64);
    }
    return n;
  }
}

/* ------------------------------------------------------------------------ */
/* Loss (loss.cpp:42-124); kEps = 1e-10 (loss.hpp:23)                        */
/* kinds: 0 gaussian 1 poisson 2 bernoulli-odds 3 gamma 4 beta-half 5 huber  */
/* ------------------------------------------------------------------------ */
static const double kEps = 1e-10;

int or_loss_check_domain(int kind, double x) { /* loss.cpp:42-62 */
  switch (kind) {
    case 0:
    case 5:
      return 0;
    case 1:
    case 3:
    case 4:
      return (x >= 0.0) ? 0 : 3;
    case 2:
      return (x != 0.0 && x != 1.0) ? 3 : 0;
  }
  return 2;
}

double or_loss_value(int kind, double delta, double x, double m) { /* loss.cpp:64-86 */
  switch (kind) {
    case 0:
      return (x - m) * (x - m);
    case 1:
      return m - x * log(m + kEps);
    case 2:
      return log(m + 1.0) - x * log(m + kEps);
    case 3:
      return x / (m + kEps) + log(m + kEps);
    case 4: {
      const double s = sqrt(m + kEps);
      return 2.0 * s + 2.0 * x / s;
    }
    case 5: {
      const double r = x - m;
      if (fabs(r) <= delta) return r * r;
      return 2.0 * delta * fabs(r) - delta * delta;
    }
  }
  return 0.0;
}

double or_loss_deriv(int kind, double delta, double x, double m) { /* loss.cpp:88-110 */
  switch (kind) {
    case 0:
      return 2.0 * (m - x);
    case 1:
      return 1.0 - x / (m + kEps);
    case 2:
      return 1.0 / (m + 1.0) - x / (m + kEps);
    case 3:
      return 1.0 / (m + kEps) - x / ((m + kEps) * (m + kEps));
    case 4: {
      const double s = sqrt(m + kEps);
      return 1.0 / s - x / (s * s * s);
    }
    case 5: {
      const double r = x - m;
      if (fabs(r) <= delta) return -2.0 * r;
      return r > 0.0 ? -2.0 * delta : 2.0 * delta;
    }
  }
  return 0.0;
}

/* ------------------------------------------------------------------------ */
/* Model and kernels                                                         */
/* ------------------------------------------------------------------------ */
static int64_t mode_offset(int d, const int64_t* dims, int64_t r, int k) {
  int64_t off = 0;
  for (int q = 0; q < k && q < d; ++q) off += dims[q] * r;
  return off;
}

double or_entry(int d, const int64_t* dims, int64_t r, const double* factors,
                const int64_t* idx) { /* kruskal.cpp:47-58 */
  double sum = 0.0;
  for (int64_t j = 0; j < r; ++j) {
    double prod = 1.0;
    int64_t off = 0;
    for (int k = 0; k < d; ++k) {
      prod *= factors[off + idx[k] * r + j];
      off += dims[k] * r;
    }
    sum += prod;
  }
  return sum;
}

void or_mttkrp_sampled_all(int d, const int64_t* dims, int64_t r, const double* factors,
                           int64_t n, const int64_t* idx, const double* y,
                           double* grad_out) { /* kernels.cpp:12-57,137-146 (serial path) */
  int64_t total = 0;
  for (int k = 0; k < d; ++k) total += dims[k] * r;
  memset(grad_out, 0, (size_t)total * sizeof(double));
  double* prefix = (double*)malloc(sizeof(double) * (size_t)(d * r));
  double* suffix = (double*)malloc(sizeof(double) * (size_t)(d * r));
  int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)d);
  for (int k = 0; k < d; ++k) off[k] = mode_offset(d, dims, r, k);
  for (int64_t e = 0; e < n; ++e) {
    const int64_t* ix = idx + e * d;
    const double ye = y[e];
    /* LeaveOneOut::compute (kernels.cpp:21-32) */
    for (int64_t j = 0; j < r; ++j) prefix[j] = 1.0;
    for (int k = 1; k < d; ++k)
      for (int64_t j = 0; j < r; ++j)
        prefix[k * r + j] = prefix[(k - 1) * r + j] * factors[off[k - 1] + ix[k - 1] * r + j];
    for (int64_t j = 0; j < r; ++j) suffix[(d - 1) * r + j] = 1.0;
    for (int k = d - 2; k >= 0; --k)
      for (int64_t j = 0; j < r; ++j)
        suffix[k * r + j] = suffix[(k + 1) * r + j] * factors[off[k + 1] + ix[k + 1] * r + j];
    /* out.row(i_k) += y * (prefix .* suffix)   (kernels.cpp:52-55) */
    for (int k = 0; k < d; ++k) {
      double* row = grad_out + off[k] + ix[k] * r;
      for (int64_t j = 0; j < r; ++j) row[j] += ye * (prefix[k * r + j] * suffix[k * r + j]);
    }
  }
  free(prefix);
  free(suffix);
  free(off);
}

void or_adam_step(int d, const int64_t* dims, int64_t r, double* factors, double* first,
                  double* second, int64_t* iterations, double learning_rate,
                  const double* grads, double beta1, double beta2, double epsilon, int has_lb,
                  double lb) { /* optimizer.cpp:47-66 */
  const int64_t t_eff = *iterations + 1;
  const double corr1 = 1.0 - pow(beta1, (double)t_eff);
  const double corr2 = 1.0 - pow(beta2, (double)t_eff);
  int64_t total = 0;
  for (int k = 0; k < d; ++k) total += dims[k] * r;
  for (int64_t i = 0; i < total; ++i) {
    const double g = grads[i];
    first[i] = beta1 * first[i] + (1.0 - beta1) * g;
    second[i] = beta2 * second[i] + (1.0 - beta2) * (g * g);
    factors[i] -= learning_rate * (first[i] / corr1) / sqrt((second[i] / corr2) + epsilon);
    if (has_lb) factors[i] = factors[i] > lb ? factors[i] : lb; /* cwiseMax */
  }
  ++*iterations;
}

/* ------------------------------------------------------------------------ */
/* Tensors                                                                   */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint64_t key;
  double value;
  int64_t order;
} or_entry_rec;

static int cmp_entry(const void* a, const void* b) {
  const or_entry_rec* x = (const or_entry_rec*)a;
  const or_entry_rec* y = (const or_entry_rec*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->order < y->order ? -1 : (x->order > y->order);
}

static int total_u64(int d, const int64_t* dims, uint64_t* total) {
  u128 t = 1;
  for (int k = 0; k < d; ++k) {
    t *= (u128)dims[k];
    if (t > (u128)UINT64_MAX) return -1;
  }
  *total = (uint64_t)t;
  return 0;
}

static uint64_t linear_key(int d, const int64_t* dims, const int64_t* idx) { /* shape.cpp:87-96 */
  uint64_t lin = 0, stride = 1;
  for (int k = 0; k < d; ++k) {
    lin += (uint64_t)idx[k] * stride;
    stride *= (uint64_t)dims[k];
  }
  return lin;
}

int64_t or_sparse_normalize(int d, const int64_t* dims, int64_t n, const int64_t* coords_in,
                            const double* values_in, int64_t* coords_out, double* values_out,
                            uint64_t* keys_out) { /* tensor.cpp:10-41 */
  uint64_t total;
  if (total_u64(d, dims, &total) != 0) return -2;
  or_entry_rec* recs = (or_entry_rec*)malloc(sizeof(or_entry_rec) * (size_t)(n > 0 ? n : 1));
  for (int64_t e = 0; e < n; ++e) {
    for (int k = 0; k < d; ++k) {
      const int64_t c = coords_in[e * d + k];
      if (c < 0 || c >= dims[k]) {
        free(recs);
        return -4;
      }
    }
    recs[e].key = linear_key(d, dims, coords_in + e * d);
    recs[e].value = values_in[e];
    recs[e].order = e;
  }
  qsort(recs, (size_t)n, sizeof(or_entry_rec), cmp_entry);
  int64_t out = 0, e = 0;
  while (e < n) {
    const uint64_t key = recs[e].key;
    double sum = 0.0;
    while (e < n && recs[e].key == key) sum += recs[e++].value;
    if (sum == 0.0) continue;
    uint64_t rem = key;
    for (int k = 0; k < d; ++k) { /* multi_index (shape.cpp:98-109) */
      coords_out[out * d + k] = (int64_t)(rem % (uint64_t)dims[k]);
      rem /= (uint64_t)dims[k];
    }
    values_out[out] = sum;
    keys_out[out] = key;
    ++out;
  }
  free(recs);
  return out;
}

static int64_t find_key(const or_tensor* x, uint64_t key) { /* tensor.cpp:43-53 */
  int64_t lo = 0, hi = x->nnz;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (x->keys[mid] < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  return (lo < x->nnz && x->keys[lo] == key) ? lo : -1;
}

static double value_at(const or_tensor* x, const int64_t* idx) { /* tensor.hpp:95-97 */
  const uint64_t key = linear_key(x->d, x->dims, idx);
  if (x->is_sparse) {
    const int64_t e = find_key(x, key);
    return e < 0 ? 0.0 : x->values[e];
  }
  return x->dense[key];
}

static double total_double(const or_tensor* x) {
  u128 t = 1;
  for (int k = 0; k < x->d; ++k) t *= (u128)x->dims[k];
  return (double)t;
}

static double zeta_double(const or_tensor* x) {
  u128 t = 1;
  for (int k = 0; k < x->d; ++k) t *= (u128)x->dims[k];
  return (double)(t - (u128)x->nnz);
}

/* ------------------------------------------------------------------------ */
/* Draw sources                                                              */
/* ------------------------------------------------------------------------ */
static uint64_t src_next_below(or_src* s, uint64_t n) {
  if (s->mode == 0) { /* ScriptedRng (tests/oracles.hpp:23-31) */
    if (s->at >= s->len) {
      s->exhausted = 1;
      return 0;
    }
    return s->script[s->at++] % n;
  }
  if (s->mode == 2) return or_rng_next_below(&s->rng, n);
  /* product Philox stream: sequential position -> (tag, t, slot) */
  const int64_t pos = s->at++;
  if (s->strategy == 0) {
    return or_draw_bounded(s->seed, s->tag_uniform, s->iter, (uint64_t)(pos / s->d),
                           (int)(pos % s->d), n);
  }
  if (pos < s->p) return or_draw_bounded(s->seed, s->tag_pick, s->iter, (uint64_t)pos, 0, n);
  const int64_t rel = pos - s->p;
  return or_draw_bounded(s->seed, s->tag_zero, s->iter, (uint64_t)(rel / s->d),
                         (int)(rel % s->d), n);
}

static void draw_index(const or_tensor* x, or_src* s, int64_t* out) { /* samplers.hpp:62-68 */
  for (int k = 0; k < x->d; ++k) out[k] = (int64_t)src_next_below(s, (uint64_t)x->dims[k]);
}

int64_t or_zero_batch_size(double total, double zeta, double rho,
                           int64_t shortfall) { /* samplers.hpp:118-122 */
  double batch_d = ceil(rho * (total / zeta) * (double)shortfall);
  if (!(batch_d >= 1.0)) batch_d = 1.0;
  if (batch_d > 9e15) batch_d = 9e15;
  return (int64_t)batch_d;
}

/* sample_zeros_rejection (samplers.hpp:100-135); writes accepted indices. */
static int zeros_rejection(const or_tensor* x, int64_t q, double rho, or_src* s, int64_t* zeros,
                           int64_t* stats) {
  if (q < 0) return 2;
  if (!(rho > 1.0)) return 2;
  const double zeta = zeta_double(x);
  {
    u128 t = 1;
    for (int k = 0; k < x->d; ++k) t *= (u128)x->dims[k];
    if (t - (u128)x->nnz < (u128)q) return 2;
  }
  const double total = total_double(x);
  int64_t got = 0;
  int64_t idx[16];
  while (got < q) {
    const int64_t batch = or_zero_batch_size(total, zeta, rho, q - got);
    for (int64_t t = 0; t < batch; ++t) {
      draw_index(x, s, idx);
      if (s->exhausted) return 5;
      const int hit = find_key(x, linear_key(x->d, x->dims, idx)) >= 0;
      if (stats) {
        ++stats[0];
        if (hit)
          ++stats[2];
        else
          ++stats[1];
      }
      if (!hit && got < q) {
        memcpy(zeros + got * x->d, idx, sizeof(int64_t) * (size_t)x->d);
        ++got;
      }
    }
  }
  return 0;
}

#define PUSH(IDX, XV, W, FLAG, Y)                                   \
  do {                                                              \
    if (n >= cap) return 6;                                         \
    memcpy(idx_out + n * d, (IDX), sizeof(int64_t) * (size_t)d);    \
    x_out[n] = (XV);                                                \
    w_out[n] = (W);                                                 \
    flag_out[n] = (FLAG);                                           \
    y_out[n] = (Y);                                                 \
    ++n;                                                            \
  } while (0)

int or_draw_gradient_samples(const or_tensor* x, int64_t r, const double* factors, int loss_kind,
                             double delta, const or_sampler* kind, or_src* src, int64_t cap,
                             int64_t* idx_out, double* x_out, double* w_out, int* flag_out,
                             double* y_out, int64_t* n_out, int64_t* stats) {
  const int d = x->d;
  int64_t n = 0;
  int64_t idx[16];
  *n_out = 0;
  if (stats) stats[0] = stats[1] = stats[2] = 0;
  src->d = d;
  src->strategy = kind->strategy;
  /* SamplerKind::validate (samplers.cpp:56-67) */
  if (kind->strategy == 0) {
    if (kind->s < 1) return 2;
  } else {
    if (kind->p < 0 || kind->q < 0 || kind->p + kind->q < 1) return 2;
    if (kind->strategy == 1 && !(kind->rho > 1.0)) return 2;
    if (!x->is_sparse) return 2; /* samplers.hpp:232-240 */
  }
  if (kind->strategy == 0) { /* sample_uniform (samplers.hpp:75-94) */
    const double weight = total_double(x) / (double)kind->s;
    for (int64_t t = 0; t < kind->s; ++t) {
      draw_index(x, src, idx);
      if (src->exhausted) return 5;
      const double m = or_entry(d, x->dims, r, factors, idx);
      const double xv = value_at(x, idx);
      if (or_loss_check_domain(loss_kind, xv)) return 3;
      PUSH(idx, xv, weight, 0, weight * or_loss_deriv(loss_kind, delta, xv, m));
    }
    *n_out = n;
    return 0;
  }
  int64_t p = kind->p, q = kind->q;
  const int64_t eta = x->nnz;
  if (eta == 0 && p > 0) { /* samplers.hpp:152-155 / 194-197 */
    q += p;
    p = 0;
  }
  src->p = p;
  const double eta_over_p = p > 0 ? (double)eta / (double)p : 0.0;
  for (int64_t t = 0; t < p; ++t) {
    const int64_t e = (int64_t)src_next_below(src, (uint64_t)eta);
    if (src->exhausted) return 5;
    const int64_t* ie = x->coords + e * d;
    const double m = or_entry(d, x->dims, r, factors, ie);
    const double xv = x->values[e];
    if (or_loss_check_domain(loss_kind, xv)) return 3;
    if (kind->strategy == 1) { /* samplers.hpp:159-165 */
      PUSH(ie, xv, eta_over_p, 0, eta_over_p * or_loss_deriv(loss_kind, delta, xv, m));
    } else { /* samplers.hpp:201-207 */
      PUSH(ie, xv, eta_over_p, 1,
           eta_over_p * (or_loss_deriv(loss_kind, delta, xv, m) -
                         or_loss_deriv(loss_kind, delta, 0.0, m)));
    }
  }
  if (q > 0) {
    if (kind->strategy == 1) { /* samplers.hpp:166-173 */
      const double zeta_over_q = zeta_double(x) / (double)q;
      int64_t* zeros = (int64_t*)malloc(sizeof(int64_t) * (size_t)(q * d));
      const int rc = zeros_rejection(x, q, kind->rho, src, zeros, stats);
      if (rc) {
        free(zeros);
        return rc;
      }
      for (int64_t t = 0; t < q; ++t) {
        const double m = or_entry(d, x->dims, r, factors, zeros + t * d);
        if (n >= cap) {
          free(zeros);
          return 6;
        }
        memcpy(idx_out + n * d, zeros + t * d, sizeof(int64_t) * (size_t)d);
        x_out[n] = 0.0;
        w_out[n] = zeta_over_q;
        flag_out[n] = 0;
        y_out[n] = zeta_over_q * or_loss_deriv(loss_kind, delta, 0.0, m);
        ++n;
      }
      free(zeros);
    } else { /* samplers.hpp:208-217 */
      const double weight = total_double(x) / (double)q;
      for (int64_t t = 0; t < q; ++t) {
        draw_index(x, src, idx);
        if (src->exhausted) return 5;
        const double m = or_entry(d, x->dims, r, factors, idx);
        PUSH(idx, 0.0, weight, 0, weight * or_loss_deriv(loss_kind, delta, 0.0, m));
      }
    }
  }
  *n_out = n;
  return 0;
}

int or_estimator_draw(const or_tensor* x, int kind, int64_t count, double rho, or_src* src,
                      int64_t cap, int64_t* idx_out, double* x_out, double* w_out,
                      int64_t* n_out) { /* samplers.hpp:263-315,353-363 */
  const int d = x->d;
  int64_t n = 0;
  int64_t idx[16];
  *n_out = 0;
  src->d = d;
  src->strategy = kind;
  if (count < 0) return 2;
  if (kind == 0) {
    const double weight = total_double(x) / (double)count;
    for (int64_t t = 0; t < count; ++t) {
      draw_index(x, src, idx);
      if (src->exhausted) return 5;
      if (n >= cap) return 6;
      memcpy(idx_out + n * d, idx, sizeof(int64_t) * (size_t)d);
      x_out[n] = value_at(x, idx);
      w_out[n] = weight;
      ++n;
    }
    *n_out = n;
    return 0;
  }
  if (!x->is_sparse) return 2;
  int64_t p = count / 2, q = count - p;
  const int64_t eta = x->nnz;
  u128 tot = 1;
  for (int k = 0; k < d; ++k) tot *= (u128)x->dims[k];
  const u128 zeta = tot - (u128)eta;
  if (eta == 0) {
    q += p;
    p = 0;
  }
  if (zeta == 0) {
    p += q;
    q = 0;
  }
  src->p = p;
  const double eta_over_p = p > 0 ? (double)eta / (double)p : 0.0;
  for (int64_t t = 0; t < p; ++t) {
    const int64_t e = (int64_t)src_next_below(src, (uint64_t)eta);
    if (src->exhausted) return 5;
    if (n >= cap) return 6;
    memcpy(idx_out + n * d, x->coords + e * d, sizeof(int64_t) * (size_t)d);
    x_out[n] = x->values[e];
    w_out[n] = eta_over_p;
    ++n;
  }
  if (q > 0) {
    const double zeta_over_q = (double)zeta / (double)q;
    int64_t* zeros = (int64_t*)malloc(sizeof(int64_t) * (size_t)(q * d));
    const int rc = zeros_rejection(x, q, rho, src, zeros, NULL);
    if (rc) {
      free(zeros);
      return rc;
    }
    for (int64_t t = 0; t < q; ++t) {
      if (n >= cap) {
        free(zeros);
        return 6;
      }
      memcpy(idx_out + n * d, zeros + t * d, sizeof(int64_t) * (size_t)d);
      x_out[n] = 0.0;
      w_out[n] = zeta_over_q;
      ++n;
    }
    free(zeros);
  }
  *n_out = n;
  return 0;
}

double or_estimate(int d, const int64_t* dims, int64_t r, const double* factors, int loss_kind,
                   double delta, int64_t n, const int64_t* idx, const double* x,
                   const double* w) { /* samplers.cpp:114-124 */
  double sum = 0.0;
  for (int64_t e = 0; e < n; ++e) {
    const double m = or_entry(d, dims, r, factors, idx + e * d);
    sum += w[e] * or_loss_value(loss_kind, delta, x[e], m);
  }
  return sum;
}
