/* gcpb.h — C-ABI of the B200-native stochastic GCP gradient engine.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj, the inner loop of fit_gcp_adam at
 * src/optimizer.cpp:115-120).  Each entry point names the reference interface
 * it replaces.  Plain pointers and sizes only; all host buffers are borrowed
 * for the duration of the call; the context owns all device memory.
 *
 * Status codes mirror the reference's exception classes:
 *   GCPB_OK 0, GCPB_ERR_RUNTIME 1 (std::runtime_error / CUDA / NCCL),
 *   GCPB_ERR_USAGE 2 (std::invalid_argument), GCPB_ERR_DOMAIN 3
 *   (std::domain_error), GCPB_ERR_RANGE 4 (std::out_of_range),
 *   GCPB_ERR_LOGIC 5 (std::logic_error).  gcpb_last_error(ctx) returns the
 *   message of the last failure on that context (gcpb_last_error(NULL) for
 *   failures of gcpb_create and the context-free helpers).
 *
 * Threading: a context is not thread-safe; use one host thread per device.
 * Work is ordered on the context's stream; calls that return host-visible
 * outputs synchronise that stream before returning.
 */
#ifndef GCPB_H
#define GCPB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GCPB_OK 0
#define GCPB_ERR_RUNTIME 1
#define GCPB_ERR_USAGE 2
#define GCPB_ERR_DOMAIN 3
#define GCPB_ERR_RANGE 4
#define GCPB_ERR_LOGIC 5

/* Factor / arithmetic type of a context.  The reference is fp64-only
 * (include/gcp/kruskal.hpp:16); fp32 is the B200 fast path. */
#define GCPB_F32 0
#define GCPB_F64 1

/* Dense tensor storage in HBM.  U8 holds exact small integers (binary or
 * count data), F32/F64 anything else. */
#define GCPB_STORE_U8 0
#define GCPB_STORE_F32 1
#define GCPB_STORE_F64 2
/* Binary data, one bit per entry: bit (lin & 31) of u32 word lin >> 5. */
#define GCPB_STORE_BIT 3

/* LossKind, same order as include/gcp/loss.hpp:8-15. */
#define GCPB_LOSS_GAUSSIAN 0
#define GCPB_LOSS_POISSON 1
#define GCPB_LOSS_BERNOULLI_ODDS 2
#define GCPB_LOSS_GAMMA 3
#define GCPB_LOSS_BETA_HALF 4
#define GCPB_LOSS_HUBER 5

/* SamplerKind::Strategy, include/gcp/samplers.hpp:32. */
#define GCPB_UNIFORM 0
#define GCPB_STRATIFIED 1
#define GCPB_SEMI_STRATIFIED 2

/* EstimatorSamples::Kind, include/gcp/samplers.hpp:259. */
#define GCPB_EST_UNIFORM 0
#define GCPB_EST_STRATIFIED 1

typedef struct gcpb_ctx gcpb_ctx;

/* LossFunction (include/gcp/loss.hpp:20-56): kind + huber delta. */
typedef struct {
  int32_t kind;
  double delta;
} gcpb_loss;

/* SamplerKind (include/gcp/samplers.hpp:31-51). */
typedef struct {
  int32_t strategy;
  int64_t num_samples;     /* s, uniform only */
  int64_t nonzero_samples; /* p */
  int64_t zero_samples;    /* q */
  double oversample;       /* rho, stratified rejection batch factor */
} gcpb_sampler;

/* RejectionStats (include/gcp/samplers.hpp:53-57). */
typedef struct {
  int64_t tested;
  int64_t accepted;
  int64_t rejected;
} gcpb_stats;

/* The FitConfig fields adam_step reads (include/gcp/optimizer.hpp:42-65),
 * plus the current learning rate (AdamState::learning_rate). */
typedef struct {
  double learning_rate;
  double beta1;
  double beta2;
  double epsilon;
  int32_t has_lower_bound;
  double lower_bound;
} gcpb_adam;

/* ---- lifetime ------------------------------------------------------------
 * Replaces KruskalModel(Shape, rank) + GradientSet/AdamState allocation
 * (src/kruskal.cpp:10-16, src/kernels.cpp:61-67, src/optimizer.cpp:19-29).
 * Factors start at zero.  dims: n_1..n_d (1 <= d <= 16, each < 2^31).      */
int gcpb_create(int device, int dtype, int ndims, const int64_t* dims, int64_t rank,
                gcpb_ctx** out);
void gcpb_destroy(gcpb_ctx* ctx);
const char* gcpb_last_error(const gcpb_ctx* ctx);
const char* gcpb_version(void);
/* Run the context's work on a caller-owned CUDA stream (cudaStream_t as void*);
 * NULL restores the context's own stream. */
int gcpb_set_stream(gcpb_ctx* ctx, void* stream);
void* gcpb_get_stream(gcpb_ctx* ctx);

/* ---- tensor data ----------------------------------------------------------
 * SparseTensor(Shape, indices, values) (src/tensor.cpp:10-41): coords are
 * nnz x d row-major int64; duplicates are summed, zeros dropped, entries
 * sorted by first-mode-fastest linear key (that order defines nonzero pick
 * ordinals).  Bad index -> GCPB_ERR_RANGE naming the mode.  Builds the
 * device SoA COO and the open-addressing hash of linear keys.              */
int gcpb_set_sparse(gcpb_ctx* ctx, int64_t nnz, const int64_t* coords, const double* values);
/* Device-resident ingest for generated data: keys_sorted (strictly
 * increasing linear keys, device pointer) and values (device pointer of
 * value_dtype GCPB_F32/GCPB_F64); copied into the context after all work
 * already queued on the device (any stream) has completed. */
int gcpb_set_sparse_device(gcpb_ctx* ctx, int64_t nnz, const uint64_t* d_keys_sorted,
                           const void* d_values, int value_dtype);
int64_t gcpb_nnz(const gcpb_ctx* ctx);
/* Normalised COO read-back (nnz x d int64, values as double). */
int gcpb_get_sparse(gcpb_ctx* ctx, int64_t* coords_out, double* values_out);
/* DenseTensor values (include/gcp/tensor.hpp:52-81), first-mode-fastest. */
int gcpb_set_dense(gcpb_ctx* ctx, const double* values, int storage);
/* Device-resident dense ingest from a device pointer in `storage` layout
 * (read after all work already queued on the device has completed). */
int gcpb_set_dense_device(gcpb_ctx* ctx, const void* d_values, int storage);
/* Synthetic dense binary tensor generated in HBM (BASELINE configs[1]):
 * x(i) ~ Bernoulli(m_i / (1 + m_i)) with m the rank-true_rank model given by
 * true_factors (double, flattened mode-major row-major), uniform from a
 * counter hash of (seed, linear index).  storage: GCPB_STORE_U8 or
 * GCPB_STORE_BIT (same values). */
int gcpb_generate_dense_bernoulli(gcpb_ctx* ctx, int64_t true_rank, const double* true_factors,
                                  uint64_t seed, int storage);
/* TensorView::norm (src/tensor.cpp:56-60,70-74): Frobenius norm of the data,
 * fp64 accumulation. */
int gcpb_tensor_norm(gcpb_ctx* ctx, double* out);
/* TensorView::value_at (include/gcp/tensor.hpp:95-97) for n indices. */
int gcpb_value_at(gcpb_ctx* ctx, int64_t n, const int64_t* idx, double* x_out);

/* ---- factors, gradient, moments -------------------------------------------
 * mode-wise n_k x r row-major double (KruskalModel::factor, GradientSet::modes,
 * AdamState::{first,second}_moment); mode = -1 means all modes flattened in
 * mode order (GradientSet::flatten order, src/kernels.cpp:74-85).           */
int gcpb_set_factors(gcpb_ctx* ctx, int mode, const double* values);
int gcpb_get_factors(gcpb_ctx* ctx, int mode, double* out);
int gcpb_get_grad(gcpb_ctx* ctx, int mode, double* out);
int gcpb_set_grad(gcpb_ctx* ctx, int mode, const double* values);
/* which: 0 = first moment B, 1 = second moment C. */
int gcpb_get_moment(gcpb_ctx* ctx, int which, int mode, double* out);
int gcpb_set_moment(gcpb_ctx* ctx, int which, int mode, const double* values);

/* ---- the hot path -------------------------------------------------------------
 * draw_gradient_samples + mttkrp_sampled_all (include/gcp/samplers.hpp:223-245,
 * src/kernels.cpp:137-168), fused: sample -> model entry -> loss derivative
 * -> weight -> d-mode sparse MTTKRP scatter.  The gradient (overwritten, not
 * accumulated) stays on the device.  Draws come from the Philox4x32-10 stream
 * keyed by `seed` at iteration `iter`; stats may be NULL.
 * Validation, forfeit rules and errors follow the reference.               */
int gcpb_stoch_grad(gcpb_ctx* ctx, const gcpb_sampler* sampler, const gcpb_loss* loss,
                    uint64_t seed, uint64_t iter, gcpb_stats* stats);

/* Parity: the sampler alone.  Writes n samples (returned in *n_out; cap is
 * the capacity) in the reference's GradientSamples order: index (n x d int64),
 * data value x, weight w, flag (1 = semi-stratified nonzero term, y uses
 * g(x,m) - g(0,m)), model entry m, final weighted derivative y. */
int gcpb_draw_samples(gcpb_ctx* ctx, const gcpb_sampler* sampler, const gcpb_loss* loss,
                      uint64_t seed, uint64_t iter, int64_t cap, int64_t* idx_out,
                      double* x_out, double* w_out, int32_t* flag_out, double* m_out,
                      double* y_out, int64_t* n_out, gcpb_stats* stats);
/* Parity: KruskalModel::entry + LossFunction::deriv + weight on given samples
 * (src/kruskal.cpp:47-58, src/loss.cpp:88-110, samplers.hpp:90-91,206).
 * flags may be NULL (all 0). */
int gcpb_eval_deriv(gcpb_ctx* ctx, int64_t n, const int64_t* idx, const double* x,
                    const double* w, const int32_t* flags, const gcpb_loss* loss,
                    double* m_out, double* y_out);
/* Parity: mttkrp_sampled_all on given (index, value) samples
 * (src/kernels.cpp:137-168); result in the context's gradient. */
int gcpb_mttkrp_samples(gcpb_ctx* ctx, int64_t n, const int64_t* idx, const double* y);

/* ---- optimizer ----------------------------------------------------------------
 * adam_step (src/optimizer.cpp:47-66): moments, bias-corrected step with
 * epsilon inside the sqrt, projection, iteration counter += 1; fused with
 * zeroing the gradient for the next stoch_grad. */
int gcpb_adam_step(gcpb_ctx* ctx, const gcpb_adam* adam);
/* AdamState::init (src/optimizer.cpp:19-29): zero moments, iterations = 0. */
int gcpb_adam_reset(gcpb_ctx* ctx);
int gcpb_get_iterations(gcpb_ctx* ctx, int64_t* out);
int gcpb_set_iterations(gcpb_ctx* ctx, int64_t iterations);

/* ---- device-resident iterations -----------------------------------------------
 * One iteration of the epoch loop body (src/optimizer.cpp:116-119):
 * stoch_grad + [all-reduce when sharded] + adam_step, with the gradient-replica
 * reduction folded into the Adam update.  No host synchronisation. */
int gcpb_step(gcpb_ctx* ctx, const gcpb_sampler* sampler, const gcpb_loss* loss, uint64_t seed,
              uint64_t iter, const gcpb_adam* adam);
/* The same iteration on a HOST-resident model, as the reference's loop body
 * sees it (draw_gradient_samples(x, model, ...) + adam_step(model&, ...) on a
 * host KruskalModel): model_in (flattened factors, GradientSet order) is
 * copied in before the step and the updated factors copied out to model_out
 * after it (either may be NULL).  One call, one synchronisation; page-locked
 * buffers (cudaHostAlloc / cudaHostRegister) are DMA'd in place (large models
 * of fp32 engines: narrowed on the host, see gcpb_last_transfer_bytes), pageable
 * ones through the context's pinned staging block.  Small problems (those
 * gcpb_run_steps runs as one cluster kernel) on page-locked in/out buffers
 * take one launch that reads and writes the host model directly. */
int gcpb_step_host(gcpb_ctx* ctx, const gcpb_sampler* sampler, const gcpb_loss* loss,
                   uint64_t seed, uint64_t iter, const gcpb_adam* adam, const double* model_in,
                   double* model_out);
/* Model bytes the last gcpb_step_host moved over the bus in each direction.
 * fp32 engines move large (>= 2^22 elements) page-locked fp64 models as fp32:
 * host threads round chunk after chunk (round-to-nearest-even, the device's own
 * conversion) into a pinned staging block while the DMA of the previous chunks
 * runs, and widen the returned chunks the same way, so half the bytes cross
 * PCIe and the result is bit-identical.  GCPB_NARROW=0 turns it off,
 * GCPB_HOST_THREADS sets the thread count (default: all cores but two, at
 * most 32), GCPB_NARROW_TAIL the percentage of an upload's rows that cross as
 * fp64 without a host pass (default 15: the host's rounding is the longer leg).
 * No reference counterpart (the reference's model never leaves the host). */
int gcpb_last_transfer_bytes(const gcpb_ctx* ctx, int64_t* h2d, int64_t* d2h);
/* n iterations iter0 .. iter0+n-1 replayed as one CUDA graph (captured once per
 * sampler/loss/seed/n configuration; the draw-stream iteration and Adam's
 * counter advance on the device).  Equivalent to n calls of gcpb_step.  For
 * the stratified sampler the rejection batches are planned on the device
 * (three per iteration); a shortfall is reported as GCPB_ERR_RUNTIME by the
 * next synchronising call. */
int gcpb_run_steps(gcpb_ctx* ctx, const gcpb_sampler* sampler, const gcpb_loss* loss,
                   uint64_t seed, uint64_t iter0, int64_t n, const gcpb_adam* adam);
/* Which engine ran the last gcpb_run_steps (or small-problem gcpb_step_host):
 * 0 = CUDA graph of fused steps,
 * 1 = the small-problem cluster kernel (all n iterations in one launch;
 * gcpb_step_host on page-locked buffers reads and writes the host model
 * from that kernel directly,
 * chosen when uniform draws, one rank, Philox, the model fits in shared
 * memory and s*d*r <= 16384; GCPB_NO_SMALL=1 disables it). */
int gcpb_steps_path(const gcpb_ctx* ctx);
/* Debug: with GCPB_GUARD=1 in the environment every device buffer is
 * allocated between two 4 KB guard bands that are verified when it is released
 * or regrown (the engine's own out-of-bounds-write check; no reference
 * counterpart).  Returns the corrupted guard bytes seen so far in this process
 * (-1 when guard mode is off); *buffers_checked = buffers verified. */
int64_t gcpb_debug_guard_failures(int64_t* buffers_checked);
/* Debug: in a checked build (-DGCPB_CHECKED, tools/checked_build.sh) the
 * gather / scatter sites of the hot path assert their indices on the device.
 * Returns the failed assertions so far (-1 when the library is not a checked
 * build) and the first failing site and value. */
int64_t gcpb_debug_check_failures(int64_t* first_site, int64_t* first_value);
/* Kernels launched by the last gcpb_run_steps call: the kernel nodes of the
 * replayed step graph (every kernel is this library's own), or 1 for the
 * one-launch small-problem path. */
int gcpb_run_steps_launches(const gcpb_ctx* ctx, int64_t* kernels);
/* Hot rows of the sparse tensor: *rows = rows selected over
 * all modes (the most frequent rows of each mode among the nonzeros, up to 32
 * per mode), *copies = privatized copies per hot row used by the last fused
 * scatter (0 = that scatter used none).  GCPB_HOT_T sets the target
 * reductions per address (default 256; 0 disables hot rows). */
int gcpb_hot_rows(const gcpb_ctx* ctx, int* rows, int* copies);
/* Interleaved factor/gradient table: *enabled = 1 when the
 * context keeps one (factor tables beyond L2, or GCPB_IL=1; GCPB_IL=0
 * disables), *last = 1 when the last fused scatter went to it (single-rank
 * iterations: gcpb_step, gcpb_step_host, gcpb_run_steps, the fit). */
int gcpb_interleaved(const gcpb_ctx* ctx, int* enabled, int* last);
/* Per-launch timing of the fused sample->MTTKRP kernel: CUDA events recorded
 * on the context's stream around each non-graph launch.  enable = 1 clears
 * and starts recording, 0 stops.  gcpb_kernel_time synchronises and returns
 * the summed event time and the number of timed launches. */
int gcpb_kernel_timing(gcpb_ctx* ctx, int enable);
int gcpb_kernel_time(gcpb_ctx* ctx, double* total_ms, int64_t* launches);
/* Draw stream of the samplers.  kind 0 (default): the Philox stream, `seed`
 * is its key and `iter` the iteration.  kind 1 (RefStream, parity mode): the
 * reference's RngStream sequence (src/rng.cpp:43-61) — `seed` is the stream
 * key (e.g. RngStream(s).split("gradients")), `iter` is ignored, and the
 * draw counter lives on the device, starts at `counter` and advances by the
 * draws each call consumes, in the reference's consumption order, so
 * successive calls continue one stream exactly like draw_gradient_samples
 * does.  A draw in next_below's rejection region (probability <= n/2^64) is
 * reported by the next synchronising call. */
int gcpb_set_draw_stream(gcpb_ctx* ctx, int kind, uint64_t counter);
int gcpb_get_draw_counter(gcpb_ctx* ctx, uint64_t* counter);
/* Wait for queued device work and report deferred device-side failures. */
int gcpb_synchronize(gcpb_ctx* ctx);

/* ---- exact gradients and sampler diagnostics (oracle-scale, on the device) -------
 * gradient_full (src/kernels.cpp:170-198): loss derivative at every entry
 * (N <= 1e8, the reference's cap) -> the context's gradient. */
int gcpb_gradient_full(gcpb_ctx* ctx, const gcpb_loss* loss);
/* gradient_poisson_implicit (src/kernels.cpp:200-235): exact Poisson gradient
 * from factor column sums plus a pass over the stored nonzeros only. */
int gcpb_gradient_poisson_implicit(gcpb_ctx* ctx, const gcpb_loss* loss);
/* empirical_bias_variance (src/samplers.cpp:134-168): `trials` stochastic
 * gradients (trial t = iteration t of the Philox stream keyed by seed; in
 * RefStream mode the stream RngStream-split(t) of the key `seed`, like the
 * reference's rng.split(t)); bias = ||mean - exact||_2, variance = mean
 * squared distance to the mean.  exact: flattened gradient (GradientSet
 * order) or NULL to use gcpb_gradient_full. */
int gcpb_bias_variance(gcpb_ctx* ctx, const gcpb_sampler* sampler, const gcpb_loss* loss,
                       int64_t trials, uint64_t seed, const double* exact, double* bias,
                       double* variance);
/* Per-coordinate moments of the same `trials` stochastic gradients: mean and
 * unbiased sample variance (M2 / (trials - 1)), GradientSet order; either
 * output may be NULL (acceptance.cpp:166-213 checks each coordinate's mean
 * against 3 standard errors). */
int gcpb_gradient_moments(gcpb_ctx* ctx, const gcpb_sampler* sampler, const gcpb_loss* loss,
                          int64_t trials, uint64_t seed, double* mean, double* variance);

/* ---- fit driver -------------------------------------------------------------------
 * fit_gcp_adam (src/optimizer.cpp:68-158) with the epoch loop on the device:
 * factors start as the reference's init (RngStream(seed).split("init") uniform
 * draws, rescaled to ||X||, kruskal.cpp:33-45,85-93) unless keep_factors;
 * the fixed estimator set and the gradient draws come from the Philox stream
 * keyed by RngStream(seed).split("estimator"/"gradients"); each epoch is
 * epoch_iters graph-replayed iterations; accept when F <= best, else roll back
 * factors, moments and counter, decay the rate, count a bad epoch. */
typedef struct {
  gcpb_sampler sampler;
  double learning_rate; /* alpha_0 */
  double beta1, beta2, epsilon;
  int64_t epoch_iters;
  int64_t max_bad_epochs;
  double decay;
  int32_t lower_bound_mode; /* 0: the loss's default bound, 1: lower_bound, 2: none */
  double lower_bound;
  int64_t estimator_samples;
  int32_t estimator_kind; /* -1: stratified if sparse, uniform if dense */
  int64_t max_epochs;
  uint64_t seed;
  int32_t keep_factors; /* 1: start from the factors already set */
  int32_t draw_stream;  /* 0: Philox streams keyed by the split keys; 1: RefStream — the
                           reference's own estimator and gradient draws */
} gcpb_fit_config;

/* FitTraceRecord (include/gcp/optimizer.hpp:30-36). */
typedef struct {
  int64_t epoch;
  double loss_estimate;
  double learning_rate;
  double seconds;
  int32_t accepted;
} gcpb_trace_record;

int gcpb_fit_gcp_adam(gcpb_ctx* ctx, const gcpb_loss* loss, const gcpb_fit_config* cfg,
                      gcpb_trace_record* trace, int64_t trace_cap, int64_t* n_trace,
                      double* final_estimate);

/* ---- loss estimator -------------------------------------------------------------
 * EstimatorSamples (include/gcp/samplers.hpp:257-351).  set: given samples;
 * draw: drawn on the device from the Philox stream (tags EST_*). */
int gcpb_estimator_set(gcpb_ctx* ctx, int64_t n, const int64_t* idx, const double* x,
                       const double* w);
int gcpb_estimator_draw(gcpb_ctx* ctx, int kind, int64_t count, double rho, uint64_t seed);
int64_t gcpb_estimator_size(const gcpb_ctx* ctx);
int gcpb_estimator_get(gcpb_ctx* ctx, int64_t* idx_out, double* x_out, double* w_out);
/* EstimatorSamples::estimate (src/samplers.cpp:114-124): fp64 accumulation in
 * a fixed order (bit-deterministic for a given model). */
int gcpb_estimate(gcpb_ctx* ctx, const gcpb_loss* loss, double* out);

/* ---- rollback snapshot (src/optimizer.cpp:101-105,129-140) ---------------------- */
int gcpb_snapshot_save(gcpb_ctx* ctx);
int gcpb_snapshot_restore(gcpb_ctx* ctx);

/* ---- multi-GPU (one process per GPU) ---------------------------------------------
 * Samples are sharded by ordinal range across ranks (gcpb_shard_range);
 * factors are replicated; the gradient is summed with an NCCL all-reduce. */
int gcpb_nccl_unique_id(char out[128]);
int gcpb_comm_init(gcpb_ctx* ctx, const char unique_id[128], int rank, int nranks);
int gcpb_set_shard(gcpb_ctx* ctx, int rank, int nranks);
/* Peer-mapped tables (NVLink / NVSwitch peer memory), the multi-GPU exchange
 * of the reference's per-worker partial reduction (src/kernels.cpp:148-166)
 * fused with adam_step (src/optimizer.cpp:47-66): after gcpb_peer_open every
 * sharded step runs ONE kernel per rank that reads its shard of rows' gradient
 * from every rank's table (P2P loads), sums it in rank order, re-zeroes it
 * there, applies Adam with its own moment rows (ZeRO-1) and writes the updated
 * factor rows into every rank's table (P2P stores), between two rank
 * barriers (NCCL, or the host communicator's all-gather).
 * gcpb_peer_handle exports this rank's table (CUDA IPC handle + layout) into
 * GCPB_PEER_HANDLE_BYTES bytes; every rank exchanges them out of band and
 * calls gcpb_peer_open with all nranks blobs in rank order (same-process peers
 * are used directly, others mapped with cudaIpcOpenMemHandle).  Only this
 * rank's moment rows are maintained afterwards (gcpb_get_moment returns the
 * shard's rows current, the others stale). */
#define GCPB_PEER_HANDLE_BYTES 256
int gcpb_peer_handle(gcpb_ctx* ctx, void* out);
int gcpb_peer_open(gcpb_ctx* ctx, const void* handles, int nranks);
/* Unmaps the peers' tables: later sharded steps take the NCCL all-reduce +
 * replicated adam_step path again (used when a rank could not map a peer).
 * After peer steps each row's Adam moments exist only on its owner (rows
 * gcpb_shard_range(sum_k n_k, rank, nranks) of the concatenated modes;
 * gcpb_get_moment is current for those rows only), so this is a usage error
 * (std::logic_error) until gcpb_adam_reset. */
int gcpb_peer_close(gcpb_ctx* ctx);
int gcpb_allreduce_grad(gcpb_ctx* ctx);
/* Host-callback communicator, an alternative to NCCL for process groups the
 * caller already has (gloo, MPI) and for in-process multi-context tests:
 * allgather: recv[i] = the value rank i sent (nranks entries);
 * allreduce: in-place element-wise sum of n doubles across ranks.
 * Callbacks return 0 on success.  Graph-replayed steps need NCCL. */
typedef int (*gcpb_allgather_i64_fn)(void* user, int64_t send, int64_t* recv);
typedef int (*gcpb_allreduce_f64_fn)(void* user, double* buf, int64_t n);
int gcpb_comm_init_host(gcpb_ctx* ctx, int rank, int nranks, gcpb_allgather_i64_fn allgather,
                        gcpb_allreduce_f64_fn allreduce, void* user);

/* ---- synthetic problems (src/synthetic.cpp), generated on the device ----------------
 * The reference's RngStream state (rng.hpp:15-47): key, draw counter and the
 * cached second Box-Muller normal.  Generators consume draws exactly as the
 * reference does and return the advanced state, so a problem generated here
 * is entry-for-entry the reference's problem for the same stream. */
typedef struct gcpb_rng {
  uint64_t key;
  uint64_t counter;
  int32_t has_cached_normal;
  double cached_normal;
} gcpb_rng;
int gcpb_rng_seed(uint64_t seed, gcpb_rng* out);                        /* RngStream(seed) */
int gcpb_rng_split(const gcpb_rng* in, uint64_t label, gcpb_rng* out);  /* rng.split(label) */
/* gen_gamma_problem (synthetic.cpp:26-41): truth = random_uniform(shape,
 * rank) -> the context's factors (and truth_out, unpadded fp64, if non-NULL);
 * dense data x = Exponential(mean = truth entry), storage F64 or F32.  No
 * 1e8-entry cap: any dense tensor that fits in HBM. */
int gcpb_gen_gamma_problem(gcpb_ctx* ctx, gcpb_rng* rng, int storage, double* truth_out);
/* BinaryProblemSpec (synthetic.hpp:22-31); the rank is the context's. */
typedef struct gcpb_binary_spec {
  double delta;   /* sparse-column keep probability, (0, 0.5) */
  double p_high;  /* one-probability at structural positions */
  double p_low;   /* noise one-probability elsewhere */
} gcpb_binary_spec;
/* gen_binary_problem (synthetic.cpp:58-146) -> sparse binary tensor + truth. */
int gcpb_gen_binary_problem(gcpb_ctx* ctx, const gcpb_binary_spec* spec, gcpb_rng* rng,
                            double* truth_out);

/* ---- tensor files (host; src/io.cpp) ------------------------------------------------
 * A coordinate list as read from / written to disk: d modes, dims[d], nnz
 * entries, coords nnz x d row-major 0-based, values[nnz].  Buffers filled by a
 * reader are owned by the struct: release with gcpb_coo_free.  Errors are
 * runtime errors "path[:line]: message" (status 1), like the reference's. */
typedef struct gcpb_coo {
  int d;
  int64_t dims[16];
  int64_t nnz;
  int64_t* coords;
  double* values;
} gcpb_coo;
/* read_tns (src/io.cpp:75-139): '#shape: n1 .. nd' header (optional; else
 * dims = per-mode index maxima), '#' comment lines, one entry per line as d
 * 1-based indices and a value.  Entries are returned in file order (not
 * normalised: gcpb_set_sparse sums duplicates and drops zeros, as the
 * reference's SparseTensor constructor does).  threads <= 0: all cores. */
int gcpb_tns_read(const char* path, int threads, gcpb_coo* out);
/* write_tns (src/io.cpp:141-151): header + 1-based entries, values %.17g. */
int gcpb_tns_write(const char* path, const gcpb_coo* coo);
/* Binary coordinate format "GCPBCOO1" (own): 40-byte header {magic[8],
 * u32 version=1, u32 d, i64 nnz, u32 index_bytes (4|8), u32 flags, u64 0},
 * i64 dims[d], coords nnz x d (index_bytes each, little-endian), f64 values. */
int gcpb_coo_write(const char* path, const gcpb_coo* coo);
int gcpb_coo_read(const char* path, int threads, gcpb_coo* out);
void gcpb_coo_free(gcpb_coo* coo);
/* read_dense / write_dense (src/io.cpp:195-250): raw little-endian f64 in
 * first-mode-fastest order, shape in the text sidecar path + ".shape".
 * gcpb_dense_shape fills d/dims; gcpb_dense_read fills values[prod(dims)]. */
int gcpb_dense_shape(const char* path, int* d, int64_t* dims);
int gcpb_dense_read(const char* path, int64_t n, double* values);
int gcpb_dense_write(const char* path, int d, const int64_t* dims, const double* values);

/* read_model / write_model (io.cpp:153-193): a 'd r' line, a dims line, then
 * each factor row by row, values %.17g (bit-exact round trip).  Read the
 * header first (d, dims[<=16], rank), then the factors (sum_k n_k*rank
 * doubles, GradientSet order). */
int gcpb_model_read_header(const char* path, int* d, int64_t* dims, int64_t* rank);
int gcpb_model_read(const char* path, double* factors);
int gcpb_model_write(const char* path, int d, const int64_t* dims, int64_t rank,
                     const double* factors);
/* write_trace_csv (io.cpp:252-260): epoch,loss_estimate,learning_rate,seconds,accepted. */
int gcpb_trace_write_csv(const char* path, const gcpb_trace_record* records, int64_t n);

/* ---- host-only helpers (no device needed) ----------------------------------------- */
/* Product Philox stream: bounded draw in [0, n). */
uint64_t gcpb_philox_bounded(uint64_t seed, uint32_t tag, uint64_t iter, uint64_t t, int slot,
                             uint64_t n);
/* One zero-rejection batch size (include/gcp/samplers.hpp:118-122). */
int64_t gcpb_zero_batch_size(double total, double zeta, double rho, int64_t shortfall);
/* Contiguous ordinal range [begin, end) of n units owned by rank of nranks. */
void gcpb_shard_range(int64_t n, int rank, int nranks, int64_t* begin, int64_t* end);
/* Stratified multi-rank merge: given every rank's count of accepted zero
 * candidates in its slice (candidate order = rank order), the global rank
 * offset of this rank's first accept and how many of its accepts to keep so
 * that exactly the first `need` accepts overall are kept. */
void gcpb_stratified_keep(const int64_t* accepted_per_rank, int nranks, int rank, int64_t need,
                          int64_t* offset, int64_t* keep);
/* Loss derivative / value in double (LossFunction::deriv/value). */
double gcpb_loss_deriv(const gcpb_loss* loss, double x, double m);
double gcpb_loss_value(const gcpb_loss* loss, double x, double m);

#ifdef __cplusplus
}
#endif
#endif /* GCPB_H */
