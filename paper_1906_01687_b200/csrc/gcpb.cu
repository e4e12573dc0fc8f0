// gcpb.cu — context layer and C-ABI (include/gcpb.h).
//
// Owns every device buffer of one GCP problem on one GPU:
//   factors A, gradient G, Adam moments B, C (+ rollback snapshots), all in
//   one padded mode-major buffer each; the tensor (dense U8/F32/F64 array, or
//   SoA int32 COO + values + sorted u64 keys + open-addressing hash); the
//   fixed estimator sample set; the device-resident scalar state.
// Errors are C++ exceptions internally, mapped at the boundary onto the
// reference's exception classes (status codes, gcpb_last_error()).
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <nccl.h>

#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/gcpb.h"
#include "gcpb_aux.cuh"
#include "gcpb_gen.cuh"
#include "gcpb_small.cuh"
#include "gcpb_kernels.cuh"
#include "rngstream.h"

namespace gcpb {  // gcpb_host.cpp
void narrow_f64_f32(const double* src, float* dst, size_t n);
void widen_f32_f64(const float* src, double* dst, size_t n);
}  // namespace gcpb

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

using namespace gcpb;

namespace {

thread_local std::string g_global_err;

struct cuda_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw cuda_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}
#define CK(x) ck((x), #x)

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw std::runtime_error(std::string("NCCL error in ") + what + ": " + ncclGetErrorString(r));
}

// Simple owning device buffer.
// Bumped whenever device scratch is (re)allocated or freed: part of the key
// of the cached step graph (gcpb_run_steps), which holds raw buffer
// addresses -- a buffer regrown by a plain call in between must not be
// replayed through a stale graph.
std::atomic<uint64_t> g_dbuf_gen{0};

#ifdef GCPB_CHECKED
__device__ unsigned long long g_chk_dev[4];  // GCPB_CHECK: failures, first site, first value
#endif
unsigned long long* chk_counters() {
#ifdef GCPB_CHECKED
  void* p = nullptr;
  ck(cudaGetSymbolAddress(&p, g_chk_dev), "cudaGetSymbolAddress");
  return static_cast<unsigned long long*>(p);
#else
  return nullptr;
#endif
}

// Guarded allocations (GCPB_GUARD=1; the pool has compute-sanitizer closed, so
// this is the engine's own out-of-bounds-write check): every device buffer
// sits between two 4 KB bands of 0xA5, the tail band starting at the exact
// requested size, and the bands are verified when the buffer is released or
// regrown.  gcpb_debug_guard_failures() reports the corrupted bytes seen so
// far; tests/conftest.py asserts it stays zero after every GPU test.
constexpr size_t kGuardBytes = 4096;
const bool g_guard_on = getenv("GCPB_GUARD") != nullptr && atoi(getenv("GCPB_GUARD")) != 0;
std::atomic<long long> g_guard_bad{0}, g_guard_checked{0};

struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  size_t asked = 0;  // guard mode: the tail band starts at p + asked
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { reset(); }
  void verify_guards() {
    std::vector<unsigned char> h(2 * kGuardBytes);
    unsigned char* raw = static_cast<unsigned char*>(p) - kGuardBytes;
    if (cudaDeviceSynchronize() != cudaSuccess) return;  // a failed context is reported elsewhere
    if (cudaMemcpy(h.data(), raw, kGuardBytes, cudaMemcpyDeviceToHost) != cudaSuccess) return;
    if (cudaMemcpy(h.data() + kGuardBytes, static_cast<unsigned char*>(p) + asked, kGuardBytes,
                   cudaMemcpyDeviceToHost) != cudaSuccess)
      return;
    long long bad = 0;
    for (unsigned char b : h) bad += b != 0xA5;
    g_guard_bad.fetch_add(bad, std::memory_order_relaxed);
    g_guard_checked.fetch_add(1, std::memory_order_relaxed);
  }
  void reset() {
    if (p) {
      if (g_guard_on) {
        verify_guards();
        cudaFree(static_cast<unsigned char*>(p) - kGuardBytes);
      } else {
        cudaFree(p);
      }
      g_dbuf_gen.fetch_add(1, std::memory_order_relaxed);
    }
    p = nullptr;
    bytes = 0;
  }
  void alloc(size_t n) {
    if (n <= bytes && p) return;
    reset();
    if (n == 0) n = 16;
    if (g_guard_on) {
      unsigned char* raw = nullptr;
      ck(cudaMalloc(reinterpret_cast<void**>(&raw), n + 2 * kGuardBytes), "cudaMalloc");
      ck(cudaMemset(raw, 0xA5, kGuardBytes), "cudaMemset");
      ck(cudaMemset(raw + kGuardBytes + n, 0xA5, kGuardBytes), "cudaMemset");
      ck(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
      p = raw + kGuardBytes;
      asked = n;
    } else {
      ck(cudaMalloc(&p, n), "cudaMalloc");
    }
    g_dbuf_gen.fetch_add(1, std::memory_order_relaxed);
    bytes = n;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Scratch of one ordered sample list (order_build).
struct OrderBufs {
  DBuf out, cnt;
  int64_t out_cap = 0, bins_cap = 0;
};

const char* loss_name(int kind) {
  switch (kind) {
    case GCPB_LOSS_GAUSSIAN: return "gaussian";
    case GCPB_LOSS_POISSON: return "poisson";
    case GCPB_LOSS_BERNOULLI_ODDS: return "bernoulli-odds";
    case GCPB_LOSS_GAMMA: return "gamma";
    case GCPB_LOSS_BETA_HALF: return "beta-half";
    case GCPB_LOSS_HUBER: return "huber";
  }
  return "?";
}

void validate_loss(const gcpb_loss* loss) {
  if (!loss) throw std::invalid_argument("loss: null");
  if (loss->kind < 0 || loss->kind > 5) throw std::invalid_argument("unknown loss kind");
  if (loss->kind == GCPB_LOSS_HUBER && !(loss->delta > 0.0))
    throw std::invalid_argument("huber: delta must be > 0");  // loss.cpp:17-18
}

// LossFunction::check_domain (loss.cpp:42-62) on one value.
void check_domain_value(int kind, double x) {
  switch (kind) {
    case GCPB_LOSS_POISSON:
    case GCPB_LOSS_GAMMA:
    case GCPB_LOSS_BETA_HALF:
      if (!(x >= 0.0))
        throw std::domain_error(std::string(loss_name(kind)) + " loss: data value " +
                                std::to_string(x) + " out of domain (x >= 0 required)");
      return;
    case GCPB_LOSS_BERNOULLI_ODDS:
      if (x != 0.0 && x != 1.0)
        throw std::domain_error(std::string(loss_name(kind)) + " loss: data value " +
                                std::to_string(x) + " out of domain (x in {0,1} required)");
      return;
    default:
      return;
  }
}

// SamplerKind::validate (samplers.cpp:56-67).
void validate_sampler(const gcpb_sampler* s) {
  if (!s) throw std::invalid_argument("sampler: null");
  if (s->strategy == GCPB_UNIFORM) {
    if (s->num_samples < 1) throw std::invalid_argument("uniform sampler: s must be >= 1");
    return;
  }
  if (s->strategy != GCPB_STRATIFIED && s->strategy != GCPB_SEMI_STRATIFIED)
    throw std::invalid_argument("unknown sampler strategy");
  if (s->nonzero_samples < 0 || s->zero_samples < 0 ||
      s->nonzero_samples + s->zero_samples < 1)
    throw std::invalid_argument("sampler: need p, q >= 0 and p + q >= 1");
  if (s->strategy == GCPB_STRATIFIED && !(s->oversample > 1.0))
    throw std::invalid_argument("stratified sampler: oversample rate must be > 1");
}

std::string u128_to_string(unsigned __int128 v) {
  if (v == 0) return "0";
  std::string s;
  while (v > 0) {
    s.push_back(static_cast<char>('0' + static_cast<int>(v % 10)));
    v /= 10;
  }
  std::reverse(s.begin(), s.end());
  return s;
}

// Bytes of dense storage for n entries.
size_t dense_bytes(int storage, uint64_t n) {
  switch (storage) {
    case GCPB_STORE_U8: return n;
    case GCPB_STORE_F32: return n * 4;
    case GCPB_STORE_F64: return n * 8;
    case GCPB_STORE_BIT: return (n + 31) / 32 * 4;
  }
  throw std::invalid_argument("unknown dense storage");
}

// Measured-choice switches, read from the environment once
// per context at gcpb_create so that every later call -- and every cached
// step graph -- sees the same values.  None changes results beyond the
// gradient's summation order.
struct Tuning {
  int il = -1;          // GCPB_IL: interleaved [A | G] table (-1: by size)
  int sortq = -1;       // GCPB_SORTQ: unrestricted draws in mode-0 order (-1: with IL)
  int qshift = 5;       // GCPB_QSHIFT: log2 mode-0 rows per ordering bin (C5 step 3.64 / 3.66 /
                        // 3.59 / 3.62 / 3.67 / 3.81 ms at 3 / 4 / 5 / 6 / 7 / 8)
  double hot_t = 256.0; // GCPB_HOT_T: reductions per address before a row is privatized
  int replicas = 0;     // GCPB_REPLICAS: forced gradient replica count (0: by load)
  bool no_small = false;  // GCPB_NO_SMALL: no one-launch small-problem path
  bool no_bloom = false;  // GCPB_NO_BLOOM: zero sampler without the Bloom prefilter
  int adam = 1;           // GCPB_ADAM: streaming Adam variant for tables in HBM (0 = off)
  // Resident fused blocks per SM on the interleaved table (0 = as many as fit):
  // GCPB_FUSED_BPS for launches of picks only, GCPB_FUSED_BPS2 for launches that
  // walk an ordered list.  C5, one launch for both: 3.46 / 2.87 / 2.95 ms at
  // 2 / 3 / 4; split launches (picks, list): step 3.72 ms at (3, 3), 3.87 at
  // (3, 4), 3.62 at (4, 3), 3.78 at (4, 4), 4.06 at (3, 2).
  int fused_bps = 0;
  int fused_bps2 = 3;
  int list_hot = 0;       // GCPB_LIST_HOT: hot-row copies also for the list segment's own launch
                          // (uniform rows: a hot row sees q / n_k reductions, no contention)
  int ord_bps = 32;       // GCPB_ORD_BPS: blocks per SM of the ordering kernels' grids (short blocks
                          // hand their SM slots to the pick launch sooner: C5 step 3.79 / 3.62 /
                          // 3.61 / 3.59 / 3.57 / 3.56 / 3.56 ms at 1 / 2 / 4 / 8 / 16 / 32 / 64)
  int ord_side = 1;       // GCPB_ORD_SIDE: ordering on the side stream, under the pick half
  int side_bps = 3;       // GCPB_SIDE_BPS: fused blocks per SM of the pick launch while the side
                          // stream works (L2-resident tables; 0 = as many as fit; C3 step 235 / 228 /
                          // 253 / 342 us at 0 / 3 / 2 / 1)
  int host_threads = 0;   // GCPB_HOST_THREADS: threads of the narrowed model transfer (0 = all cores
                          // but two, at most 32)
  int pick_ahead = 0;     // GCPB_PICK_AHEAD: captured multi-rank steps compact the next step's picks
                          // under the current step's exchange kernel (second pick list).  Off by
                          // default: it pays only where the exchange leaves the SMs idle (NVLink),
                          // which one GPU cannot show (lone-rank probe: 4.65 vs 4.67 ms at 8 ranks,
                          // 3.66 vs 3.48 at 4, the local "exchange" being 0.2 ms of HBM traffic)
  bool lone_rank = false; // GCPB_DEBUG_LONE_RANK: a sharded rank alone on one GPU (timing and capture
                          // checks, tools/shard_probe.py): rank barriers are skipped and the step
                          // graph is captured without a communicator; the result is not a valid step
  int pick_side = 1;      // GCPB_PICK_SIDE: nonzero-sharded ranks compact their picks of the global stream on
                          // the side stream under the ordered list launch (which then goes first);
                          // 0 = off, 1 = on with 1 (3 from six ranks on) compaction blocks per SM,
                          // >= 2 = that many blocks per SM
  int narrow_tail = 15;   // GCPB_NARROW_TAIL: percent of a narrowed upload's rows (the last ones) that
                          // cross as fp64 without a host pass
  int narrow = 1;         // GCPB_NARROW: fp32 engines move large page-locked fp64 models as fp32,
                          // rounded / widened on the host while the DMA runs (0 = fp64 over the bus)
  void read_env() {
    if (const char* e = getenv("GCPB_HOST_THREADS")) host_threads = std::max(0, atoi(e));
    if (const char* e = getenv("GCPB_PICK_SIDE")) pick_side = atoi(e);
    lone_rank = getenv("GCPB_DEBUG_LONE_RANK") != nullptr;
    if (const char* e = getenv("GCPB_PICK_AHEAD")) pick_ahead = atoi(e);
    if (const char* e = getenv("GCPB_NARROW")) narrow = atoi(e);
    if (const char* e = getenv("GCPB_NARROW_TAIL")) narrow_tail = atoi(e);
    if (const char* e = getenv("GCPB_SIDE_BPS")) side_bps = std::max(0, atoi(e));
    if (const char* e = getenv("GCPB_LIST_HOT")) list_hot = atoi(e);
    if (const char* e = getenv("GCPB_FUSED_BPS2")) fused_bps2 = std::max(0, atoi(e));
    if (const char* e = getenv("GCPB_ORD_SIDE")) ord_side = atoi(e);
    if (const char* e = getenv("GCPB_ORD_BPS")) ord_bps = std::max(1, atoi(e));
    if (const char* e = getenv("GCPB_FUSED_BPS")) fused_bps = std::max(0, atoi(e));
    if (const char* e = getenv("GCPB_ADAM")) adam = atoi(e);
    if (const char* e = getenv("GCPB_IL")) il = atoi(e) != 0;
    if (const char* e = getenv("GCPB_SORTQ")) sortq = atoi(e) != 0;
    if (const char* e = getenv("GCPB_QSHIFT")) qshift = std::max(0, std::min(20, atoi(e)));
    if (const char* e = getenv("GCPB_HOT_T")) hot_t = atof(e);
    if (const char* e = getenv("GCPB_REPLICAS")) replicas = std::max(1, atoi(e));
    no_small = getenv("GCPB_NO_SMALL") != nullptr;
    no_bloom = getenv("GCPB_NO_BLOOM") != nullptr;
  }
};

}  // namespace

// ---------------------------------------------------------------------------
// The context
// ---------------------------------------------------------------------------
struct gcpb_ctx {
  int device = 0;
  int dtype = GCPB_F32;
  Tuning tune;  // environment switches, read once at gcpb_create
  size_t tsize = 4;
  int d = 0;
  int64_t dims[kMaxModes] = {};
  int64_t r = 0, rp = 0;
  int vw = 4;  // elements per 16-byte chunk
  unsigned __int128 total128 = 0;
  bool total_fits = true;  // N < 2^64
  bool wide = false;        // N >= 2^64: 128-bit keys (sparse tensors only)
  bool off64 = false;       // > 2^31 padded factor elements: 64-bit row offsets
  uint64_t stride_lo[kMaxModes] = {}, stride_hi[kMaxModes] = {};  // 128-bit strides
  uint64_t total = 0;
  double total_d = 0.0;
  int64_t off[kMaxModes + 1] = {};
  int64_t nelem = 0;  // padded elements of all modes
  int num_sms = 148;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  // Side stream for the ordering of the unrestricted draws (order_build): it
  // depends only on (seed, iteration), so it runs under the pick half of the
  // fused launch and joins before the ordered half (stoch_grad_impl,
  // run_fused); inside a step-graph capture the fork/join become graph edges.
  cudaStream_t side_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool join_pending = false;  // run_fused: wait for ev_join before the last segment
  int join_where = 0;         // 0: before the last segment (its list is built on the side stream);
                              // 1: before the FIRST segments (their pick list is compacted on the
                              // side stream), the last segment launched first; 2: before everything
  // peer steps keep each row's Adam moments on its owner only (ZeRO-1): set by
  // peer_adam_launch, cleared by gcpb_adam_reset; gcpb_peer_close refuses while set
  bool moments_sharded = false;
  std::string err;

  DBuf A, Gr, B, C, As, Bs, Cs;
  // Interleaved factor/gradient table for factor tables beyond L2 (C5):
  // rows [A row | G row] (pitch 2 rp), so a sample's row gather and its row
  // reduction share one 128-byte line (one DRAM burst) instead of two random
  // 64-byte accesses (tools/randbw.cu: +21..40%).  Used by the fused step
  // (scatter folded into Adam, one rank).  The IL Adam updates the factors in
  // AG only; A is refreshed from AG (a_current) before anything else reads
  // it.  ag_ok: AG's factor rows are current and its gradient rows zero;
  // a_stale: A is older than AG (implies ag_ok); il_pending: the last fused
  // scatter went to AG.
  DBuf AG;
  bool il_enabled = false;
  bool ag_ok = false;
  bool il_pending = false;
  bool il_gpack = false;  // sharded step: gradient packed from AG into Gr, factors in AG
  bool in_step = false;   // inside step_impl (the interleaved table is used only there)
  bool il_last = false;  // the last fused scatter used AG (gcpb_interleaved)
  bool a_stale = false;
  DBuf Grep;            // privatized gradient replicas (L2-resident), zero at rest
  int nrep = 1;         // replicas used by the current call
  int nrep_cap = 1;     // replicas allocated
  int64_t rep_stride = 0;
  DBuf dstate;
  DevState host_state{};
  double* pinned_params = nullptr;  // pinned staging block for Adam scalars
  bool adam_params_valid = false;
  bool grad_zero = false;
  bool have_snapshot = false;

  // tensor
  int tensor_kind = 0;  // 0 none, 1 dense, 2 sparse
  int dense_storage = GCPB_STORE_F64;
  DBuf dense;
  int64_t nnz = 0;
  DBuf nzrec, vals, keys;  // AoS nonzero records, values, sorted linear keys
  DBuf keys_hi, hkeys_hi;  // wide: high words of the keys and of the hash slots
  // Nonzero sharding: with nranks > 1 the records hold only
  // this rank's contiguous range [nz_begin, nz_end) of the sorted order; keys
  // and values stay whole (membership hash, value lookups).
  int64_t nz_begin = 0, nz_end = 0;
  DBuf pick_list;           // picks of the global stream in range (pick_compact_kernel)
  int64_t pick_cap = 0;
  // the next step's picks compacted ahead, under the current step's exchange
  // (captured multi-rank step graphs): second list, which list the current step
  // reads, the spec of the last compaction, steps left in the capture
  DBuf pick_list2;
  int pick_cur = 0;
  bool pick_ahead = false;
  bool pick_spec_valid = false;
  PickSpec pick_spec;
  int64_t steps_left = 0;
  cudaEvent_t ev_ahead = nullptr;
  DBuf mr_counts;           // multi-rank stratified: all-gathered accept counts
  int rec_words = 4;
  DBuf hkeys, hvals;
  uint64_t hmask = 0;
  DBuf bloom;          // blocked Bloom prefilter of the keys (32-byte blocks)
  uint64_t bmask = 0;
  bool hash_ready = false;
  int domain_flags = -1;  // cached domain scan of the stored data
  // hot rows (FusedArgs::hslot / Ghot): selected from the nonzeros' per-mode
  // row counts on the first sparse scatter after the tensor changes
  DBuf hslot, Ghot, hot_off;
  int64_t hot_version = -1;  // tensor_version the selection belongs to
  int hot_n = 0;             // hot rows over all modes
  int hot_rh_cap = 0;        // copies allocated per hot row
  int hot_last = 0;          // copies used by the last fused scatter
  int hot_pending = 0;       // copies the next adam_launch folds (0 = none)
  uint32_t hot_base[kMaxModes + 1] = {};
  uint32_t row_base[kMaxModes + 1] = {};
  double hot_fmax[kMaxModes] = {};  // largest share of the nonzeros in one row, per mode

  // fused-kernel event timing (gcpb_kernel_timing)
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tevents;
  size_t tevents_used = 0;

  // draw stream: 0 = Philox (default), 1 = RefStream (reference RngStream)
  int draw_stream = 0;

  // graph-replayed iterations (gcpb_run_steps)
  cudaGraphExec_t graph_exec = nullptr;
  std::string graph_key;
  int64_t tensor_version = 0;

  // sharding and communicator (NCCL or host callbacks)
  int rank = 0, nranks = 1;
  ncclComm_t comm = nullptr;
  gcpb_allgather_i64_fn host_allgather = nullptr;
  gcpb_allreduce_f64_fn host_allreduce = nullptr;
  void* host_user = nullptr;
  DBuf comm_buf;
  // peer-mapped factor/gradient tables of every rank (gcpb_peer_open): the
  // fused reduce-scatter + Adam + all-gather kernel (peer_adam_kernel)
  bool peer_ok = false;
  std::vector<void*> peer_a, peer_g;  // row bases per rank
  std::vector<void*> peer_ipc;        // mappings to close
  DBuf barrier_buf;                   // one int64 all-reduced as a rank barrier
  DBuf zscratch;  // multi-rank stratified: this rank's accepts of one batch
  int64_t zscratch_cap = 0;

  // stratified zero sampler
  DBuf zero_list, zstatus, ztbits;
  // semi-stratified unrestricted draws in mode-0 row order (large tables)
  OrderBufs qorder;
  int64_t zero_cap = 0, zstatus_cap = 0, z_nchunks_first = 0;

  // estimator
  int64_t est_n = 0;
  DBuf est_idx, est_x, est_w, est_partials, est_out;

  // scratch for parity / record paths
  DBuf s_idx, s_x, s_w, s_flag, s_m, s_y, s_aux;
  DBuf dims_dev;

  // factor-sized host<->device transfers: pinned staging + device staging
  // (unpadded fp64 rows), packed/unpacked by a kernel; one copy per call
  double* xfer_host = nullptr;
  size_t xfer_cap = 0;
  DBuf small_g;               // triple-buffered gradient of the small-problem kernel
  bool small_g_zero = false;
  int last_steps_path = 0;    // 0: CUDA graph of fused steps, 1: small-problem cluster kernel
  int64_t graph_kernels = 0;  // kernel nodes of the cached step graph
  DBuf xfer_dev;
  cudaEvent_t xfer_done = nullptr;
  // narrowed transfers (fp32 engines, page-locked host buffers, large models):
  // pinned fp32 staging, one event per chunk, bytes moved by the last transfer
  float* x32_host = nullptr;
  size_t x32_cap = 0;
  std::vector<cudaEvent_t> x32_ev;
  int64_t last_h2d_bytes = 0, last_d2h_bytes = 0;

  ~gcpb_ctx() {
    for (auto& pr : tevents) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    if (pinned_params) {
      cudaStreamSynchronize(stream);
      cudaFreeHost(pinned_params);
    }
    if (xfer_host) {
      cudaStreamSynchronize(stream);
      cudaFreeHost(xfer_host);
    }
    if (xfer_done) cudaEventDestroy(xfer_done);
    if (x32_host) {
      cudaStreamSynchronize(stream);
      cudaFreeHost(x32_host);
    }
    for (cudaEvent_t e : x32_ev) cudaEventDestroy(e);
    for (void* pmap : peer_ipc) cudaIpcCloseMemHandle(pmap);
    if (comm) ncclCommDestroy(comm);
    if (ev_ahead) cudaEventDestroy(ev_ahead);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (side_stream) cudaStreamDestroy(side_stream);
    if (own_stream) cudaStreamDestroy(own_stream);
  }

  void sync() { CK(cudaStreamSynchronize(stream)); }
  DevState* dst() const { return dstate.as<DevState>(); }

  void push_state() {
    CK(cudaMemcpyAsync(dstate.p, &host_state, sizeof(DevState), cudaMemcpyHostToDevice, stream));
  }
  void pull_state() {
    CK(cudaMemcpyAsync(&host_state, dstate.p, sizeof(DevState), cudaMemcpyDeviceToHost, stream));
    sync();
  }
  void check_mode(int mode) const {
    if (mode < -1 || mode >= d) throw std::invalid_argument("mode out of range");
  }
  int64_t mode_elems(int mode) const {  // unpadded n_k * r (or all modes)
    if (mode >= 0) return dims[mode] * r;
    int64_t s = 0;
    for (int k = 0; k < d; ++k) s += dims[k] * r;
    return s;
  }
};

namespace {

// NVTX range around a C-ABI call (visible in Nsight Systems / ncu --nvtx; a
// no-op without an attached tool).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

template <typename F>
int guard(gcpb_ctx* ctx, F&& f) {
  std::string* err = ctx ? &ctx->err : &g_global_err;
  if (ctx) {  // no side-stream join survives a call that threw
    ctx->join_pending = false;
    ctx->join_where = 0;
    ctx->pick_ahead = false;
    ctx->steps_left = 0;
  }
  try {
    f();
    return GCPB_OK;
  } catch (const std::invalid_argument& e) {
    *err = e.what();
    return GCPB_ERR_USAGE;
  } catch (const std::domain_error& e) {
    *err = e.what();
    return GCPB_ERR_DOMAIN;
  } catch (const std::out_of_range& e) {
    *err = e.what();
    return GCPB_ERR_RANGE;
  } catch (const std::logic_error& e) {
    *err = e.what();
    return GCPB_ERR_LOGIC;
  } catch (const std::exception& e) {
    *err = e.what();
    return GCPB_ERR_RUNTIME;
  } catch (...) {
    *err = "unknown error";
    return GCPB_ERR_RUNTIME;
  }
}

int grid_for(int64_t n, int threads, int num_sms, int per_sm = 8) {
  int64_t b = (n + threads - 1) / threads;
  const int64_t cap = static_cast<int64_t>(num_sms) * per_sm;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return static_cast<int>(b);
}

// check_index (shape.cpp:73-85) message format.
void check_index_host(const gcpb_ctx* c, const int64_t* idx) {
  for (int k = 0; k < c->d; ++k) {
    if (idx[k] < 0 || idx[k] >= c->dims[k])
      throw std::out_of_range("index " + std::to_string(idx[k]) + " out of range [0, " +
                              std::to_string(c->dims[k]) + ") in mode " + std::to_string(k));
  }
}

// Host-side factor layout conversion: n_k x r double <-> padded n_k x rp T.
// Rows of modes [k0, k1) are contiguous in both layouts: unpadded n_k x r
// (host, GradientSet order) and padded n_k x rp (device, from off[k0]).
void xfer_reserve(gcpb_ctx* c, size_t elems) {
  if (!c->xfer_done) CK(cudaEventCreateWithFlags(&c->xfer_done, cudaEventDisableTiming));
  if (elems > c->xfer_cap) {
    if (c->xfer_host) {
      CK(cudaEventSynchronize(c->xfer_done));
      CK(cudaFreeHost(c->xfer_host));
      c->xfer_host = nullptr;
    }
    CK(cudaMallocHost(reinterpret_cast<void**>(&c->xfer_host), elems * sizeof(double)));
    c->xfer_cap = elems;
  }
  c->xfer_dev.alloc(std::max<size_t>(elems, 1) * sizeof(double));
}

void mode_rows(const gcpb_ctx* c, int mode, int* k0, int* k1, int64_t* rows) {
  *k0 = mode < 0 ? 0 : mode;
  *k1 = mode < 0 ? c->d : mode + 1;
  *rows = 0;
  for (int k = *k0; k < *k1; ++k) *rows += c->dims[k];
}

// Page-locked (cudaHostAlloc / cudaHostRegister) host memory can be the DMA
// source or target itself, skipping the staging copy.
// Device address of page-locked host memory (null when p is not mapped).
const void* host_device_alias(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// direct: `values` is pinned and the caller synchronises before returning
// (gcpb_step_host), so the DMA reads it in place.
template <typename T>
void a_current_t(gcpb_ctx* c) {
  const int64_t nchunk = c->nelem / c->vw;
  ag_unsync_kernel<T><<<grid_for(nchunk, 256, c->num_sms, 8), 256, 0, c->stream>>>(
      c->AG.as<T>(), c->A.as<T>(), nchunk, static_cast<int>(c->rp));
  CK(cudaGetLastError());
}
// Refreshes A from the interleaved table when interleaved Adam updates left it stale.
void a_current(gcpb_ctx* c) {
  if (!c->a_stale) return;
  if (c->dtype == GCPB_F32)
    a_current_t<float>(c);
  else
    a_current_t<double>(c);
  c->a_stale = false;
}

// ---- narrowed model transfers (host halves in gcpb_host.cpp) -----------------------

constexpr size_t kNarrowChunk = size_t{1} << 19;  // elements per chunk (2 MB of fp32: short pipeline
                                                  // fill and drain, still full-rate DMAs)
constexpr size_t kNarrowMin = size_t{1} << 22;    // smaller transfers go as fp64 in one copy

bool narrow_eligible(const gcpb_ctx* c, size_t n, bool direct) {
  return direct && c->tune.narrow != 0 && c->dtype == GCPB_F32 && n >= kNarrowMin;
}

int narrow_threads(const gcpb_ctx* c, size_t nchunks) {
  // default: all cores but two (the calling thread queues the DMAs; C5 on 16
  // cores: 41.9 / 38.8 / 34.3 / 33.2 / 31.8 / 32.7 / 33.7 ms per host-buffer step
  // at 6 / 8 / 10 / 12 / 14 / 15 / 16 threads, 44.4 ms with fp64 over the bus)
  int t = c->tune.host_threads > 0 ? c->tune.host_threads
                                   : static_cast<int>(std::thread::hardware_concurrency()) - 2;
  t = std::max(1, std::min(t, 32));
  return static_cast<int>(std::min<size_t>(static_cast<size_t>(t), nchunks));
}

// Staging for a transfer whose first n_head elements cross as fp32 and whose
// last n_tail elements cross as fp64: pinned fp32 block of n_head, one event
// per chunk, and a device block holding the fp64 tail followed (padded rows
// only) by the fp32 head.
void narrow_reserve(gcpb_ctx* c, size_t n_head, size_t n_tail, size_t nchunks, bool padded) {
  if (!c->xfer_done) CK(cudaEventCreateWithFlags(&c->xfer_done, cudaEventDisableTiming));
  if (n_head > c->x32_cap) {
    if (c->x32_host) {
      CK(cudaStreamSynchronize(c->stream));
      CK(cudaFreeHost(c->x32_host));
      c->x32_host = nullptr;
    }
    CK(cudaMallocHost(reinterpret_cast<void**>(&c->x32_host), n_head * sizeof(float)));
    c->x32_cap = n_head;
  }
  while (c->x32_ev.size() < nchunks) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->x32_ev.push_back(e);
  }
  const size_t bytes = n_tail * sizeof(double) + (padded ? n_head * sizeof(float) : 0);
  if (bytes) c->xfer_dev.alloc(bytes);
}

// Rows that cross as fp64 without a host pass (the last rows of the transfer):
// the host's rounding, not the DMA, is the longer leg of a narrowed transfer, so
// a share of the rows goes the old way while the workers handle the rest.
// Measured on C5 (16 cores, tools/xfer_probe.py): copy-in leg 15.8 / 13.4 / 14.7 ms
// at 0 / 15 / 30 % (19.9 ms all fp64); the copy-out leg does not gain (12.7 / 13.5 /
// 14.4 ms, 19.2 ms all fp64), so only uploads take a tail.
int64_t narrow_tail_rows(const gcpb_ctx* c, int64_t rows, bool upload) {
  if (!upload) return 0;
  return rows * std::max(0, std::min(90, c->tune.narrow_tail)) / 100;
}

// Host fp64 rows -> device fp32 rows.  Head rows: worker threads round chunk
// after chunk into the pinned fp32 staging block, the calling thread queues each
// chunk's DMA as soon as it is ready (unpadded rows, r == rp, land in the table
// itself).  Tail rows: one fp64 DMA, queued first so the bus is busy while the
// first chunks are being rounded, converted by the unpack kernel.
void upload_narrow(gcpb_ctx* c, DBuf& buf, int k0, int64_t rows, const double* values) {
  const int64_t rows_tail = narrow_tail_rows(c, rows, true), rows_head = rows - rows_tail;
  const size_t n = static_cast<size_t>(rows_head * c->r);       // head elements
  const size_t n_tail = static_cast<size_t>(rows_tail * c->r);
  const size_t nchunks = (n + kNarrowChunk - 1) / kNarrowChunk;
  const bool padded = c->rp != c->r;
  narrow_reserve(c, n, n_tail, nchunks, padded);
  CK(cudaEventSynchronize(c->xfer_done));  // the previous transfer left the staging block
  double* dev_tail = c->xfer_dev.as<double>();
  float* dev_head = reinterpret_cast<float*>(dev_tail + n_tail);  // padded rows only
  float* table = buf.as<float>() + c->off[k0];
  float* dev = padded ? dev_head : table;
  const int nt = narrow_threads(c, nchunks);
  std::unique_ptr<std::atomic<int>[]> ready(new std::atomic<int>[nchunks]);
  for (size_t i = 0; i < nchunks; ++i) ready[i].store(0, std::memory_order_relaxed);
  float* stage = c->x32_host;
  std::vector<std::thread> pool;
  pool.reserve(static_cast<size_t>(nt));
  try {
    for (int t = 0; t < nt; ++t)
      pool.emplace_back([=, &ready] {
        for (size_t ch = static_cast<size_t>(t); ch < nchunks; ch += static_cast<size_t>(nt)) {
          const size_t b = ch * kNarrowChunk, e = std::min(n, b + kNarrowChunk);
          gcpb::narrow_f64_f32(values + b, stage + b, e - b);
          ready[ch].store(1, std::memory_order_release);
        }
      });
  } catch (...) {  // a thread could not be started: its chunks would never arrive
    for (auto& th : pool) th.join();
    throw;
  }
  cudaError_t err = cudaSuccess;
  if (n_tail) {
    err = cudaMemcpyAsync(dev_tail, values + n, n_tail * sizeof(double), cudaMemcpyHostToDevice,
                          c->stream);
    if (err == cudaSuccess) {
      const int64_t total = rows_tail * c->rp;
      unpack_rows_kernel<float, double><<<grid_for(total, 256, c->num_sms, 8), 256, 0, c->stream>>>(
          dev_tail, table + rows_head * c->rp, total, static_cast<int>(c->r),
          static_cast<int>(c->rp));
      err = cudaGetLastError();
    }
  }
  for (size_t ch = 0; ch < nchunks; ++ch) {
    while (!ready[ch].load(std::memory_order_acquire))  // leave the cores to the workers
      std::this_thread::sleep_for(std::chrono::microseconds(20));
    const size_t b = ch * kNarrowChunk, e = std::min(n, b + kNarrowChunk);
    if (err == cudaSuccess)
      err = cudaMemcpyAsync(dev + b, stage + b, (e - b) * sizeof(float), cudaMemcpyHostToDevice,
                            c->stream);
  }
  for (auto& th : pool) th.join();
  CK(err);
  CK(cudaEventRecord(c->xfer_done, c->stream));
  if (padded && rows_head > 0) {
    const int64_t total = rows_head * c->rp;
    unpack_rows_kernel<float, float><<<grid_for(total, 256, c->num_sms, 8), 256, 0, c->stream>>>(
        dev_head, table, total, static_cast<int>(c->r), static_cast<int>(c->rp));
    CK(cudaGetLastError());
  }
  c->last_h2d_bytes += static_cast<int64_t>(n * sizeof(float) + n_tail * sizeof(double));
}

// Device fp32 rows -> host fp64 rows.  Head rows: the chunks' DMAs are queued
// with an event each; worker threads widen a chunk into the caller's buffer once
// its event has passed.  Tail rows: widened on the device and copied as fp64
// straight into the caller's buffer, queued last (no host pass waits on them).
// Returns with the stream idle.
void download_narrow(gcpb_ctx* c, const DBuf& buf, int k0, int64_t rows, double* out) {
  const int64_t rows_tail = narrow_tail_rows(c, rows, false), rows_head = rows - rows_tail;
  const size_t n = static_cast<size_t>(rows_head * c->r);
  const size_t n_tail = static_cast<size_t>(rows_tail * c->r);
  const size_t nchunks = (n + kNarrowChunk - 1) / kNarrowChunk;
  const bool padded = c->rp != c->r;
  narrow_reserve(c, n, n_tail, nchunks, padded);
  CK(cudaEventSynchronize(c->xfer_done));
  double* dev_tail = c->xfer_dev.as<double>();
  float* dev_head = reinterpret_cast<float*>(dev_tail + n_tail);
  const float* table = buf.as<float>() + c->off[k0];
  const float* dev = table;
  if (padded && rows_head > 0) {
    pack_rows_kernel<float, float><<<grid_for(static_cast<int64_t>(n), 256, c->num_sms, 8), 256, 0,
                                     c->stream>>>(table, dev_head, static_cast<int64_t>(n),
                                                  static_cast<int>(c->r), static_cast<int>(c->rp));
    CK(cudaGetLastError());
    dev = dev_head;
  }
  float* stage = c->x32_host;
  for (size_t ch = 0; ch < nchunks; ++ch) {
    const size_t b = ch * kNarrowChunk, e = std::min(n, b + kNarrowChunk);
    CK(cudaMemcpyAsync(stage + b, dev + b, (e - b) * sizeof(float), cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaEventRecord(c->x32_ev[ch], c->stream));
  }
  if (n_tail) {
    pack_rows_kernel<float, double><<<grid_for(static_cast<int64_t>(n_tail), 256, c->num_sms, 8),
                                      256, 0, c->stream>>>(
        table + rows_head * c->rp, dev_tail, static_cast<int64_t>(n_tail), static_cast<int>(c->r),
        static_cast<int>(c->rp));
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out + n, dev_tail, n_tail * sizeof(double), cudaMemcpyDeviceToHost,
                       c->stream));
  }
  CK(cudaEventRecord(c->xfer_done, c->stream));
  const int nt = narrow_threads(c, nchunks);
  std::atomic<int> failed{0};
  const int device = c->device;
  cudaEvent_t* evs = c->x32_ev.data();
  std::vector<std::thread> pool;
  pool.reserve(static_cast<size_t>(nt));
  try {
    for (int t = 0; t < nt; ++t)
      pool.emplace_back([=, &failed] {
        cudaSetDevice(device);
        for (size_t ch = static_cast<size_t>(t); ch < nchunks; ch += static_cast<size_t>(nt)) {
          if (cudaEventSynchronize(evs[ch]) != cudaSuccess) {
            failed.store(1);
            return;
          }
          const size_t b = ch * kNarrowChunk, e = std::min(n, b + kNarrowChunk);
          gcpb::widen_f32_f64(stage + b, out + b, e - b);
        }
      });
  } catch (...) {
    for (auto& th : pool) th.join();
    cudaStreamSynchronize(c->stream);  // the staging block is still a DMA target
    throw;
  }
  for (auto& th : pool) th.join();
  if (failed.load()) CK(cudaStreamSynchronize(c->stream));  // surfaces the stream's error
  CK(cudaEventSynchronize(c->xfer_done));
  c->last_d2h_bytes += static_cast<int64_t>(n * sizeof(float) + n_tail * sizeof(double));
}

template <typename T>
void upload_modes(gcpb_ctx* c, DBuf& buf, int mode, const double* values, bool direct = false) {
  int k0, k1;
  int64_t rows;
  mode_rows(c, mode, &k0, &k1, &rows);
  const size_t n = static_cast<size_t>(rows * c->r);
  if (narrow_eligible(c, n, direct)) {
    upload_narrow(c, buf, k0, rows, values);
    return;
  }
  c->last_h2d_bytes += static_cast<int64_t>(n * sizeof(double));
  xfer_reserve(c, n);
  if (direct) {
    CK(cudaMemcpyAsync(c->xfer_dev.p, values, n * sizeof(double), cudaMemcpyHostToDevice,
                       c->stream));
  } else {
    CK(cudaEventSynchronize(c->xfer_done));  // the previous transfer left the staging block
    std::memcpy(c->xfer_host, values, n * sizeof(double));
    CK(cudaMemcpyAsync(c->xfer_dev.p, c->xfer_host, n * sizeof(double), cudaMemcpyHostToDevice,
                       c->stream));
    CK(cudaEventRecord(c->xfer_done, c->stream));
  }
  const int64_t total = rows * c->rp;
  unpack_rows_kernel<T><<<grid_for(total, 256, c->num_sms, 8), 256, 0, c->stream>>>(
      c->xfer_dev.as<double>(), buf.as<T>() + c->off[k0], total, static_cast<int>(c->r),
      static_cast<int>(c->rp));
  CK(cudaGetLastError());
}

template <typename T>
void download_modes(gcpb_ctx* c, const DBuf& buf, int mode, double* out, bool direct = false) {
  int k0, k1;
  int64_t rows;
  mode_rows(c, mode, &k0, &k1, &rows);
  const size_t n = static_cast<size_t>(rows * c->r);
  if (narrow_eligible(c, n, direct)) {
    download_narrow(c, buf, k0, rows, out);
    return;
  }
  c->last_d2h_bytes += static_cast<int64_t>(n * sizeof(double));
  xfer_reserve(c, n);
  CK(cudaEventSynchronize(c->xfer_done));
  pack_rows_kernel<T><<<grid_for(static_cast<int64_t>(n), 256, c->num_sms, 8), 256, 0, c->stream>>>(
      buf.as<T>() + c->off[k0], c->xfer_dev.as<double>(), static_cast<int64_t>(n),
      static_cast<int>(c->r), static_cast<int>(c->rp));
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(direct ? static_cast<void*>(out) : static_cast<void*>(c->xfer_host),
                     c->xfer_dev.p, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaEventRecord(c->xfer_done, c->stream));
  CK(cudaEventSynchronize(c->xfer_done));
  if (!direct) std::memcpy(out, c->xfer_host, n * sizeof(double));
}

void upload(gcpb_ctx* c, DBuf& buf, int mode, const double* v, bool direct = false) {
  if (&buf == &c->A) {
    if (mode < 0)
      c->a_stale = false;  // every row is overwritten
    else
      a_current(c);        // the other modes' rows must be current
    c->ag_ok = false;
  }
  if (c->dtype == GCPB_F32)
    upload_modes<float>(c, buf, mode, v, direct);
  else
    upload_modes<double>(c, buf, mode, v, direct);
}
void download(gcpb_ctx* c, const DBuf& buf, int mode, double* v, bool direct = false) {
  if (&buf == &c->A) a_current(c);
  if (c->dtype == GCPB_F32)
    download_modes<float>(c, buf, mode, v, direct);
  else
    download_modes<double>(c, buf, mode, v, direct);
}

void ensure_grad_zero(gcpb_ctx* c) {
  if (!c->grad_zero) {
    CK(cudaMemsetAsync(c->Gr.p, 0, c->nelem * c->tsize, c->stream));
    c->grad_zero = true;
  }
}

// Hash of the nonzero linear keys, built on first use.
// Membership hash + Bloom prefilter of 128-bit keys (N >= 2^64), built on the
// host from the sorted keys (same bucket layout as the 64-bit hash, high
// words in a parallel table; hash_find_wide / wide_digest).
void build_hash_wide(gcpb_ctx* c) {
  const int64_t n = c->nnz;
  std::vector<uint64_t> lo(static_cast<size_t>(n)), hi(static_cast<size_t>(n));
  if (n > 0) {
    CK(cudaMemcpyAsync(lo.data(), c->keys.p, n * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(hi.data(), c->keys_hi.p, n * 8, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
  }
  uint64_t buckets = 1;
  while (buckets * 2 < static_cast<uint64_t>(n)) buckets <<= 1;
  c->hmask = buckets - 1;
  std::vector<uint64_t> tlo(buckets * 4, kEmptyKey), thi(buckets * 4, kEmptyKey);
  std::vector<uint32_t> tv(buckets * 4, 0u);
  uint64_t blocks = 1;
  while (blocks * 32 < static_cast<uint64_t>(n)) blocks <<= 1;
  c->bmask = blocks - 1;
  std::vector<uint32_t> bl(static_cast<size_t>(blocks) * 8, 0u);
  for (int64_t e = 0; e < n; ++e) {
    const uint64_t dg = wide_digest(lo[e], hi[e]);
    for (uint64_t b = mix64(dg) & c->hmask;; b = (b + 1) & c->hmask) {
      int s = 0;
      while (s < 4 && !(tlo[b * 4 + s] == kEmptyKey && thi[b * 4 + s] == kEmptyKey)) ++s;
      if (s < 4) {
        tlo[b * 4 + s] = lo[e];
        thi[b * 4 + s] = hi[e];
        tv[b * 4 + s] = static_cast<uint32_t>(e);
        break;
      }
    }
    const uint64_t h = bloom_hash(dg);  // bloom_build_kernel's bits
    uint32_t* blk = bl.data() + (h & c->bmask) * 8;
    for (int b = 0; b < 3; ++b) {
      const uint32_t pos = static_cast<uint32_t>(h >> (40 + 8 * b)) & 255u;
      blk[pos >> 5] |= 1u << (pos & 31u);
    }
  }
  c->hkeys.alloc(tlo.size() * 8);
  c->hkeys_hi.alloc(thi.size() * 8);
  c->hvals.alloc(tv.size() * 4);
  c->bloom.alloc(bl.size() * 4);
  CK(cudaMemcpyAsync(c->hkeys.p, tlo.data(), tlo.size() * 8, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->hkeys_hi.p, thi.data(), thi.size() * 8, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->hvals.p, tv.data(), tv.size() * 4, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->bloom.p, bl.data(), bl.size() * 4, cudaMemcpyHostToDevice, c->stream));
  c->sync();  // host vectors die here
  c->hash_ready = true;
}

void ensure_hash(gcpb_ctx* c) {
  if (c->tensor_kind != 2) throw std::logic_error("hash requested without a sparse tensor");
  if (c->hash_ready) return;
  if (c->nnz >= (int64_t{1} << 32))
    throw std::invalid_argument("membership hash supports nnz < 2^32");
  if (c->wide) {
    build_hash_wide(c);
    return;
  }
  uint64_t buckets = 1;
  while (buckets * 2 < static_cast<uint64_t>(c->nnz)) buckets <<= 1;  // load <= 0.5
  if (buckets < 1) buckets = 1;
  c->hmask = buckets - 1;
  c->hkeys.alloc(buckets * 4 * sizeof(uint64_t));
  c->hvals.alloc(buckets * 4 * sizeof(uint32_t));
  CK(cudaMemsetAsync(c->hkeys.p, 0xFF, buckets * 4 * sizeof(uint64_t), c->stream));
  if (c->nnz > 0) {
    hash_build_kernel<<<grid_for(c->nnz, 256, c->num_sms), 256, 0, c->stream>>>(
        c->keys.as<uint64_t>(), c->nnz, c->hkeys.as<unsigned long long>(),
        c->hvals.as<uint32_t>(), c->hmask);
    CK(cudaGetLastError());
  }
  // Bloom prefilter: at most 32 keys per 32-byte block on average (C3: 16 MB,
  // 19 keys per block, ~1 % false positives with 3 bits per key).
  uint64_t blocks = 1;
  while (blocks * 32 < static_cast<uint64_t>(c->nnz)) blocks <<= 1;
  c->bmask = blocks - 1;
  c->bloom.alloc(blocks * 32);
  CK(cudaMemsetAsync(c->bloom.p, 0, blocks * 32, c->stream));
  if (c->nnz > 0) {
    bloom_build_kernel<<<grid_for(c->nnz, 256, c->num_sms), 256, 0, c->stream>>>(
        c->keys.as<uint64_t>(), c->nnz, c->bloom.as<uint32_t>(), c->bmask);
    CK(cudaGetLastError());
  }
  c->hash_ready = true;
}

// Data-domain scan (cached) -> domain_error like LossFunction::check_domain.
void check_data_domain(gcpb_ctx* c, int loss_kind) {
  if (loss_kind == GCPB_LOSS_GAUSSIAN || loss_kind == GCPB_LOSS_HUBER) return;
  if (c->tensor_kind == 0) return;
  if (c->domain_flags < 0) {
    c->s_aux.alloc(16);
    CK(cudaMemsetAsync(c->s_aux.p, 0, 4, c->stream));
    unsigned* f = c->s_aux.as<unsigned>();
    if (c->tensor_kind == 2) {
      if (c->nnz > 0) {
        if (c->dtype == GCPB_F32)
          domain_scan_kernel<float><<<grid_for(c->nnz, 256, c->num_sms), 256, 0, c->stream>>>(
              c->vals.as<float>(), c->nnz, f);
        else
          domain_scan_kernel<double><<<grid_for(c->nnz, 256, c->num_sms), 256, 0, c->stream>>>(
              c->vals.as<double>(), c->nnz, f);
      }
    } else {
      const int64_t n = static_cast<int64_t>(c->total);
      if (c->dense_storage == GCPB_STORE_BIT)
        ;  // values are 0/1 by construction
      else if (c->dense_storage == GCPB_STORE_U8)
        domain_scan_kernel<uint8_t><<<grid_for(n, 256, c->num_sms), 256, 0, c->stream>>>(
            c->dense.as<uint8_t>(), n, f);
      else if (c->dense_storage == GCPB_STORE_F32)
        domain_scan_kernel<float><<<grid_for(n, 256, c->num_sms), 256, 0, c->stream>>>(
            c->dense.as<float>(), n, f);
      else
        domain_scan_kernel<double><<<grid_for(n, 256, c->num_sms), 256, 0, c->stream>>>(
            c->dense.as<double>(), n, f);
    }
    CK(cudaGetLastError());
    unsigned flags = 0;
    CK(cudaMemcpyAsync(&flags, f, 4, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    c->domain_flags = static_cast<int>(flags);
  }
  const int f = c->domain_flags;
  if (loss_kind == GCPB_LOSS_BERNOULLI_ODDS && (f & 6))
    throw std::domain_error(std::string(loss_name(loss_kind)) +
                            " loss: data value out of domain (x in {0,1} required)");
  if ((loss_kind == GCPB_LOSS_POISSON || loss_kind == GCPB_LOSS_GAMMA ||
       loss_kind == GCPB_LOSS_BETA_HALF) &&
      (f & 5))
    throw std::domain_error(std::string(loss_name(loss_kind)) +
                            " loss: data value out of domain (x >= 0 required)");
}

bool nz_sharded(const gcpb_ctx* c) { return c->tensor_kind == 2 && c->nranks > 1; }

void no_nz_shard(const gcpb_ctx* c, const char* what) {
  if (nz_sharded(c))
    throw std::invalid_argument(std::string(what) +
                                " needs the whole nonzero set: not available on a "
                                "nonzero-sharded context (gcpb_set_shard with nranks > 1)");
}

// (Re)builds the nonzero records for this rank's range (all of them on one
// rank) from the sorted keys and values; the hot-row selection and cached
// step graphs follow the tensor version.
template <typename T>
void apply_nz_shard_t(gcpb_ctx* c) {
  int64_t b = 0, e = c->nnz;
  if (c->nranks > 1) gcpb_shard_range(c->nnz, c->rank, c->nranks, &b, &e);
  const bool whole = b == 0 && e == c->nnz;
  if (c->tensor_kind != 2 || (b == c->nz_begin && e == c->nz_end)) {
    c->nz_begin = b;
    c->nz_end = e;
    return;
  }
  const bool had_whole = c->nz_begin == 0 && c->nz_end == c->nnz;
  c->nz_begin = b;
  c->nz_end = e;
  c->tensor_version += 1;
  if (whole && had_whole) return;
  const int64_t n = e - b;
  c->nzrec.reset();  // shrink to the range
  c->nzrec.alloc(static_cast<size_t>(std::max<int64_t>(n, 1)) * c->rec_words * sizeof(uint32_t));
  if (n > 0) {
    T* v = c->vals.as<T>() + b;
    keys_to_records_kernel<T, T><<<grid_for(n, 256, c->num_sms), 256, 0, c->stream>>>(
        c->keys.as<uint64_t>() + b, v, n, c->d, c->dims_dev.as<int64_t>(), c->nzrec.as<uint32_t>(),
        c->rec_words, v, c->wide ? c->keys_hi.as<uint64_t>() + b : nullptr);
    CK(cudaGetLastError());
  }
  c->sync();
}

void apply_nz_shard(gcpb_ctx* c) {
  if (c->dtype == GCPB_F32)
    apply_nz_shard_t<float>(c);
  else
    apply_nz_shard_t<double>(c);
}

template <typename T>
FusedArgs<T> base_args(gcpb_ctx* c, const gcpb_loss* loss, uint64_t seed, uint64_t iter) {
  FusedArgs<T> a;
  std::memset(&a, 0, sizeof(a));
  a.A = c->A.as<T>();
  a.G = c->Gr.as<T>();
  a.chk = chk_counters();
  a.chk_tbl = c->nelem;
  a.nrep = 1;
  a.rep_stride = c->rep_stride;
  a.d = c->d;
  a.rp = static_cast<int>(c->rp);
  a.pitch = a.rp;
  a.nchunks = static_cast<int>((c->r + c->vw - 1) / c->vw);
  a.loss = loss ? loss->kind : 0;
  a.delta = static_cast<T>(loss ? loss->delta : 0.0);
  uint64_t stride = 1;
  for (int k = 0; k < c->d; ++k) {
    a.off[k] = c->off[k];
    a.dims[k] = static_cast<uint32_t>(c->dims[k]);
    a.thr[k] = lemire_threshold32(static_cast<uint64_t>(c->dims[k]));
    a.stride[k] = stride;
    stride *= static_cast<uint64_t>(c->dims[k]);
  }
  if (c->wide) {
    a.wide = 1;
    for (int k = 0; k < c->d; ++k) {
      a.stride[k] = c->stride_lo[k];
      a.stride_hi[k] = c->stride_hi[k];
    }
  }
  a.seed = seed;
  a.iter = iter;
  if (c->draw_stream == 1) {
    a.refstream = 1;
    a.ref_key = seed;
    a.ref_ctr = &c->dst()->ref_ctr;
    a.ref_flag = &c->dst()->ref_flag;
    for (int k = 0; k < c->d; ++k) {
      const uint64_t n = static_cast<uint64_t>(c->dims[k]);
      a.thr64[k] = (0 - n) % n;
    }
    const uint64_t eta = static_cast<uint64_t>(c->nnz > 0 ? c->nnz : 1);
    a.thr64_eta = (0 - eta) % eta;
  }
  if (c->tensor_kind == 1) {
    a.xkind = c->dense_storage == GCPB_STORE_BIT
                  ? X_DENSE_BIT
                  : (c->dense_storage == GCPB_STORE_U8
                         ? X_DENSE_U8
                         : (c->dense_storage == GCPB_STORE_F32 ? X_DENSE_F32 : X_DENSE_F64));
    a.dense = c->dense.p;
  } else if (c->tensor_kind == 2) {
    a.xkind = X_SPARSE;
    a.nzrec = c->nzrec.as<uint32_t>();
    a.rec_words = c->rec_words;
    a.vals = c->vals.as<T>();
    a.eta = static_cast<uint64_t>(c->nnz);
    a.thr_eta = c->nnz > 0 && static_cast<uint64_t>(c->nnz) <= (1ull << 32)
                    ? lemire_threshold32(static_cast<uint64_t>(c->nnz))
                    : 0u;
    a.nz_begin = c->nz_begin;
    a.nz_end = c->nz_end;
    if (c->hash_ready) {
      a.hkeys = c->hkeys.as<uint64_t>();
      a.hkeys_hi = c->hkeys_hi.as<uint64_t>();
      a.hvals = c->hvals.as<uint32_t>();
      a.hmask = c->hmask;
    }
  }
  a.scatter = 1;
  a.off64 = c->off64 ? 1 : 0;
  if (c->off64 && !((c->d == 3 || c->d == 4) && a.nchunks <= 32))
    throw std::invalid_argument("factor tables beyond 2^31 padded elements: the device path "
                                "supports d = 3, 4 and rows of at most 32 chunks (r <= 128 fp32, "
                                "r <= 64 fp64)");
  return a;
}

template <typename T>
int64_t finish_segments(FusedArgs<T>& a) {
  int64_t tiles = 0;
  for (int s = 0; s < a.nseg; ++s) {
    a.seg[s].tiles_begin = tiles;
    const int64_t len = a.seg[s].t_end - a.seg[s].t_begin;
    tiles += len > 0 ? (len + 31) / 32 : 0;
  }
  return tiles;
}

constexpr int kHotRows = 32;  // hot rows per mode

// Replicas worth using for a scatter of n samples: contention scales with the
// updates per 16-byte gradient chunk; one replica per ~4 updates per chunk on
// average, or per ~128 updates of a row of the shortest mode, capped by what
// is allocated (GCPB_REPLICAS forces the count).
int replicas_for(const gcpb_ctx* c, int64_t n) {
  if (c->nrep_cap < 2) return 1;
  if (c->tune.replicas > 0) return std::min(c->tune.replicas, c->nrep_cap);
  const int64_t chunks = std::max<int64_t>(1, c->nelem / c->vw);
  int64_t want = n / (4 * chunks);
  // short modes concentrate the reductions: a mode with n_k rows sees about
  // n / n_k per row; keep that under ~128 per replica (C4's 183-row mode:
  // R 2 -> 8, step 34.8 -> 32.6 us)
  // (modes of at most kHotRows rows are covered by hot-row copies on sparse data)
  for (int k = 0; k < c->d; ++k)
    if (c->tensor_kind != 2 || c->dims[k] > kHotRows)
      want = std::max<int64_t>(want, n / (128 * std::max<int64_t>(1, c->dims[k])));
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, c->nrep_cap)));
}

// Hot-row selection: per mode, up to kHotRows rows holding at
// least 1/1024 of the nonzeros each, from a device histogram of the records.
constexpr int kHotCopiesMax = 256;

void ensure_hot(gcpb_ctx* c) {
  if (c->hot_version == c->tensor_version) return;
  c->hot_version = c->tensor_version;
  c->hot_n = 0;
  if (c->tensor_kind != 2 || c->nz_end <= c->nz_begin || c->d > 4) return;
  int64_t rows = 0;
  for (int k = 0; k < c->d; ++k) {
    c->row_base[k] = static_cast<uint32_t>(rows);
    rows += c->dims[k];
  }
  if (rows >= (int64_t{1} << 31)) return;
  c->row_base[c->d] = static_cast<uint32_t>(rows);
  DBuf hist;
  hist.alloc(static_cast<size_t>(rows) * sizeof(uint32_t));
  CK(cudaMemsetAsync(hist.p, 0, static_cast<size_t>(rows) * sizeof(uint32_t), c->stream));
  RowBase rb;
  std::memset(&rb, 0, sizeof(rb));
  for (int k = 0; k < c->d; ++k) rb.v[k] = c->row_base[k];
  const int64_t nloc = c->nz_end - c->nz_begin;  // this rank's records
  row_hist_kernel<<<grid_for(nloc, 256, c->num_sms), 256, 0, c->stream>>>(
      c->nzrec.as<uint32_t>(), c->rec_words, static_cast<int>(c->tsize / 4), nloc, c->d, rb,
      hist.as<uint32_t>());
  CK(cudaGetLastError());
  std::vector<uint32_t> h(static_cast<size_t>(rows));
  CK(cudaMemcpyAsync(h.data(), hist.p, h.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                     c->stream));
  CK(cudaStreamSynchronize(c->stream));
  std::vector<uint8_t> slot(static_cast<size_t>(rows), 0xFF);
  std::vector<int64_t> hoff;
  const double nnz = static_cast<double>(std::max<int64_t>(1, nloc));
  for (int k = 0; k < c->d; ++k) {
    c->hot_base[k] = static_cast<uint32_t>(hoff.size());
    c->hot_fmax[k] = 0.0;
    std::vector<std::pair<uint32_t, uint32_t>> cand;  // (count, row)
    for (int64_t i = 0; i < c->dims[k]; ++i) {
      const uint32_t n = h[c->row_base[k] + i];
      if (static_cast<double>(n) * 1024.0 >= nnz) cand.emplace_back(n, static_cast<uint32_t>(i));
    }
    const size_t keep = std::min<size_t>(cand.size(), kHotRows);
    std::partial_sort(cand.begin(), cand.begin() + keep, cand.end(),
                      [](const auto& x, const auto& y) {
                        return x.first != y.first ? x.first > y.first : x.second < y.second;
                      });
    for (size_t j = 0; j < keep; ++j) {
      slot[c->row_base[k] + cand[j].second] = static_cast<uint8_t>(j);
      hoff.push_back(c->off[k] + static_cast<int64_t>(cand[j].second) * c->rp);
    }
    if (keep > 0) c->hot_fmax[k] = static_cast<double>(cand[0].first) / nnz;
  }
  c->hot_base[c->d] = static_cast<uint32_t>(hoff.size());
  c->hot_n = static_cast<int>(hoff.size());
  if (c->hot_n == 0) return;
  // copies per hot row: up to kHotCopiesMax within 8 MB (the copies stay in L2)
  const int64_t row_bytes = c->rp * static_cast<int64_t>(c->tsize);
  int cap = kHotCopiesMax;
  while (cap > 2 && static_cast<int64_t>(cap) * c->hot_n * row_bytes > (int64_t{8} << 20)) cap >>= 1;
  c->hot_rh_cap = cap;
  c->hslot.alloc(slot.size());
  CK(cudaMemcpyAsync(c->hslot.p, slot.data(), slot.size(), cudaMemcpyHostToDevice, c->stream));
  c->hot_off.alloc(hoff.size() * sizeof(int64_t));
  CK(cudaMemcpyAsync(c->hot_off.p, hoff.data(), hoff.size() * sizeof(int64_t),
                     cudaMemcpyHostToDevice, c->stream));
  const size_t gbytes = static_cast<size_t>(cap) * c->hot_n * row_bytes;
  c->Ghot.alloc(gbytes);
  CK(cudaMemsetAsync(c->Ghot.p, 0, gbytes, c->stream));
  CK(cudaStreamSynchronize(c->stream));  // host vectors die here
}

// Copies per hot row for one scatter (0 = hot rows off): the busiest row's
// expected reductions per step, picks at the mode's largest nonzero share
// plus its share of the unrestricted draws, over a target of kHotTarget
// reductions per address (GCPB_HOT_T), when that beats the block replicas.
template <typename T>
int hot_copies(gcpb_ctx* c, const FusedArgs<T>& a, int nrep) {
  const double target = c->tune.hot_t;
  if (target <= 0.0 || c->tensor_kind != 2 || c->d > 4 || c->rp / c->vw > 64) return 0;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(c->stream, &cs);
  if (cs == cudaStreamCaptureStatusNone)
    ensure_hot(c);
  else if (c->hot_version != c->tensor_version)
    return 0;
  if (c->hot_n == 0) return 0;
  double picks = 0.0, unif = 0.0;
  for (int s = 0; s < a.nseg; ++s) {
    const double len = static_cast<double>(std::max<int64_t>(0, a.seg[s].t_end - a.seg[s].t_begin));
    if (a.seg[s].kind == SEG_PICK) picks += len;
    else if (a.seg[s].kind <= SEG_ZERO_LIST) unif += len;
    else return 0;
  }
  double load = 0.0;
  for (int k = 0; k < c->d; ++k)
    load = std::max(load, picks * c->hot_fmax[k] + unif / static_cast<double>(c->dims[k]));
  int rh = 1;
  while (rh < c->hot_rh_cap && static_cast<double>(rh) * target < load) rh <<= 1;
  return rh > nrep ? rh : 0;
}

// Allocates AG and, unless AG already mirrors A (ag_ok), rebuilds it from A.
// Inside a graph capture the caller (run_steps_impl) has done this already.
template <typename T>
void ag_prepare(gcpb_ctx* c) {
  if (!c->AG.p) {
    const size_t bytes = static_cast<size_t>(2 * c->nelem) * c->tsize;
    c->AG.alloc(bytes);
    c->ag_ok = false;
  }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(c->stream, &cs));
  if (c->ag_ok || cs != cudaStreamCaptureStatusNone) return;
  const int64_t nchunk = c->nelem / c->vw;
  ag_sync_kernel<T><<<grid_for(nchunk, 256, c->num_sms, 8), 256, 0, c->stream>>>(
      c->A.as<T>(), c->AG.as<T>(), nchunk, static_cast<int>(c->rp));
  CK(cudaGetLastError());
  c->ag_ok = true;
}

template <typename T>
void run_fused(gcpb_ctx* c, FusedArgs<T>& a, bool record, bool fold = false) {
  const int64_t tiles = finish_segments(a);
  cudaEvent_t ev1 = nullptr;
  if (c->timing) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(c->stream, &cs);
    if (cs == cudaStreamCaptureStatusNone) {
      if (c->tevents_used == c->tevents.size()) {
        cudaEvent_t x, y;
        CK(cudaEventCreate(&x));
        CK(cudaEventCreate(&y));
        c->tevents.emplace_back(x, y);
      }
      auto& pr = c->tevents[c->tevents_used++];
      CK(cudaEventRecord(pr.first, c->stream));
      ev1 = pr.second;
    }
  }
  c->il_pending = false;
  c->il_gpack = false;
  // interleaved table: iterations only (folded single-rank steps, or sharded
  // steps whose gradient is packed back for the all-reduce)
  const bool il = a.scatter && !record && c->il_enabled && c->in_step && (fold || c->nranks > 1);
  if (il) {
    // interleaved table: the scatter goes to AG's gradient rows, Adam reads them
    ag_prepare<T>(c);
    a.A = c->AG.as<T>();
    a.G = c->AG.as<T>() + c->rp;
    a.pitch = static_cast<int>(2 * c->rp);
    for (int k = 0; k < c->d; ++k) a.off[k] = 2 * c->off[k];
    a.chk_tbl = 2 * c->nelem - c->rp;
    c->nrep = 1;
    a.nrep = 1;
    c->il_pending = fold;
    c->il_last = true;
  } else if (a.scatter) {
    a_current(c);
    c->il_last = false;
    int64_t n = 0;
    for (int s = 0; s < a.nseg; ++s) n += std::max<int64_t>(0, a.seg[s].t_end - a.seg[s].t_begin);
    c->nrep = replicas_for(c, n);
    a.nrep = c->nrep;
    a.G = c->nrep > 1 ? c->Grep.as<T>() : c->Gr.as<T>();
  } else {
    a_current(c);
  }
  if (a.scatter) {
    if (!record) {
      a.rh = hot_copies<T>(c, a, c->nrep);
      if (a.rh > 0) {
        a.hslot = c->hslot.as<uint8_t>();
        a.Ghot = c->Ghot.as<T>();
        a.chk_ghot = static_cast<int64_t>(c->Ghot.bytes / sizeof(T));
        for (int k = 0; k < c->d; ++k) {
          a.rowbase[k] = c->row_base[k];
          a.hbase[k] = c->hot_base[k];
        }
      }
    }
  }
  bool used_hot = false;
  const bool listed = a.zero_list32 != nullptr;  // the last segment walks an ordered list
  const int bps = il ? (listed && !c->join_pending ? c->tune.fused_bps2 : c->tune.fused_bps) : 0;
  if (c->join_pending) {
    // the last segment's ordered list is being built on the side stream: the
    // segments before it go first, the join, then the ordered segment
    c->join_pending = false;
    const int where = c->join_where;
    c->join_where = 0;
    if (a.nseg >= 2 && where == 1) {
      // the FIRST segments' pick list is being compacted on the side stream: the
      // ordered last segment goes first, the join, then the segments before it
      FusedArgs<T> a2 = a;
      a2.seg[0] = a.seg[a.nseg - 1];
      a2.nseg = 1;
      if (!c->tune.list_hot) a2.rh = 0;
      const int64_t t2 = finish_segments(a2);
      bool hot2 = false;
      CK(launch_fused<T>(a2, t2, record, c->stream, c->num_sms, &hot2,
                         il && listed ? c->tune.fused_bps2 : bps));
      CK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
      FusedArgs<T> a1 = a;
      a1.nseg = a.nseg - 1;
      const int64_t t1 = finish_segments(a1);
      CK(launch_fused<T>(a1, t1, record, c->stream, c->num_sms, &used_hot,
                         il ? c->tune.fused_bps : c->tune.side_bps));
      used_hot = used_hot || hot2;
    } else if (a.nseg >= 2 && where == 0) {
      FusedArgs<T> a1 = a;
      a1.nseg = a.nseg - 1;
      const int64_t t1 = finish_segments(a1);
      CK(launch_fused<T>(a1, t1, record, c->stream, c->num_sms, &used_hot,
                         il ? bps : c->tune.side_bps));
      CK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
      FusedArgs<T> a2 = a;
      a2.seg[0] = a.seg[a.nseg - 1];
      a2.nseg = 1;
      // uniformly drawn rows: straight into the gradient rows (the Adam fold
      // adds a hot row's copies to its gradient row), no hot-slot lookups
      if (!c->tune.list_hot) a2.rh = 0;
      const int64_t t2 = finish_segments(a2);
      bool hot2 = false;
      CK(launch_fused<T>(a2, t2, record, c->stream, c->num_sms, &hot2,
                         il && listed ? c->tune.fused_bps2 : bps));
      used_hot = used_hot || hot2;
    } else {
      CK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
      CK(launch_fused<T>(a, tiles, record, c->stream, c->num_sms, &used_hot, bps));
    }
  } else {
    CK(launch_fused<T>(a, tiles, record, c->stream, c->num_sms, &used_hot, bps));
  }
  if (a.scatter) c->hot_last = used_hot ? a.rh : 0;
  if (ev1) CK(cudaEventRecord(ev1, c->stream));
  if (il && !fold && !c->peer_ok) {  // the all-reduce needs the gradient contiguous
    const int64_t nchunk = c->nelem / c->vw;
    CK(launch_k(ag_pack_kernel<T>, dim3(grid_for(nchunk, 256, c->num_sms, 8)), dim3(256), 0,
                c->stream, c->AG.as<T>(), c->Gr.as<T>(), nchunk, static_cast<int>(c->rp)));
    c->il_gpack = true;
  }
  if (a.scatter && c->nrep > 1 && !fold) {  // fold: Adam sums the replicas itself
    const int64_t nchunk = c->nelem / c->vw;
    CK(launch_k(grad_reduce_kernel<T>, dim3(grid_for(nchunk * 8, 256, c->num_sms, 8)), dim3(256), 0,
                c->stream, c->Gr.as<T>(), c->Grep.as<T>(), nchunk, c->nrep, c->rep_stride));
  }
  c->hot_pending = 0;
  if (used_hot && fold) {  // the fused Adam folds the hot rows' copies itself
    c->hot_pending = a.rh;
  } else if (used_hot && il && c->peer_ok) {  // into the table's gradient rows (peer path)
    CK(launch_k(hot_fold_kernel<T>, dim3(c->hot_n), dim3(256), 0, c->stream, c->Ghot.as<T>(), a.rh,
                static_cast<int>(c->rp), c->hot_off.as<int64_t>(), c->AG.as<T>(), 1));
  } else if (used_hot) {   // hot rows' copies into the gradient
    CK(launch_k(hot_fold_kernel<T>, dim3(c->hot_n), dim3(256), 0, c->stream, c->Ghot.as<T>(), a.rh,
                static_cast<int>(c->rp), c->hot_off.as<int64_t>(), c->Gr.as<T>(), 0));
  }
}

Seg make_seg(int kind, uint32_t tag, int64_t tb, int64_t te, double w, int flag, int64_t out,
             int64_t ref_off = 0) {
  Seg s;
  std::memset(&s, 0, sizeof(s));
  s.ref_off = ref_off;
  s.kind = kind;
  s.tag = tag;
  s.t_begin = tb;
  s.t_end = te;
  s.weight = w;
  s.flag = flag;
  s.out_offset = out;
  return s;
}

// Sizes the zero-sampler buffers and uploads its per-call scalars (q, N, zeta,
// rho).  Kept out of graph capture (pageable-memory copies).
void prepare_zero_sampler(gcpb_ctx* c, int64_t q, double rho) {
  ensure_hash(c);
  const double zeta = static_cast<double>(c->total128 - static_cast<unsigned __int128>(c->nnz));
  const int64_t first_batch = zero_batch_size_dev(c->total_d, zeta, rho, q);
  const int64_t nchunks = (first_batch + kZcChunk - 1) / kZcChunk;
  if (c->zero_cap < q) {
    c->zero_list.alloc(static_cast<size_t>(q) * sizeof(uint64_t));
    c->zero_cap = q;
  }
  if (c->zstatus_cap < nchunks) {
    c->zstatus.alloc(static_cast<size_t>(nchunks) * sizeof(unsigned long long));
    c->ztbits.alloc(static_cast<size_t>(nchunks) * kZcThreads * sizeof(uint32_t));
    c->zstatus_cap = nchunks;
  }
  c->z_nchunks_first = nchunks;
  DevState* st = c->dst();
  c->host_state.z_q = q;
  c->host_state.z_total = c->total_d;
  c->host_state.z_zeta = zeta;
  c->host_state.z_rho = rho;
  c->host_state.z_status_cap = c->zstatus_cap;
  CK(cudaMemcpyAsync(&st->z_q, &c->host_state.z_q, sizeof(int64_t), cudaMemcpyHostToDevice,
                     c->stream));
  CK(cudaMemcpyAsync(&st->z_total, &c->host_state.z_total, 3 * sizeof(double),
                     cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(&st->z_status_cap, &c->host_state.z_status_cap, sizeof(int64_t),
                     cudaMemcpyHostToDevice, c->stream));
}

enum ZeroMode { ZERO_HOST_CHECK = 0, ZERO_DEVICE_ONLY = 1, ZERO_CAPTURE = 2 };

// Runs the stratified zero sampler for q accepts: fills zero_list[0..q) with
// candidate ordinals.  Three device-planned batches are queued without a host
// round trip; ZERO_HOST_CHECK then synchronises and continues host-side until
// exactly q accepts exist (reference semantics for any q); ZERO_CAPTURE (graph
// mode, prepared beforehand) only counts shortfalls on the device.
void fill_refstream(const gcpb_ctx* c, ZeroArgs& za, uint64_t key, int64_t p_ref) {
  if (c->draw_stream != 1) return;
  za.refstream = 1;
  za.ref_key = key;
  za.ref_off = p_ref;
  for (int k = 0; k < c->d; ++k) {
    const uint64_t n = static_cast<uint64_t>(c->dims[k]);
    za.thr64[k] = (0 - n) % n;
  }
}

void launch_zero_cand(const gcpb_ctx* c, int grid, const ZeroArgs& za) {
  if (c->wide) {  // 128-bit keys: the general-d instantiation
    CK(launch_k(zero_cand_kernel<0>, dim3(grid), dim3(kZcThreads), 0, c->stream, za));
    return;
  }
  switch (c->d) {
    case 3: CK(launch_k(zero_cand_kernel<3>, dim3(grid), dim3(kZcThreads), 0, c->stream, za)); break;
    case 4: CK(launch_k(zero_cand_kernel<4>, dim3(grid), dim3(kZcThreads), 0, c->stream, za)); break;
    default: CK(launch_k(zero_cand_kernel<0>, dim3(grid), dim3(kZcThreads), 0, c->stream, za)); break;
  }
}

ZeroArgs zero_args(gcpb_ctx* c, uint64_t seed, uint64_t iter, const uint64_t* iter_base,
                   uint32_t tag, int64_t p_ref) {
  DevState* st = c->dst();
  ZeroArgs za;
  std::memset(&za, 0, sizeof(za));
  za.d = c->d;
  uint64_t stride = 1;
  for (int k = 0; k < c->d; ++k) {
    za.dims[k] = static_cast<uint32_t>(c->dims[k]);
    za.thr[k] = lemire_threshold32(static_cast<uint64_t>(c->dims[k]));
    za.stride[k] = stride;
    stride *= static_cast<uint64_t>(c->dims[k]);
  }
  if (c->wide) {
    za.wide = 1;
    for (int k = 0; k < c->d; ++k) {
      za.stride[k] = c->stride_lo[k];
      za.stride_hi[k] = c->stride_hi[k];
    }
    za.hkeys_hi = c->hkeys_hi.as<uint64_t>();
  }
  za.seed = seed;
  za.iter = iter;
  za.iter_base = iter_base;
  za.tag = tag;
  za.hkeys = c->nnz > 0 ? c->hkeys.as<uint64_t>() : nullptr;
  za.hmask = c->hmask;
  za.bloom = c->nnz > 0 && !c->tune.no_bloom ? c->bloom.as<uint32_t>() : nullptr;
  za.bmask = c->bmask;
  za.st = st;
  za.status = c->zstatus.as<unsigned long long>();
  za.tbits = c->ztbits.as<uint32_t>();
  za.zero_list = c->zero_list.as<uint64_t>();
  fill_refstream(c, za, seed, p_ref);
  return za;
}

void run_zero_sampler(gcpb_ctx* c, int64_t q, double rho, uint64_t seed, uint64_t iter,
                      const uint64_t* iter_base, uint32_t tag, int mode, int64_t p_ref = 0) {
  if (mode != ZERO_CAPTURE) prepare_zero_sampler(c, q, rho);
  const int64_t nchunks = c->z_nchunks_first;
  DevState* st = c->dst();
  const ZeroArgs za = zero_args(c, seed, iter, iter_base, tag, p_ref);
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(nchunks, c->num_sms * 4)));
  for (int b = 0; b < 3; ++b) {
    CK(launch_k(zero_plan_kernel, dim3(1), dim3(1), 0, c->stream, st, b == 0 ? 1 : 0));
    launch_zero_cand(c, grid, za);
    CK(launch_k(zero_scatter_kernel, dim3(grid), dim3(kZcThreads), 0, c->stream, za));
  }
  CK(cudaGetLastError());
  if (mode == ZERO_CAPTURE) {
    CK(launch_k(zero_check_kernel, dim3(1), dim3(1), 0, c->stream, st));
    CK(cudaGetLastError());
    return;
  }
  if (mode != ZERO_HOST_CHECK) return;
  for (;;) {
    c->pull_state();
    if (c->host_state.z_overflow) throw std::logic_error("zero sampler: status overflow");
    if (std::min(c->host_state.z_accepted, q) >= q) break;
    CK(launch_k(zero_plan_kernel, dim3(1), dim3(1), 0, c->stream, st, 0));
    launch_zero_cand(c, grid, za);
    CK(launch_k(zero_scatter_kernel, dim3(grid), dim3(kZcThreads), 0, c->stream, za));
    CK(cudaGetLastError());
  }
}

// ---- communicator helpers -----------------------------------------------------
bool has_comm(const gcpb_ctx* c) { return c->comm != nullptr || c->host_allgather != nullptr; }

std::vector<int64_t> comm_allgather_i64(gcpb_ctx* c, int64_t v) {
  std::vector<int64_t> out(static_cast<size_t>(c->nranks), 0);
  if (c->nranks == 1) {
    out[0] = v;
    return out;
  }
  if (c->host_allgather) {
    c->sync();
    if (c->host_allgather(c->host_user, v, out.data()) != 0)
      throw std::runtime_error("host allgather callback failed");
    return out;
  }
  if (!c->comm) throw std::logic_error("multi-rank call without a communicator");
  c->comm_buf.alloc(static_cast<size_t>(c->nranks + 1) * sizeof(int64_t));
  int64_t* d = c->comm_buf.as<int64_t>();
  CK(cudaMemcpyAsync(d + c->nranks, &v, 8, cudaMemcpyHostToDevice, c->stream));
  nck(ncclAllGather(d + c->nranks, d, 1, ncclInt64, c->comm, c->stream), "ncclAllGather");
  CK(cudaMemcpyAsync(out.data(), d, c->nranks * 8, cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  return out;
}

template <typename T>
void comm_allreduce_grad(gcpb_ctx* c) {
  if (c->nranks == 1) return;
  if (c->comm) {
    nck(ncclAllReduce(c->Gr.p, c->Gr.p, static_cast<size_t>(c->nelem),
                      sizeof(T) == 4 ? ncclFloat : ncclDouble, ncclSum, c->comm, c->stream),
        "ncclAllReduce");
    return;
  }
  if (!c->host_allreduce) throw std::logic_error("multi-rank call without a communicator");
  std::vector<T> h(static_cast<size_t>(c->nelem));
  CK(cudaMemcpyAsync(h.data(), c->Gr.p, c->nelem * sizeof(T), cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  std::vector<double> hd(h.begin(), h.end());
  if (c->host_allreduce(c->host_user, hd.data(), c->nelem) != 0)
    throw std::runtime_error("host allreduce callback failed");
  for (size_t i = 0; i < h.size(); ++i) h[i] = static_cast<T>(hd[i]);
  CK(cudaMemcpyAsync(c->Gr.p, h.data(), c->nelem * sizeof(T), cudaMemcpyHostToDevice, c->stream));
  c->sync();
}

// Multi-rank stratified zero sampler, device-planned
// (zero_plan_mr_kernel and friends, gcpb_aux.cuh): per batch, plan -> test
// this rank's slice -> all-gather the accept counts -> keep the accepts below
// the global need -> commit.  Three batches per call are queued; inside a
// step graph (ZERO_CAPTURE, NCCL all-gather captured) a shortfall is flagged
// like the single-rank sampler's; eager calls continue on the host until q
// accepts exist.  This rank's kept list is zero_list[0, zg_kept).

// Sizes the multi-rank scratch and uploads the per-call scalars (not inside
// a graph capture).
void prepare_zero_sampler_mr(gcpb_ctx* c, int64_t q, double rho) {
  ensure_hash(c);
  const double zeta = static_cast<double>(c->total128 - static_cast<unsigned __int128>(c->nnz));
  const int64_t first_batch = zero_batch_size_dev(c->total_d, zeta, rho, q);
  const int64_t slice = first_batch / c->nranks + 1;  // batches shrink with the shortfall
  const int64_t nchunks = (slice + kZcChunk - 1) / kZcChunk;
  if (c->zero_cap < q) {
    c->zero_list.alloc(static_cast<size_t>(q) * sizeof(uint64_t));
    c->zero_cap = q;
  }
  if (c->zscratch_cap < slice) {
    c->zscratch.alloc(static_cast<size_t>(slice) * sizeof(uint64_t));
    c->zscratch_cap = slice;
  }
  if (c->zstatus_cap < nchunks) {
    c->zstatus.alloc(static_cast<size_t>(nchunks) * sizeof(unsigned long long));
    c->ztbits.alloc(static_cast<size_t>(nchunks) * kZcThreads * sizeof(uint32_t));
    c->zstatus_cap = nchunks;
  }
  c->mr_counts.alloc(static_cast<size_t>(c->nranks + 1) * sizeof(int64_t));
  c->z_nchunks_first = nchunks;
  DevState* st = c->dst();
  c->host_state.zg_q = q;
  c->host_state.z_total = c->total_d;
  c->host_state.z_zeta = zeta;
  c->host_state.z_rho = rho;
  c->host_state.z_status_cap = c->zstatus_cap;
  CK(cudaMemcpyAsync(&st->zg_q, &c->host_state.zg_q, sizeof(int64_t), cudaMemcpyHostToDevice,
                     c->stream));
  CK(cudaMemcpyAsync(&st->z_total, &c->host_state.z_total, 3 * sizeof(double),
                     cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(&st->z_status_cap, &c->host_state.z_status_cap, sizeof(int64_t),
                     cudaMemcpyHostToDevice, c->stream));
}

// All ranks' z_accepted (this batch's accepts) -> mr_counts[0, nranks).
void allgather_accepts(gcpb_ctx* c) {
  int64_t* counts = c->mr_counts.as<int64_t>();
  if (c->comm) {
    nck(ncclAllGather(&c->dst()->z_accepted, counts, 1, ncclInt64, c->comm, c->stream),
        "ncclAllGather");
    return;
  }
  if (!c->host_allgather) throw std::logic_error("multi-rank call without a communicator");
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(c->stream, &cs));
  if (cs != cudaStreamCaptureStatusNone)
    throw std::logic_error("the host communicator cannot be captured in a step graph");
  int64_t mine = 0;
  CK(cudaMemcpyAsync(&mine, &c->dst()->z_accepted, 8, cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  std::vector<int64_t> all(static_cast<size_t>(c->nranks), 0);
  if (c->host_allgather(c->host_user, mine, all.data()) != 0)
    throw std::runtime_error("host allgather callback failed");
  CK(cudaMemcpyAsync(counts, all.data(), all.size() * 8, cudaMemcpyHostToDevice, c->stream));
  c->sync();
}

void zero_batch_mr(gcpb_ctx* c, const ZeroArgs& za, int grid, bool first) {
  DevState* st = c->dst();
  CK(launch_k(zero_plan_mr_kernel, dim3(1), dim3(1), 0, c->stream, st, first ? 1 : 0, c->rank,
              c->nranks));
  launch_zero_cand(c, grid, za);
  CK(launch_k(zero_scatter_kernel, dim3(grid), dim3(kZcThreads), 0, c->stream, za));
  allgather_accepts(c);
  const int64_t* counts = c->mr_counts.as<int64_t>();
  const int kgrid = static_cast<int>(
      std::max<int64_t>(1, std::min<int64_t>((c->zscratch_cap + 255) / 256, c->num_sms * 2)));
  CK(launch_k(zero_keep_mr_kernel, dim3(kgrid), dim3(256), 0, c->stream,
              static_cast<const DevState*>(st), counts, c->rank,
              static_cast<const uint64_t*>(c->zscratch.as<uint64_t>()), c->zero_list.as<uint64_t>()));
  CK(launch_k(zero_commit_mr_kernel, dim3(1), dim3(1), 0, c->stream, st, counts, c->rank,
              c->nranks));
  CK(cudaGetLastError());
}

void run_zero_sampler_mr(gcpb_ctx* c, int64_t q, double rho, uint64_t seed, uint64_t iter,
                         const uint64_t* iter_base, uint32_t tag, int mode, int64_t p_ref,
                         gcpb_stats* stats) {
  if (mode != ZERO_CAPTURE) prepare_zero_sampler_mr(c, q, rho);
  ZeroArgs za = zero_args(c, seed, iter, iter_base, tag, p_ref);
  za.zero_list = c->zscratch.as<uint64_t>();  // this rank's accepts of one batch
  const int grid = static_cast<int>(
      std::max<int64_t>(1, std::min<int64_t>(c->z_nchunks_first, c->num_sms * 4)));
  for (int b = 0; b < 3; ++b) zero_batch_mr(c, za, grid, b == 0);
  if (mode == ZERO_CAPTURE) {
    CK(launch_k(zero_check_mr_kernel, dim3(1), dim3(1), 0, c->stream, c->dst()));
    CK(cudaGetLastError());
    return;
  }
  for (;;) {
    c->pull_state();
    if (c->host_state.z_overflow) throw std::logic_error("zero sampler: status overflow");
    if (c->host_state.zg_accepted >= q) break;
    zero_batch_mr(c, za, grid, false);
  }
  if (stats) {
    stats->tested = c->host_state.zg_tested;
    stats->accepted = c->host_state.zg_accepted;
    stats->rejected = c->host_state.zg_rejected;
  }
}

uint64_t* pick_list_of(gcpb_ctx* c, int which) {
  return which ? c->pick_list2.as<uint64_t>() : c->pick_list.as<uint64_t>();
}
int64_t* pick_count_of(gcpb_ctx* c, int which) {
  return which ? &c->dst()->pick_n2 : &c->dst()->pick_n;
}

void launch_pick_compact(gcpb_ctx* c, const PickSpec& ps, int which, int bps, cudaStream_t stream) {
  int64_t* cnt = pick_count_of(c, which);
  CK(cudaMemsetAsync(cnt, 0, sizeof(int64_t), stream));
  const int64_t chunks = (ps.p + 256 * kPickItems - 1) / (256 * kPickItems);
  const int grid = static_cast<int>(
      std::max<int64_t>(1, std::min<int64_t>(chunks, static_cast<int64_t>(c->num_sms) * bps)));
  CK(launch_k(pick_compact_kernel, dim3(grid), dim3(256), 0, stream, ps, pick_list_of(c, which),
              cnt));
  CK(cudaGetLastError());
}

// Captured multi-rank steps: the NEXT step's picks are compacted into the other
// list on the side stream while the exchange kernel (NVLink-bound) runs; the
// iteration they belong to is rng_iter + 1, snapshotted first because the
// exchange kernel advances rng_iter.  The next step's pick launch joins.
void pick_compact_ahead(gcpb_ctx* c) {
  CK(launch_k(iter_next_kernel, dim3(1), dim3(32), 0, c->stream, c->dst()));
  CK(cudaEventRecord(c->ev_fork, c->stream));
  CK(cudaStreamWaitEvent(c->side_stream, c->ev_fork, 0));
  PickSpec ps = c->pick_spec;
  ps.iter = 0;
  ps.iter_base = &c->dst()->rng_iter_next;
  launch_pick_compact(c, ps, c->pick_cur ^ 1, 8, c->side_stream);
  CK(cudaEventRecord(c->ev_ahead, c->side_stream));
  c->pick_ahead = true;
}

// Nonzero-sharded ranks: the picks of the global stream that fall in this
// rank's nonzero range, compacted into pick_list[0, pick_n) (pick_compact_kernel).
template <typename T>
void build_pick_list(gcpb_ctx* c, const FusedArgs<T>& a, uint32_t tag, int64_t p, int bps = 8) {
  if (c->pick_cap < p) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(c->stream, &cs));
    if (cs != cudaStreamCaptureStatusNone)
      throw std::logic_error("pick list not reserved before the step-graph capture");
    c->pick_list.alloc(static_cast<size_t>(p) * sizeof(uint64_t));
    c->pick_cap = p;
  }
  PickSpec ps;
  std::memset(&ps, 0, sizeof(ps));
  ps.seed = a.seed;
  ps.iter = a.iter;
  ps.iter_base = a.iter_base;
  ps.tag = tag;
  ps.thr_eta = a.thr_eta;
  ps.p = p;
  ps.eta = a.eta;
  ps.nz_begin = c->nz_begin;
  ps.nz_end = c->nz_end;
  ps.refstream = a.refstream;
  ps.ref_key = a.ref_key;
  ps.thr64_eta = a.thr64_eta;
  ps.ref_ctr = a.ref_ctr;
  ps.ref_flag = a.ref_flag;
  c->pick_spec = ps;
  c->pick_spec_valid = !a.refstream;  // RefStream draws follow a counter the steps advance
  launch_pick_compact(c, ps, c->pick_cur, bps, c->stream);
}

// ---- unrestricted draws walked in memory order (tables beyond L2) ----------
// For factor tables beyond L2 (the interleaved table) the q unrestricted
// draws of semi-stratified sampling (samplers.hpp:211-216) are walked in the
// order of their mode-0 row block instead of ordinal order: ordinals t
// counting-sorted by (mode-0 row >> shift), the row recomputed exactly as
// phase_a draws it, then walked as a SEG_ZERO_LIST segment of the same tag.
// Same draws, same weights; only the gradient's summation order changes.
struct SortSpec {
  uint64_t seed, iter;
  const uint64_t* iter_base;
  uint32_t tag;
  int64_t b0, n;
  uint64_t range;  // n_0
  uint32_t thr;    // Lemire threshold of range (32-bit draws)
  int shift;
  unsigned long long* chk;  // checked builds: failure counters, bins of the sort
  int64_t nbins;
};

__device__ __forceinline__ uint32_t sort_bin(const SortSpec& sp, uint64_t it, uint64_t t) {
  uint64_t key;
  if (sp.range <= (1ull << 32)) {  // phase_a: group 0, word 0, attempt 0 first
    const U4 b = philox_block(sp.seed, sp.tag, 0u, 0u, it, t);
    const uint64_t prod = static_cast<uint64_t>(b.x) * sp.range;
    key = (static_cast<uint32_t>(prod) >= sp.thr)
              ? (prod >> 32)
              : bounded32_from(sp.seed, sp.tag, it, t, 0, sp.range, sp.thr, 1u);
  } else {
    key = bounded64(sp.seed, sp.tag, it, t, 0, sp.range);
  }
  return static_cast<uint32_t>(key >> sp.shift);
}

// Both passes keep kOrdIlp atomics in flight per thread: they are bound by the
// L2 atomic round trip, and next to the fused kernel's pick half they get one
// or two blocks per SM.
#ifndef GCPB_ORD_ILP
#define GCPB_ORD_ILP 8
#endif
constexpr int kOrdIlp = GCPB_ORD_ILP;
__global__ void __launch_bounds__(256, 4) order_count_kernel(SortSpec sp, uint32_t* cnt) {
  const uint64_t it = sp.iter + (sp.iter_base ? *sp.iter_base : 0ull);
  const int64_t nthr = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < sp.n;
       i += nthr * kOrdIlp) {
    uint32_t bin[kOrdIlp];
#pragma unroll
    for (int j = 0; j < kOrdIlp; ++j) {
      const int64_t ij = i + j * nthr;
      bin[j] = ij < sp.n ? sort_bin(sp, it, static_cast<uint64_t>(sp.b0 + ij)) : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int j = 0; j < kOrdIlp; ++j)
      if (bin[j] != 0xFFFFFFFFu) {
        GCPB_CHECK(sp.chk, bin[j] < sp.nbins, 10, bin[j]);
        atomicAdd(cnt + bin[j], 1u);
      }
  }
}

// out[position] = ordinal relative to sp.b0 (32 bits: order_build takes n < 2^32).
__global__ void __launch_bounds__(256, 4) order_scatter_kernel(SortSpec sp, uint32_t* cursor,
                                                            uint32_t* out) {
  const uint64_t it = sp.iter + (sp.iter_base ? *sp.iter_base : 0ull);
  const int64_t nthr = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < sp.n;
       i += nthr * kOrdIlp) {
    uint32_t pos[kOrdIlp];
#pragma unroll
    for (int j = 0; j < kOrdIlp; ++j) {
      const int64_t ij = i + j * nthr;
      pos[j] = 0xFFFFFFFFu;
      if (ij < sp.n)
        pos[j] = atomicAdd(cursor + sort_bin(sp, it, static_cast<uint64_t>(sp.b0 + ij)), 1u);
    }
#pragma unroll
    for (int j = 0; j < kOrdIlp; ++j)
      if (pos[j] != 0xFFFFFFFFu) {
        GCPB_CHECK(sp.chk, pos[j] < sp.n, 11, pos[j]);
        out[pos[j]] = static_cast<uint32_t>(i + j * nthr);
      }
  }
}

// Exclusive scan of the bin counts into the cursors, without any dependency
// between blocks: block b owns bins [b * 1024, (b + 1) * 1024), sums every
// count before them itself (coalesced, L2-resident: <= a few 100k bins) and
// scans its own 1024.  (A one-block scan of C5's 75k bins took 64 us.)
constexpr int kScanThreads = 1024;
__global__ void __launch_bounds__(kScanThreads) order_scan_kernel(const uint32_t* __restrict__ cnt,
                                                                  uint32_t* __restrict__ cur,
                                                                  int64_t n) {
  __shared__ uint32_t wsum[32];
  __shared__ uint32_t wpre[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t start = static_cast<int64_t>(blockIdx.x) * kScanThreads;
  uint32_t before = 0;
  for (int64_t i = threadIdx.x; i < start; i += kScanThreads) before += __ldg(cnt + i);
  const int64_t mine = start + threadIdx.x;
  const uint32_t v = mine < n ? __ldg(cnt + mine) : 0u;
  uint32_t inc = v;  // inclusive warp scan of this block's bins
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) before += __shfl_xor_sync(0xffffffffu, before, o);
  if (lane == 31) wpre[wid] = inc;
  if (lane == 0) wsum[wid] = before;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = wpre[lane];
    uint32_t tot = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += u;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    wpre[lane] = w - wpre[lane] + tot;  // exclusive warp offset + everything before the block
  }
  __syncthreads();
  if (mine < n) cur[mine] = wpre[wid] + inc - v;
}

bool order_wanted(const gcpb_ctx* c) {
  return c->tune.sortq >= 0 ? c->tune.sortq != 0 : c->il_enabled;
}

// Writes the ordered list for sp into ob.out; false when it cannot (scratch
// too small inside a graph capture): the caller walks ordinal order instead.
// Sizes ob for n items in nbins bins; false inside a graph capture when it
// would have to allocate.
bool order_reserve(gcpb_ctx* c, OrderBufs& ob, int64_t n, int64_t nbins) {
  if (n <= ob.out_cap && nbins <= ob.bins_cap) return true;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(c->stream, &cs);
  if (cs != cudaStreamCaptureStatusNone) return false;
  if (n > ob.out_cap) {
    ob.out.alloc(static_cast<size_t>(n) * sizeof(uint32_t));
    ob.out_cap = n;
  }
  if (nbins > ob.bins_cap) {
    ob.cnt.alloc(static_cast<size_t>(2 * nbins) * sizeof(uint32_t));
    ob.bins_cap = nbins;
  }
  return true;
}

int64_t order_bins(const SortSpec& sp) {
  return static_cast<int64_t>((sp.range - 1) >> sp.shift) + 1;
}

bool order_build(gcpb_ctx* c, OrderBufs& ob, const SortSpec& sp, cudaStream_t stream) {
  if (sp.n <= 0 || sp.n >= (int64_t{1} << 32)) return false;
  const int64_t nbins = order_bins(sp);
  if (nbins >= (int64_t{1} << 31)) return false;
  if (!order_reserve(c, ob, sp.n, nbins)) return false;
  uint32_t* cnt = ob.cnt.as<uint32_t>();
  uint32_t* cur = cnt + nbins;
  const int grid = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>((sp.n + 255) / 256, static_cast<int64_t>(c->num_sms) * c->tune.ord_bps)));
  CK(cudaMemsetAsync(cnt, 0, static_cast<size_t>(nbins) * sizeof(uint32_t), stream));
  order_count_kernel<<<grid, 256, 0, stream>>>(sp, cnt);
  CK(cudaGetLastError());
  order_scan_kernel<<<static_cast<unsigned>((nbins + kScanThreads - 1) / kScanThreads), kScanThreads, 0,
                      stream>>>(cnt, cur, nbins);
  CK(cudaGetLastError());
  order_scatter_kernel<<<grid, 256, 0, stream>>>(sp, cur, ob.out.as<uint32_t>());
  CK(cudaGetLastError());
  return true;
}

template <typename T>
SortSpec order_spec(const gcpb_ctx* c, const FusedArgs<T>& a, uint32_t tag, int64_t b0, int64_t b1) {
  SortSpec sp;
  std::memset(&sp, 0, sizeof(sp));
  sp.seed = a.seed;
  sp.iter = a.iter;
  sp.iter_base = a.iter_base;
  sp.tag = tag;
  sp.b0 = b0;
  sp.n = b1 - b0;
  sp.range = a.dims[0];
  sp.thr = a.thr[0];
  sp.shift = c->tune.qshift;  // 32 mode-0 rows per bin by default
  sp.chk = chk_counters();
  sp.nbins = order_bins(sp);
  return sp;
}

struct SampleResult {
  int64_t n = 0;
  gcpb_stats stats{0, 0, 0};
};

// The fused sample -> eval -> MTTKRP (and/or record) for one sampler call.
template <typename T>
SampleResult stoch_grad_impl(gcpb_ctx* c, const gcpb_sampler* sk, const gcpb_loss* loss,
                             uint64_t seed, uint64_t iter, bool scatter, bool record,
                             bool host_check, bool estimator_tags, int est_kind,
                             const uint64_t* iter_base = nullptr, bool fold = false,
                             int zero_mode = -1) {
  SampleResult res;
  FusedArgs<T> a = base_args<T>(c, loss, seed, iter);
  a.iter_base = iter_base;
  if (zero_mode < 0) zero_mode = host_check ? ZERO_HOST_CHECK : ZERO_DEVICE_ONLY;
  a.scatter = scatter ? 1 : 0;
  if (record) {
    a.r_idx = c->s_idx.as<int64_t>();
    a.r_x = c->s_x.as<double>();
    a.r_w = c->s_w.as<double>();
    a.r_flag = c->s_flag.as<int32_t>();
    a.r_m = c->s_m.as<double>();
    a.r_y = c->s_y.as<double>();
  }
  const uint32_t tag_u = estimator_tags ? TAG_EST_UNIFORM : TAG_GRAD_UNIFORM;
  const uint32_t tag_p = estimator_tags ? TAG_EST_NZ_PICK : TAG_GRAD_NZ_PICK;
  const uint32_t tag_z = estimator_tags ? TAG_EST_ZERO_CAND : TAG_GRAD_ZERO_CAND;
  int64_t b0 = 0, b1 = 0;
  if (sk->strategy == GCPB_UNIFORM) {
    const int64_t s = sk->num_samples;
    gcpb_shard_range(s, c->rank, c->nranks, &b0, &b1);
    const double w = c->total_d / static_cast<double>(s);  // samplers.hpp:83
    a.nseg = 1;
    a.seg[0] = make_seg(SEG_UNIFORM, tag_u, b0, b1, w, 0, 0);
    if (c->tensor_kind == 2) {
      ensure_hash(c);
      a.hkeys = c->hkeys.as<uint64_t>();
      a.hkeys_hi = c->hkeys_hi.as<uint64_t>();
      a.hvals = c->hvals.as<uint32_t>();
      a.hmask = c->hmask;
    }
    res.n = s;
    run_fused(c, a, record, fold);
    if (c->draw_stream == 1) {  // sample_uniform consumed s * d draws
      CK(launch_k(ref_advance_kernel, dim3(1), dim3(1), 0, c->stream, c->dst(), static_cast<uint64_t>(s) * c->d, 0, c->d));
      CK(cudaGetLastError());
    }
    return res;
  }
  // stratified / semi-stratified (samplers.hpp:141-219), estimator split
  // (samplers.hpp:283-315) when est_kind >= 0.
  int64_t p = sk->nonzero_samples, q = sk->zero_samples;
  const int64_t eta = c->nnz;
  const unsigned __int128 zeta128 = c->total128 - static_cast<unsigned __int128>(eta);
  if (eta == 0 && p > 0) {
    q += p;
    p = 0;
  }
  if (est_kind >= 0 && zeta128 == 0) {
    p += q;
    q = 0;
  }
  const double eta_over_p = p > 0 ? static_cast<double>(eta) / static_cast<double>(p) : 0.0;
  const bool strat = sk->strategy == GCPB_STRATIFIED;
  bool zero_mr = false;  // multi-rank: this rank's zero list length is on the device
  if (strat && q > 0) {
    if (zeta128 < static_cast<unsigned __int128>(q))
      throw std::invalid_argument("sample_zeros_rejection: requested " + std::to_string(q) +
                                  " zeros but only " + u128_to_string(zeta128) + " exist");
    if (c->nranks > 1) {
      if (record)
        throw std::invalid_argument("multi-rank stratified sampling records no samples");
      if (p > 0 && eta > 0 && c->tune.ord_side != 0 && c->side_stream != nullptr) {
        // as on one rank: the sampler (plan, test, all-gather of the accept counts,
        // keep, commit per batch) runs on the side stream under the pick segment's
        // launch; the communicator is used by one stream at a time (fork after the
        // main stream's last collective, join before its next)
        CK(cudaEventRecord(c->ev_fork, c->stream));
        CK(cudaStreamWaitEvent(c->side_stream, c->ev_fork, 0));
        cudaStream_t main_stream = c->stream;
        c->stream = c->side_stream;
        try {
          run_zero_sampler_mr(c, q, sk->oversample, seed, iter, iter_base, tag_z, zero_mode, p,
                              &res.stats);
        } catch (...) {
          c->stream = main_stream;
          throw;
        }
        c->stream = main_stream;
        CK(cudaEventRecord(c->ev_join, c->side_stream));
        c->join_pending = true;
      } else {
        run_zero_sampler_mr(c, q, sk->oversample, seed, iter, iter_base, tag_z, zero_mode, p,
                            &res.stats);
      }
      zero_mr = true;
    } else if (zero_mode != ZERO_HOST_CHECK && p > 0 && eta > 0 && c->tune.ord_side != 0 &&
               c->side_stream != nullptr) {
      // device-planned batches (no host round trip): the zero sampler runs on
      // the side stream under the pick segment's launch -- it is issue-bound
      // (Philox + hashing), the picks are bound by the L2 reductions -- and
      // run_fused joins before the zero-list segment
      CK(cudaEventRecord(c->ev_fork, c->stream));
      CK(cudaStreamWaitEvent(c->side_stream, c->ev_fork, 0));
      cudaStream_t main_stream = c->stream;
      c->stream = c->side_stream;
      try {
        run_zero_sampler(c, q, sk->oversample, seed, iter, iter_base, tag_z, zero_mode, p);
      } catch (...) {
        c->stream = main_stream;
        throw;
      }
      c->stream = main_stream;
      CK(cudaEventRecord(c->ev_join, c->side_stream));
      c->join_pending = true;
    } else {
      run_zero_sampler(c, q, sk->oversample, seed, iter, iter_base, tag_z, zero_mode, p);
    }
    a.zero_list = c->zero_list.as<uint64_t>();
    a.chk_zl = static_cast<int64_t>(c->zero_list.bytes / sizeof(uint64_t));
  }
  a.nseg = 0;
  const bool ordered = scatter && !record && est_kind < 0 && c->draw_stream == 0 &&
                       order_wanted(c);
  bool pick_on_side = false;
  if (p > 0) {
    gcpb_shard_range(p, c->rank, c->nranks, &b0, &b1);
    // (walking the picks in COO order measured slower on C5 at every bin
    // width: fused 2.84 -> 3.11 ms plus 0.5 ms of ordering)
    const int pflag = (!strat && est_kind < 0) ? 1 : 0;
    if (nz_sharded(c)) {
      // every rank draws the whole global pick stream and keeps its range
      if (record) throw std::invalid_argument("nonzero-sharded ranks record no samples");
      // With an ordered list segment after the picks, the compaction (Philox-bound:
      // N x p draws on N ranks) runs on the side stream under that segment's launch
      // (memory-bound), which run_fused then launches first; the ordering itself
      // stays on the main stream ahead of it.
      pick_on_side = ordered && !strat && q > 0 && c->tune.pick_side != 0 &&
                     c->tune.ord_side != 0 && c->side_stream != nullptr && c->il_enabled &&
                     !c->pick_ahead;
      if (c->pick_ahead) {
        // compacted ahead by the previous step of this capture (pick_compact_ahead):
        // the other list holds this step's picks once the side stream's event passes
        c->pick_ahead = false;
        c->pick_cur ^= 1;
        CK(cudaStreamWaitEvent(c->stream, c->ev_ahead, 0));
        c->pick_spec_valid = !a.refstream;
      } else if (pick_on_side) {
        CK(cudaEventRecord(c->ev_fork, c->stream));
        CK(cudaStreamWaitEvent(c->side_stream, c->ev_fork, 0));
        cudaStream_t main_stream = c->stream;
        c->stream = c->side_stream;
        try {
          // blocks per SM beside the list launch (captured C5 step of a lone rank,
          // tools/lone_rank_probe.py: 3.51 / 3.34 / 4.99 ms at 2 / 4 / 8 ranks with one
          // block per SM, 3.57 / 3.66 / 4.52 ms with three)
          const int side_bps = c->tune.pick_side >= 2 ? c->tune.pick_side : (c->nranks >= 6 ? 3 : 1);
          build_pick_list<T>(c, a, tag_p, p, side_bps);
        } catch (...) {
          c->stream = main_stream;
          throw;
        }
        c->stream = main_stream;
        CK(cudaEventRecord(c->ev_join, c->side_stream));
      } else {
        build_pick_list<T>(c, a, tag_p, p);
      }
      a.pick_list = pick_list_of(c, c->pick_cur);
      Seg sg = make_seg(SEG_PICK, tag_p, 0, p, eta_over_p, pflag, 0);
      sg.len_dev = pick_count_of(c, c->pick_cur);
      a.seg[a.nseg++] = sg;
    } else {
      a.seg[a.nseg++] = make_seg(SEG_PICK, tag_p, b0, b1, eta_over_p, pflag, 0);
    }
  }
  if (q > 0) {
    const double zeta_d = static_cast<double>(zeta128);
    if (strat) {
      Seg sg = make_seg(SEG_ZERO_LIST, tag_z, 0, q, zeta_d / static_cast<double>(q), 0, p, p);
      if (zero_mr) sg.len_dev = &c->dst()->zg_kept;
      a.seg[a.nseg++] = sg;
    } else {
      gcpb_shard_range(q, c->rank, c->nranks, &b0, &b1);
      const double wq = c->total_d / static_cast<double>(q);
      bool built = false;
      if (ordered) {
        // The ordering depends only on (seed, iteration): with a pick segment
        // ahead of it, it runs on the side stream under that segment's launch
        // and run_fused joins before the ordered segment.
        const bool side = c->tune.ord_side != 0 && a.nseg == 1 && c->side_stream != nullptr &&
                          !pick_on_side;
        cudaStream_t os = c->stream;
        if (side) {
          CK(cudaEventRecord(c->ev_fork, c->stream));
          CK(cudaStreamWaitEvent(c->side_stream, c->ev_fork, 0));
          os = c->side_stream;
        }
        built = order_build(c, c->qorder, order_spec(c, a, TAG_GRAD_SEMI_Q, b0, b1), os);
        if (side) {
          CK(cudaEventRecord(c->ev_join, c->side_stream));
          c->join_pending = true;
        }
      }
      if (pick_on_side) {  // the join now guards the pick segment (first), not the list
        c->join_pending = true;
        c->join_where = built ? 1 : 2;  // no ordered list after all: join ahead of one launch
      }
      if (built) {
        a.zero_list32 = c->qorder.out.as<uint32_t>();  // the same draws, in mode-0 row order
        a.zl_base = static_cast<uint64_t>(b0);
        a.chk_zl = c->qorder.out_cap;
        a.seg[a.nseg++] = make_seg(SEG_ZERO_LIST, TAG_GRAD_SEMI_Q, 0, b1 - b0, wq, 0, p, p);
      } else {
        a.seg[a.nseg++] = make_seg(SEG_DRAW_ZERO, TAG_GRAD_SEMI_Q, b0, b1, wq, 0, p, p);
      }
    }
  }
  res.n = p + q;
  run_fused(c, a, record, fold);
  if (c->draw_stream == 1) {  // p picks, then d draws per tested candidate / q draw
    if (strat && q > 0 && zero_mr)
      CK(launch_k(ref_advance_kernel, dim3(1), dim3(1), 0, c->stream, c->dst(),
                  static_cast<uint64_t>(p), 2, c->d));
    else if (strat && q > 0)
      CK(launch_k(ref_advance_kernel, dim3(1), dim3(1), 0, c->stream, c->dst(), static_cast<uint64_t>(p), 1, c->d));
    else
      CK(launch_k(ref_advance_kernel, dim3(1), dim3(1), 0, c->stream, c->dst(), static_cast<uint64_t>(p + q * c->d), 0,
                                                 c->d));
    CK(cudaGetLastError());
  }
  if (strat && q > 0 && zero_mode == ZERO_HOST_CHECK && c->nranks == 1) {
    res.stats.tested = c->host_state.z_tested;
    res.stats.accepted = c->host_state.z_accepted;
    res.stats.rejected = c->host_state.z_rejected;
  }
  return res;
}

void alloc_record(gcpb_ctx* c, int64_t n) {
  const size_t nn = static_cast<size_t>(std::max<int64_t>(n, 1));
  c->s_idx.alloc(nn * c->d * sizeof(int64_t));
  c->s_x.alloc(nn * sizeof(double));
  c->s_w.alloc(nn * sizeof(double));
  c->s_flag.alloc(nn * sizeof(int32_t));
  c->s_m.alloc(nn * sizeof(double));
  c->s_y.alloc(nn * sizeof(double));
}

int64_t expected_samples(const gcpb_ctx* c, const gcpb_sampler* s) {
  if (s->strategy == GCPB_UNIFORM) return s->num_samples;
  return s->nonzero_samples + s->zero_samples;
  (void)c;
}

// fold_reps > 0: the gradient is the sum of that many replicas (read and
// re-zeroed by the kernel).  advance_rng: also step the device draw-stream base.
template <typename T>
void adam_launch(gcpb_ctx* c, int fold_reps = 0, int advance_rng = 0, int hot_rh = 0) {
  HotAdam<T> hot;
  std::memset(&hot, 0, sizeof(hot));
  if (hot_rh > 0) {  // hot rows' copies folded by extra blocks
    hot.hslot = c->hslot.as<uint8_t>();
    hot.Ghot = c->Ghot.as<T>();
    hot.hot_off = c->hot_off.as<int64_t>();
    hot.rh = hot_rh;
    hot.n = c->hot_n;
    hot.d = c->d;
    for (int k = 0; k < c->d; ++k) {
      hot.rowbase[k] = c->row_base[k];
      hot.off[k] = c->off[k];
    }
  }
  // replica fold: lanes per chunk so that each sums at most four replicas
  // (C2 Adam 10 -> 7.3 us); with hot rows the fold blocks of the hot copies
  // are the long pole and the wider grid measured slower (C3 11.5 -> 22 us)
  int lp = 1;
  while (hot.n == 0 && lp < 8 && 4 * lp < fold_reps) lp <<= 1;
  const int64_t cpr = c->rp / c->vw;  // chunks per row
  int cpr_shift = 0;
  while ((int64_t{1} << cpr_shift) < cpr) ++cpr_shift;
  const bool il_now = c->il_pending || c->il_gpack;
  if (fold_reps == 0 && c->tune.adam > 0 && (int64_t{1} << cpr_shift) == cpr &&
      c->nelem >= (int64_t{1} << 20)) {
    // streaming Adam for tables in HBM (adam_stream_kernel)
    ILTab<T> il{};
    if (il_now) {
      il.ag = c->AG.as<T>();
      il.rp = static_cast<int>(c->rp);
      il.gcontig = c->il_gpack ? 1 : 0;
    } else {
      a_current(c);
    }
    const bool nopad = c->r == c->rp;
    const int v = c->tune.adam;
    const int per_sm = v == 2 ? 4 : 2;
    const int grid = grid_for(c->nelem / c->vw, 256, c->num_sms, per_sm) + hot.n;
    auto go = [&](auto kern) {
      CK(launch_k(kern, dim3(grid), dim3(256), 0, c->stream, c->A.as<T>(), c->Gr.as<T>(),
                  c->B.as<T>(), c->C.as<T>(), c->nelem, static_cast<int>(c->rp), cpr_shift,
                  static_cast<int>(c->r), c->dst(), advance_rng, hot, il));
    };
    constexpr bool F32 = sizeof(T) == 4;
#define GCPB_ADAM_GO(ILV)                                                                      \
    if (v == 3 || !F32) {                                                                      \
      nopad ? go(adam_stream_kernel<T, ILV, false, true, 4, 2>)                                \
            : go(adam_stream_kernel<T, ILV, false, false, 4, 2>);                              \
    } else if (v == 2) {                                                                       \
      nopad ? go(adam_stream_kernel<T, ILV, F32, true, 2, 4>)                                  \
            : go(adam_stream_kernel<T, ILV, F32, false, 2, 4>);                                \
    } else {                                                                                   \
      nopad ? go(adam_stream_kernel<T, ILV, F32, true, 4, 2>)                                  \
            : go(adam_stream_kernel<T, ILV, F32, false, 4, 2>);                                \
    }
    if (il_now) {
      GCPB_ADAM_GO(true)
      c->il_pending = false;
      c->il_gpack = false;
      c->a_stale = true;
    } else {
      GCPB_ADAM_GO(false)
      c->ag_ok = false;
    }
#undef GCPB_ADAM_GO
    CK(cudaGetLastError());
    return;
  }
  const int grid = grid_for(c->nelem / c->vw * lp, 256, c->num_sms, 8) + hot.n;
  if (il_now) {  // factors (and unless packed, the gradient) in AG
    ILTab<T> il;
    il.ag = c->AG.as<T>();
    il.rp = static_cast<int>(c->rp);
    il.gcontig = c->il_gpack ? 1 : 0;
    CK(launch_k(adam_kernel<T, true>, dim3(grid), dim3(256), 0, c->stream, c->A.as<T>(),
                c->Gr.as<T>(), c->B.as<T>(), c->C.as<T>(), c->nelem, static_cast<int>(c->rp),
                static_cast<int>(c->r), c->dst(), c->Grep.as<T>(), fold_reps, c->rep_stride,
                advance_rng, hot, il, lp));
    c->il_pending = false;
    c->il_gpack = false;
    c->a_stale = true;
  } else {
    a_current(c);
    CK(launch_k(adam_kernel<T, false>, dim3(grid), dim3(256), 0, c->stream, c->A.as<T>(),
                c->Gr.as<T>(), c->B.as<T>(), c->C.as<T>(), c->nelem, static_cast<int>(c->rp),
                static_cast<int>(c->r), c->dst(), c->Grep.as<T>(), fold_reps, c->rep_stride,
                advance_rng, hot, ILTab<T>{}, lp));
    c->ag_ok = false;  // A changed without AG
  }
  CK(cudaGetLastError());
}

template <typename T>
void estimate_launch(gcpb_ctx* c, const gcpb_loss* loss) {
  a_current(c);
  ModelDesc<T> md;
  std::memset(&md, 0, sizeof(md));
  md.A = c->A.as<T>();
  md.d = c->d;
  md.rp = static_cast<int>(c->rp);
  md.r = static_cast<int>(c->r);
  for (int k = 0; k < c->d; ++k) md.off[k] = c->off[k];
  constexpr int kGrid = 296;  // fixed => bit-deterministic summation order
  c->est_partials.alloc(kGrid * sizeof(double));
  c->est_out.alloc(sizeof(double));
  estimate_partial_kernel<T><<<kGrid, 256, 0, c->stream>>>(
      md, c->est_idx.as<int64_t>(), c->est_x.as<double>(), c->est_w.as<double>(), c->est_n,
      loss->kind, loss->delta, c->est_partials.as<double>());
  sum_partials_kernel<<<1, 32, 0, c->stream>>>(c->est_partials.as<double>(), kGrid,
                                                c->est_out.as<double>());
  CK(cudaGetLastError());
}

int record_words(int d, size_t tsize) {
  const int need = static_cast<int>(tsize / 4) + d;
  int w = 4;
  while (w < need) w <<= 1;
  return w;
}

// Sorted unique keys + f64 values already on the device -> records.
void set_sparse_normalized_device(gcpb_ctx* c, const uint64_t* d_keys, const double* d_vals,
                                  int64_t n) {
  c->nnz = n;
  c->tensor_kind = 2;
  c->tensor_version += 1;
  c->hash_ready = false;
  c->domain_flags = -1;
  c->dense.reset();
  c->rec_words = record_words(c->d, c->tsize);
  const size_t nn = static_cast<size_t>(std::max<int64_t>(n, 1));
  c->keys.alloc(nn * sizeof(uint64_t));
  c->nzrec.alloc(nn * c->rec_words * sizeof(uint32_t));
  c->vals.alloc(nn * c->tsize);
  if (n > 0) {
    CK(cudaMemcpyAsync(c->keys.p, d_keys, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice,
                       c->stream));
    const int g = grid_for(n, 256, c->num_sms);
    if (c->dtype == GCPB_F32)
      keys_to_records_kernel<double, float><<<g, 256, 0, c->stream>>>(
          c->keys.as<uint64_t>(), d_vals, n, c->d, c->dims_dev.as<int64_t>(),
          c->nzrec.as<uint32_t>(), c->rec_words, c->vals.as<float>());
    else
      keys_to_records_kernel<double, double><<<g, 256, 0, c->stream>>>(
          c->keys.as<uint64_t>(), d_vals, n, c->d, c->dims_dev.as<int64_t>(),
          c->nzrec.as<uint32_t>(), c->rec_words, c->vals.as<double>());
    CK(cudaGetLastError());
  }
  c->sync();
  c->nz_begin = 0;
  c->nz_end = n;
  apply_nz_shard(c);
}

void set_sparse_normalized(gcpb_ctx* c, const std::vector<uint64_t>& keys,
                           const std::vector<double>& values) {
  const int64_t n = static_cast<int64_t>(keys.size());
  c->nnz = n;
  c->tensor_kind = 2;
  c->tensor_version += 1;
  c->hash_ready = false;
  c->domain_flags = -1;
  c->dense.reset();
  c->rec_words = record_words(c->d, c->tsize);
  const size_t nn = static_cast<size_t>(std::max<int64_t>(n, 1));
  c->keys.alloc(nn * sizeof(uint64_t));
  c->nzrec.alloc(nn * c->rec_words * sizeof(uint32_t));
  c->vals.alloc(nn * c->tsize);
  if (n > 0) {
    DBuf dv;
    dv.alloc(n * sizeof(double));
    CK(cudaMemcpyAsync(c->keys.p, keys.data(), n * sizeof(uint64_t), cudaMemcpyHostToDevice,
                       c->stream));
    CK(cudaMemcpyAsync(dv.p, values.data(), n * sizeof(double), cudaMemcpyHostToDevice,
                       c->stream));
    const int g = grid_for(n, 256, c->num_sms);
    if (c->dtype == GCPB_F32)
      keys_to_records_kernel<double, float><<<g, 256, 0, c->stream>>>(
          c->keys.as<uint64_t>(), dv.as<double>(), n, c->d, c->dims_dev.as<int64_t>(),
          c->nzrec.as<uint32_t>(), c->rec_words, c->vals.as<float>());
    else
      keys_to_records_kernel<double, double><<<g, 256, 0, c->stream>>>(
          c->keys.as<uint64_t>(), dv.as<double>(), n, c->d, c->dims_dev.as<int64_t>(),
          c->nzrec.as<uint32_t>(), c->rec_words, c->vals.as<double>());
    CK(cudaGetLastError());
    c->sync();
  }
  c->sync();
  c->nz_begin = 0;
  c->nz_end = n;
  apply_nz_shard(c);
}

template <typename T>
void given_launch(gcpb_ctx* c, int64_t n, const gcpb_loss* loss, bool y_given, bool record,
                  bool scatter) {
  FusedArgs<T> a = base_args<T>(c, loss, 0, 0);
  a.scatter = scatter ? 1 : 0;
  a.g_idx = c->s_idx.as<int64_t>();
  if (y_given) {
    a.g_y = c->s_y.as<double>();
  } else {
    a.g_x = c->s_x.as<double>();
    a.g_w = c->s_w.as<double>();
    a.g_flag = c->s_flag.as<int32_t>();
  }
  if (record) {
    a.r_m = c->s_m.as<double>();
    a.r_y = c->s_aux.as<double>();
  }
  a.nseg = 1;
  a.seg[0] = make_seg(SEG_GIVEN, 0, 0, n, 0.0, 0, 0);
  run_fused(c, a, record);
}

// Uploads the Adam scalars (FitConfig fields + learning rate) through the
// context's pinned block when they changed; no host synchronisation.
void set_adam_params(gcpb_ctx* ctx, const gcpb_adam* adam) {
  if (!adam) throw std::invalid_argument("adam: null");
  DevState* st = ctx->dst();
  DevState& h = ctx->host_state;
  const int32_t has = adam->has_lower_bound ? 1 : 0;
  const bool changed = !ctx->adam_params_valid || h.lr != adam->learning_rate ||
                       h.beta1 != adam->beta1 || h.beta2 != adam->beta2 ||
                       h.eps != adam->epsilon || h.lb != adam->lower_bound || h.has_lb != has;
  if (!changed) return;
  h.lr = adam->learning_rate;
  h.beta1 = adam->beta1;
  h.beta2 = adam->beta2;
  h.eps = adam->epsilon;
  h.lb = adam->lower_bound;
  h.has_lb = has;
  double* pin = ctx->pinned_params;
  CK(cudaStreamSynchronize(ctx->stream));  // the pinned block may still be in flight
  pin[0] = h.lr;
  pin[1] = h.beta1;
  pin[2] = h.beta2;
  pin[3] = h.eps;
  pin[4] = h.lb;
  std::memcpy(&pin[5], &has, sizeof(has));
  CK(cudaMemcpyAsync(&st->lr, pin, 5 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(&st->has_lb, &pin[5], sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
  ctx->adam_params_valid = true;
}

void check_step_args(gcpb_ctx* ctx, const gcpb_sampler* sampler, const gcpb_loss* loss) {
  validate_sampler(sampler);
  validate_loss(loss);
  if (ctx->tensor_kind == 0) throw std::invalid_argument("no tensor set");
  if (sampler->strategy != GCPB_UNIFORM && ctx->tensor_kind != 2)
    throw std::invalid_argument(sampler->strategy == GCPB_STRATIFIED
                                    ? "stratified sampling requires a sparse tensor"
                                    : "semi-stratified sampling requires a sparse tensor");
  check_data_domain(ctx, loss->kind);
}

// Barrier over the ranks: every rank's queued work completes before any
// rank's later work starts (NCCL: a one-element all-reduce in stream order,
// capturable; host communicator: synchronise + an all-gather callback).
void rank_barrier(gcpb_ctx* c) {
  if (c->nranks == 1 || c->tune.lone_rank) return;
  if (c->comm) {
    c->barrier_buf.alloc(sizeof(int64_t));
    nck(ncclAllReduce(c->barrier_buf.p, c->barrier_buf.p, 1, ncclInt64, ncclSum, c->comm,
                      c->stream),
        "ncclAllReduce(barrier)");
    return;
  }
  if (!c->host_allgather) throw std::logic_error("multi-rank call without a communicator");
  c->sync();
  std::vector<int64_t> sink(static_cast<size_t>(c->nranks));
  if (c->host_allgather(c->host_user, 0, sink.data()) != 0)
    throw std::runtime_error("host allgather callback failed");
}

template <typename T>
void peer_adam_launch(gcpb_ctx* c, int advance_rng) {
  PeerTabs<T> pt;
  std::memset(&pt, 0, sizeof(pt));
  for (int p = 0; p < c->nranks; ++p) {
    pt.a[p] = static_cast<T*>(c->peer_a[static_cast<size_t>(p)]);
    pt.g[p] = static_cast<T*>(c->peer_g[static_cast<size_t>(p)]);
  }
  pt.npeers = c->nranks;
  pt.self = c->rank;
  const bool il = c->il_enabled;
  pt.pitch = static_cast<int>(il ? 2 * c->rp : c->rp);
  int cpr_shift = 0;
  while ((int64_t{1} << cpr_shift) < c->rp / c->vw) ++cpr_shift;
  const int64_t rows = c->nelem / c->rp;
  int64_t row0 = 0, row1 = 0;
  gcpb_shard_range(rows, c->rank, c->nranks, &row0, &row1);
  const int grid = grid_for(std::max<int64_t>(1, (row1 - row0) << cpr_shift), 256, c->num_sms, 4);
  constexpr bool FAST = sizeof(T) == 4;
  CK(launch_k(peer_adam_kernel<T, FAST>, dim3(grid), dim3(256), 0, c->stream, pt, c->B.as<T>(),
              c->C.as<T>(), row0, row1, static_cast<int>(c->rp), cpr_shift,
              static_cast<int>(c->r), c->dst(), advance_rng));
  CK(cudaGetLastError());
  c->moments_sharded = true;
  if (il) {
    c->a_stale = true;  // the factors live in the tables (AG)
    c->il_pending = false;
    c->il_gpack = false;
  } else {
    c->ag_ok = false;
  }
}

// One iteration: fused sample->MTTKRP, all-reduce when sharded, fused Adam
// (which folds the replica reduction when not sharded).
template <typename T>
void step_impl(gcpb_ctx* c, const gcpb_sampler* sk, const gcpb_loss* loss, uint64_t seed,
               uint64_t iter, const uint64_t* iter_base, int zero_mode) {
  const bool multi = c->nranks > 1;
  try {
    c->in_step = true;
    stoch_grad_impl<T>(c, sk, loss, seed, iter, true, false, zero_mode == ZERO_HOST_CHECK, false,
                       -1, iter_base, /*fold=*/!multi, zero_mode);
    c->in_step = false;
    int fold = 0;
    if (multi) {
      if (!has_comm(c) && !c->tune.lone_rank)
        throw std::logic_error("sharded step without a communicator");
      if (c->peer_ok) {  // reduce-scatter + sharded Adam + all-gather, one kernel
        if (iter_base && c->steps_left > 0 && c->tune.pick_ahead != 0 && c->pick_spec_valid &&
            nz_sharded(c) && c->side_stream != nullptr && c->pick_list2.p)
          pick_compact_ahead(c);
        c->pick_spec_valid = false;
        rank_barrier(c);
        peer_adam_launch<T>(c, iter_base ? 1 : 0);
        rank_barrier(c);
        c->in_step = false;
        c->hot_pending = 0;
        c->grad_zero = true;
        return;
      }
      comm_allreduce_grad<T>(c);
    } else if (c->nrep > 1) {
      fold = c->nrep;
    }
    adam_launch<T>(c, fold, iter_base ? 1 : 0, c->hot_pending);
  } catch (...) {
    c->in_step = false;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(c->stream, &cs);
    if ((c->il_pending || c->il_gpack) && cs == cudaStreamCaptureStatusNone) {
      // AG's gradient rows (or Gr) may hold a partial gradient: keep AG's
      // factor rows (A refreshed from them), rebuild AG on the next
      // interleaved step, re-zero Gr on the next use
      c->il_pending = false;
      c->il_gpack = false;
      a_current(c);
      c->ag_ok = false;
      c->grad_zero = false;
    }
    c->il_pending = false;
    c->il_gpack = false;
    throw;
  }
  c->hot_pending = 0;
  c->grad_zero = true;
}

void set_rng_iter(gcpb_ctx* c, uint64_t iter0) {
  CK(cudaStreamSynchronize(c->stream));
  std::memcpy(&c->pinned_params[8], &iter0, 8);
  CK(cudaMemcpyAsync(&c->dst()->rng_iter, &c->pinned_params[8], 8, cudaMemcpyHostToDevice,
                     c->stream));
}

std::string steps_key(const gcpb_ctx* c, const gcpb_sampler* sk, const gcpb_loss* loss,
                      uint64_t seed, int64_t n) {
  char buf[512];
  std::snprintf(buf, sizeof(buf), "%d|%lld|%lld|%lld|%.17g|%d|%.17g|%llu|%lld|%lld|%d|%d|%d",
                sk->strategy, static_cast<long long>(sk->num_samples),
                static_cast<long long>(sk->nonzero_samples),
                static_cast<long long>(sk->zero_samples), sk->oversample, loss->kind, loss->delta,
                static_cast<unsigned long long>(seed), static_cast<long long>(n),
                static_cast<long long>(c->tensor_version), c->rank, c->nranks,
                c->hash_ready ? 1 : 0);
  return std::string(buf) + (c->draw_stream ? "|ref" : "|philox") + "|g" +
         std::to_string(g_dbuf_gen.load(std::memory_order_relaxed));
}

// Small problems (model L2-resident, few samples, uniform draws, one rank,
// Philox): all n iterations in one cluster launch (gcpb_small.cuh).
// GCPB_NO_SMALL=1 forces the graph path.
constexpr size_t kSmallModelMax = 200 * 1024;  // A, B, C replicas in shared memory

template <typename T>
bool small_eligible(const gcpb_ctx* c, const gcpb_sampler* sk) {
  if (c->tune.no_small || c->wide || c->nranks != 1 || c->draw_stream != 0 || c->timing) return false;
  // red.global issue costs ~1.3 cycles per lane on the issuing SM: keep the
  // per-iteration scatter of the 8 cluster SMs well under a microsecond
  if (sk->strategy != GCPB_UNIFORM || sk->num_samples * c->d * c->r > 16384) return false;
  if (c->d > 8 || (c->tensor_kind == 2 && !c->hash_ready)) return false;
  for (int k = 0; k < c->d; ++k)
    if (static_cast<uint64_t>(c->dims[k]) > 0xffffffffull) return false;
  return 3 * static_cast<size_t>(c->nelem) * sizeof(T) <= kSmallModelMax;
}

template <typename T, int DM>
void small_launch_dm(const SmallArgs<T>& a, T* G, cudaStream_t stream) {
  const size_t smem = 3 * static_cast<size_t>(a.nelem) * sizeof(T);
  static const cudaError_t attr_set = cudaFuncSetAttribute(  // once per instantiation
      small_steps_kernel<T, DM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
      static_cast<int>(kSmallModelMax));
  CK(attr_set);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kSmallCluster, 1, 1);
  cfg.blockDim = dim3(kSmallThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kSmallCluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, small_steps_kernel<T, DM>, a, G));
}

template <typename T>
void small_launch(gcpb_ctx* c, const gcpb_sampler* sk, const gcpb_loss* loss, uint64_t seed,
                  int64_t n, const double* host_in = nullptr, double* host_out = nullptr,
                  const uint64_t* iter = nullptr) {
  a_current(c);
  c->ag_ok = false;  // the cluster kernel writes A
  const FusedArgs<T> f = base_args<T>(c, loss, seed, 0);
  SmallArgs<T> a;
  std::memset(&a, 0, sizeof(a));
  a.A = c->A.as<T>();
  a.B = c->B.as<T>();
  a.C = c->C.as<T>();
  a.nelem = c->nelem;
  a.d = c->d;
  a.r = static_cast<int>(c->r);
  a.rp = static_cast<int>(c->rp);
  for (int k = 0; k < c->d; ++k) {
    a.off[k] = f.off[k];
    a.dims[k] = f.dims[k];
    a.thr[k] = f.thr[k];
    a.stride[k] = f.stride[k];
  }
  a.xkind = f.xkind;
  a.dense = f.dense;
  a.hkeys = f.hkeys;
  a.hvals = f.hvals;
  a.hmask = f.hmask;
  a.vals = f.vals;
  a.loss = f.loss;
  a.delta = f.delta;
  a.s = sk->num_samples;
  a.w = c->total_d / static_cast<double>(sk->num_samples);  // samplers.hpp:83
  a.seed = seed;
  a.tag = TAG_GRAD_UNIFORM;
  a.n_steps = n;
  a.st = c->dst();
  a.host_in = host_in;
  a.host_out = host_out;
  a.iter_given = iter ? 1 : 0;
  a.iter = iter ? *iter : 0;
  c->small_g.alloc(3 * static_cast<size_t>(c->nelem) * sizeof(T));
  if (!c->small_g_zero) {
    CK(cudaMemsetAsync(c->small_g.p, 0, 3 * static_cast<size_t>(c->nelem) * sizeof(T), c->stream));
    c->small_g_zero = true;  // the kernel leaves all three buffers zero
  }
  T* G = c->small_g.as<T>();
  switch (c->d) {
    case 1: small_launch_dm<T, 1>(a, G, c->stream); break;
    case 2: small_launch_dm<T, 2>(a, G, c->stream); break;
    case 3: small_launch_dm<T, 3>(a, G, c->stream); break;
    case 4: small_launch_dm<T, 4>(a, G, c->stream); break;
    case 5: small_launch_dm<T, 5>(a, G, c->stream); break;
    case 6: small_launch_dm<T, 6>(a, G, c->stream); break;
    case 7: small_launch_dm<T, 7>(a, G, c->stream); break;
    default: small_launch_dm<T, 8>(a, G, c->stream); break;
  }
  CK(cudaGetLastError());
}

template <typename T>
void run_steps_impl(gcpb_ctx* c, const gcpb_sampler* sk, const gcpb_loss* loss, uint64_t seed,
                    uint64_t iter0, int64_t n, const gcpb_adam* adam) {
  set_adam_params(c, adam);
  ensure_grad_zero(c);
  if (c->nranks > 1 && !c->comm && !c->tune.lone_rank) {
    // the host communicator cannot be captured in a graph: step eagerly
    for (int64_t k = 0; k < n; ++k)
      step_impl<T>(c, sk, loss, seed, iter0 + static_cast<uint64_t>(k), nullptr, ZERO_HOST_CHECK);
    c->last_steps_path = 0;
    c->graph_kernels = 0;
    return;
  }
  if (nz_sharded(c) && sk->strategy != GCPB_UNIFORM && sk->nonzero_samples > 0 &&
      c->pick_cap < sk->nonzero_samples) {  // pick list, before the capture
    c->pick_list.alloc(static_cast<size_t>(sk->nonzero_samples) * sizeof(uint64_t));
    c->pick_cap = sk->nonzero_samples;
  }
  if (nz_sharded(c) && sk->strategy != GCPB_UNIFORM && sk->nonzero_samples > 0 &&
      c->tune.pick_ahead != 0 && c->peer_ok)  // the next step's picks, compacted ahead
    c->pick_list2.alloc(static_cast<size_t>(c->pick_cap) * sizeof(uint64_t));
  c->pick_ahead = false;
  if (sk->strategy == GCPB_STRATIFIED) {
    int64_t q = sk->zero_samples + (c->nnz == 0 ? sk->nonzero_samples : 0);
    if (q > 0) {
      const unsigned __int128 zeta = c->total128 - static_cast<unsigned __int128>(c->nnz);
      if (zeta < static_cast<unsigned __int128>(q))
        throw std::invalid_argument("sample_zeros_rejection: requested " + std::to_string(q) +
                                    " zeros but only " + u128_to_string(zeta) + " exist");
      if (c->nranks > 1)
        prepare_zero_sampler_mr(c, q, sk->oversample);
      else
        prepare_zero_sampler(c, q, sk->oversample);
    }
  } else if (sk->strategy == GCPB_UNIFORM && c->tensor_kind == 2) {
    ensure_hash(c);
  }
  if (c->tensor_kind == 2) ensure_hot(c);  // host work: not inside the capture
  if (sk->strategy == GCPB_SEMI_STRATIFIED && sk->zero_samples > 0 && c->draw_stream == 0 &&
      order_wanted(c)) {  // ordering scratch for the unrestricted draws, before the capture
    int64_t b0 = 0, b1 = 0;
    gcpb_shard_range(sk->zero_samples, c->rank, c->nranks, &b0, &b1);
    FusedArgs<T> fa = base_args<T>(c, nullptr, seed, iter0);
    const SortSpec sp = order_spec(c, fa, TAG_GRAD_SEMI_Q, b0, b1);
    if (sp.n > 0) order_reserve(c, c->qorder, sp.n, order_bins(sp));
  }
  set_rng_iter(c, iter0);
  if (small_eligible<T>(c, sk)) {
    small_launch<T>(c, sk, loss, seed, n);
    c->grad_zero = true;
    c->last_steps_path = 1;
    return;
  }
  c->last_steps_path = 0;
  const bool il = c->il_enabled;
  if (il)
    ag_prepare<T>(c);  // not inside the capture
  else
    a_current(c);
  const std::string key = steps_key(c, sk, loss, seed, n);
  if (!c->graph_exec || key != c->graph_key) {
    if (c->graph_exec) {
      cudaGraphExecDestroy(c->graph_exec);
      c->graph_exec = nullptr;
    }
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    try {
      for (int64_t k = 0; k < n; ++k) {
        c->steps_left = n - 1 - k;
        step_impl<T>(c, sk, loss, seed, 0, &c->dst()->rng_iter, ZERO_CAPTURE);
      }
      c->steps_left = 0;
    } catch (...) {
      c->steps_left = 0;
      c->pick_ahead = false;
      cudaStreamEndCapture(c->stream, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    CK(cudaStreamEndCapture(c->stream, &g));
    size_t nn = 0;
    CK(cudaGraphGetNodes(g, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    if (nn) CK(cudaGraphGetNodes(g, nodes.data(), &nn));
    c->graph_kernels = 0;
    for (cudaGraphNode_t nd : nodes) {
      cudaGraphNodeType ty;
      CK(cudaGraphNodeGetType(nd, &ty));
      if (ty == cudaGraphNodeTypeKernel) ++c->graph_kernels;
    }
    cudaGraphExec_t ex = nullptr;
    const cudaError_t e = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    ck(e, "cudaGraphInstantiate");
    c->graph_exec = ex;
    c->graph_key = key;
  }
  CK(cudaGraphLaunch(c->graph_exec, c->stream));
  c->grad_zero = true;
  if (il) {  // a cached graph's interleaved Adam updates leave A stale on every replay
    c->a_stale = true;
    c->il_last = true;
  }
}

// Synchronise and surface deferred device-side failures (graph-mode
// stratified shortfalls).
void sync_and_check(gcpb_ctx* c) {
  // both flags come back with the one synchronisation the caller needs
  uint32_t* flags = reinterpret_cast<uint32_t*>(&c->pinned_params[12]);
  CK(cudaMemcpyAsync(&flags[0], &c->dst()->ref_flag, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(&flags[1], &c->dst()->z_incomplete, 4, cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  const uint32_t rf = flags[0];
  const int32_t inc = static_cast<int32_t>(flags[1]);
  if (c->draw_stream == 1) {
    if (rf)
      throw std::runtime_error("RefStream: a draw fell in RngStream::next_below's rejection "
                               "region (p <= n/2^64); the reference would have redrawn");
  }
  if (inc != 0) {
    const int32_t zero = 0;
    CK(cudaMemcpyAsync(&c->dst()->z_incomplete, &zero, 4, cudaMemcpyHostToDevice, c->stream));
    c->sync();
    throw std::runtime_error("stratified zero sampler: " + std::to_string(inc) +
                             " graph-replayed iteration(s) found fewer than q zeros in the three "
                             "device-planned batches; use gcpb_step for this problem");
  }
}

double model_norm_host(const std::vector<std::vector<double>>& F, int64_t r) {
  // KruskalModel::norm (kruskal.cpp:75-83): 1' (hadamard_k A_k' A_k) 1.
  std::vector<double> gram(static_cast<size_t>(r * r), 1.0);
  for (const auto& f : F) {
    const int64_t n = static_cast<int64_t>(f.size()) / r;
    for (int64_t a = 0; a < r; ++a)
      for (int64_t b = 0; b < r; ++b) {
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) s += f[i * r + a] * f[i * r + b];
        gram[a * r + b] *= s;
      }
  }
  double ss = 0.0;
  for (double v : gram) ss += v;
  return std::sqrt(std::max(0.0, ss));
}

// ---- exact gradients and bias/variance ------------------------------------------
template <typename T>
void gradient_full_impl(gcpb_ctx* c, const gcpb_loss* loss) {
  if (c->tensor_kind == 0) throw std::invalid_argument("no tensor set");
  if (!c->total_fits || c->total > 100000000ull)  // kernels.cpp:176-179
    throw std::invalid_argument("gradient: tensor too large for the full-entry walk: " +
                                u128_to_string(c->total128) + " entries");
  check_data_domain(c, loss->kind);
  if (c->tensor_kind == 2) ensure_hash(c);
  FusedArgs<T> a = base_args<T>(c, loss, 0, 0);
  a.refstream = 0;
  if (c->tensor_kind == 2) {
    a.hkeys = c->hkeys.as<uint64_t>();
    a.hvals = c->hvals.as<uint32_t>();
    a.hmask = c->hmask;
  }
  a.nseg = 1;
  a.seg[0] = make_seg(SEG_FULL, 0, 0, static_cast<int64_t>(c->total), 1.0, 0, 0);
  CK(cudaMemsetAsync(c->Gr.p, 0, c->nelem * c->tsize, c->stream));
  run_fused(c, a, false);
  c->grad_zero = false;
}

template <typename T>
void poisson_implicit_impl(gcpb_ctx* c, const gcpb_loss* loss) {
  a_current(c);
  if (loss->kind != GCPB_LOSS_POISSON)
    throw std::invalid_argument(std::string("implicit gradient requires the poisson loss, got ") +
                                loss_name(loss->kind));  // kernels.cpp:202-205
  if (c->tensor_kind != 2) throw std::invalid_argument("implicit gradient requires a sparse tensor");
  check_data_domain(c, loss->kind);
  const int d = c->d, r = static_cast<int>(c->r);
  // sparse part first (it overwrites G when gradient replicas are in use)
  FusedArgs<T> a = base_args<T>(c, loss, 0, 0);
  a.refstream = 0;
  a.nseg = 1;
  a.seg[0] = make_seg(SEG_NZ_ALL, 0, 0, c->nnz, 1.0, 2, 0);
  CK(cudaMemsetAsync(c->Gr.p, 0, c->nelem * c->tsize, c->stream));
  if (c->nnz > 0) run_fused(c, a, false);
  // all-ones part: rows += prod of the other factors' column sums (LeaveOneOut order)
  DBuf cs, offd, rowc;
  cs.alloc(static_cast<size_t>(d) * r * sizeof(double));
  offd.alloc(kMaxModes * sizeof(int64_t));
  CK(cudaMemcpyAsync(offd.p, c->off, kMaxModes * sizeof(int64_t), cudaMemcpyHostToDevice,
                     c->stream));
  colsum_kernel<T><<<d * r, 256, 0, c->stream>>>(c->A.as<T>(), offd.as<int64_t>(),
                                                 c->dims_dev.as<int64_t>(),
                                                 static_cast<int>(c->rp), r, cs.as<double>());
  std::vector<double> h(static_cast<size_t>(d) * r);
  CK(cudaMemcpyAsync(h.data(), cs.p, h.size() * 8, cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  std::vector<double> pre(static_cast<size_t>(d) * r), suf(static_cast<size_t>(d) * r),
      out(static_cast<size_t>(d) * r);
  for (int j = 0; j < r; ++j) pre[j] = 1.0;
  for (int k = 1; k < d; ++k)
    for (int j = 0; j < r; ++j) pre[k * r + j] = pre[(k - 1) * r + j] * h[(k - 1) * r + j];
  for (int j = 0; j < r; ++j) suf[(d - 1) * r + j] = 1.0;
  for (int k = d - 2; k >= 0; --k)
    for (int j = 0; j < r; ++j) suf[k * r + j] = suf[(k + 1) * r + j] * h[(k + 1) * r + j];
  for (size_t i = 0; i < out.size(); ++i) out[i] = pre[i] * suf[i];
  rowc.alloc(out.size() * 8);
  CK(cudaMemcpyAsync(rowc.p, out.data(), out.size() * 8, cudaMemcpyHostToDevice, c->stream));
  add_rowconst_kernel<T><<<grid_for(c->nelem, 256, c->num_sms), 256, 0, c->stream>>>(
      c->Gr.as<T>(), rowc.as<double>(), c->nelem, static_cast<int>(c->rp), r, offd.as<int64_t>(),
      d);
  CK(cudaGetLastError());
  c->sync();
  c->grad_zero = false;
}

// Per-element running moments (Welford, fp64) of `trials` stochastic
// gradients: trial t = Philox iteration t, or in RefStream mode the stream
// split(t) of the key `seed` from counter 0 (samplers.cpp:140-141).
template <typename T>
void trial_moments(gcpb_ctx* c, const gcpb_sampler* sk, const gcpb_loss* loss, int64_t trials,
                   uint64_t seed, DBuf& mean, DBuf& m2) {
  const int64_t n = c->nelem;
  mean.alloc(n * 8);
  m2.alloc(n * 8);
  CK(cudaMemsetAsync(mean.p, 0, n * 8, c->stream));
  CK(cudaMemsetAsync(m2.p, 0, n * 8, c->stream));
  const HostRngStream parent = HostRngStream::from_key(seed);
  for (int64_t t = 0; t < trials; ++t) {
    uint64_t key = seed, it = static_cast<uint64_t>(t);
    if (c->draw_stream == 1) {
      key = parent.split(static_cast<uint64_t>(t)).key();
      const uint64_t zero = 0;
      CK(cudaMemcpyAsync(&c->dst()->ref_ctr, &zero, 8, cudaMemcpyHostToDevice, c->stream));
      it = 0;
    }
    ensure_grad_zero(c);
    stoch_grad_impl<T>(c, sk, loss, key, it, true, false, true, false, -1);
    c->grad_zero = false;
    welford_kernel<T><<<grid_for(n, 256, c->num_sms), 256, 0, c->stream>>>(
        c->Gr.as<T>(), mean.as<double>(), m2.as<double>(), n, static_cast<double>(t + 1));
    CK(cudaGetLastError());
  }
}

// Padded device fp64 -> unpadded host (GradientSet order), optional scale.
void padded_to_host(gcpb_ctx* c, const DBuf& src, double* out, double scale) {
  std::vector<double> h(static_cast<size_t>(c->nelem));
  CK(cudaMemcpyAsync(h.data(), src.p, h.size() * 8, cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  for (int k = 0; k < c->d; ++k)
    for (int64_t i = 0; i < c->dims[k]; ++i)
      for (int64_t j = 0; j < c->r; ++j) *out++ = h[c->off[k] + i * c->rp + j] * scale;
}

template <typename T>
void gradient_moments_impl(gcpb_ctx* c, const gcpb_sampler* sk, const gcpb_loss* loss,
                           int64_t trials, uint64_t seed, double* mean_out, double* var_out) {
  if (trials < 2) throw std::invalid_argument("gradient moments: need >= 2 trials");
  DBuf mean, m2;
  trial_moments<T>(c, sk, loss, trials, seed, mean, m2);
  if (mean_out) padded_to_host(c, mean, mean_out, 1.0);
  if (var_out) padded_to_host(c, m2, var_out, 1.0 / static_cast<double>(trials - 1));
}

template <typename T>
void bias_variance_impl(gcpb_ctx* c, const gcpb_sampler* sk, const gcpb_loss* loss,
                        int64_t trials, uint64_t seed, const double* exact, double* bias,
                        double* variance) {
  if (trials < 2) throw std::invalid_argument("empirical_bias_variance: need >= 2 trials");
  const int64_t n = c->nelem;
  DBuf E, mean, m2, parts;
  E.alloc(n * 8);
  mean.alloc(n * 8);
  m2.alloc(n * 8);
  if (exact) {  // unpadded GradientSet order -> padded layout
    std::vector<double> h(static_cast<size_t>(n), 0.0);
    const double* src = exact;
    for (int k = 0; k < c->d; ++k)
      for (int64_t i = 0; i < c->dims[k]; ++i)
        for (int64_t j = 0; j < c->r; ++j) h[c->off[k] + i * c->rp + j] = *src++;
    CK(cudaMemcpyAsync(E.p, h.data(), n * 8, cudaMemcpyHostToDevice, c->stream));
    c->sync();
  } else {
    gradient_full_impl<T>(c, loss);
    to_double_kernel<T><<<grid_for(n, 256, c->num_sms), 256, 0, c->stream>>>(c->Gr.as<T>(),
                                                                              E.as<double>(), n);
  }
  trial_moments<T>(c, sk, loss, trials, seed, mean, m2);
  constexpr int kGrid = 296;
  parts.alloc(2 * kGrid * 8);
  sqdiff_sum_kernel<<<kGrid, 256, 0, c->stream>>>(mean.as<double>(), E.as<double>(),
                                                  m2.as<double>(), n, parts.as<double>());
  std::vector<double> hp(2 * kGrid);
  CK(cudaMemcpyAsync(hp.data(), parts.p, hp.size() * 8, cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  double sb = 0.0, sv = 0.0;
  for (int b = 0; b < kGrid; ++b) {
    sb += hp[2 * b];
    sv += hp[2 * b + 1];
  }
  *bias = std::sqrt(sb);
  *variance = sv / static_cast<double>(trials);
}

#include "gcpb_gen_host.inc"

// SparseTensor(shape, indices, values) on the device (tensor.cpp:10-41): keys
// + index check, stable radix sort of (key, value), left-to-right run sums,
// zero sums dropped, then the usual records.  Same result as a host stable
// sort; the reference's std::sort can order duplicates differently, which
// only matters in the last bit of sums of three or more duplicates.
// SparseTensor normalisation with 128-bit keys (N >= 2^64; tensor.cpp:10-53
// with Index128 keys, shape.cpp:87-96): keys, sort, sum duplicates, drop
// zeros on the host; keys (low / high words), values and records to the
// device.
void normalize_wide(gcpb_ctx* c, int64_t nnz, const int64_t* coords, const double* values) {
  const int d = c->d;
  std::vector<unsigned __int128> key(static_cast<size_t>(nnz));
  for (int64_t e = 0; e < nnz; ++e) {
    check_index_host(c, coords + e * d);  // tensor.cpp:21 (out_of_range)
    unsigned __int128 l = 0;
    for (int k = 0; k < d; ++k)
      l += static_cast<unsigned __int128>(coords[e * d + k]) *
           ((static_cast<unsigned __int128>(c->stride_hi[k]) << 64) | c->stride_lo[k]);
    key[static_cast<size_t>(e)] = l;
  }
  std::vector<int64_t> ord(static_cast<size_t>(nnz));
  std::iota(ord.begin(), ord.end(), int64_t{0});
  std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return key[a] < key[b]; });
  std::vector<uint64_t> lo, hi;
  std::vector<double> v;
  for (size_t i = 0; i < ord.size();) {
    const unsigned __int128 k = key[static_cast<size_t>(ord[i])];
    double sum = 0.0;
    for (; i < ord.size() && key[static_cast<size_t>(ord[i])] == k; ++i) sum += values[ord[i]];
    if (sum != 0.0) {  // exact zeros dropped (tensor.cpp:35)
      lo.push_back(static_cast<uint64_t>(k));
      hi.push_back(static_cast<uint64_t>(k >> 64));
      v.push_back(sum);
    }
  }
  const int64_t n = static_cast<int64_t>(lo.size());
  c->nnz = n;
  c->tensor_kind = 2;
  c->tensor_version += 1;
  c->hash_ready = false;
  c->domain_flags = -1;
  c->dense.reset();
  c->rec_words = record_words(d, c->tsize);
  const size_t nn = static_cast<size_t>(std::max<int64_t>(n, 1));
  c->keys.alloc(nn * 8);
  c->keys_hi.alloc(nn * 8);
  c->nzrec.alloc(nn * c->rec_words * sizeof(uint32_t));
  c->vals.alloc(nn * c->tsize);
  if (n > 0) {
    DBuf dv;
    dv.alloc(n * 8);
    CK(cudaMemcpyAsync(c->keys.p, lo.data(), n * 8, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->keys_hi.p, hi.data(), n * 8, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(dv.p, v.data(), n * 8, cudaMemcpyHostToDevice, c->stream));
    const int g = grid_for(n, 256, c->num_sms);
    if (c->dtype == GCPB_F32)
      keys_to_records_kernel<double, float><<<g, 256, 0, c->stream>>>(
          c->keys.as<uint64_t>(), dv.as<double>(), n, d, c->dims_dev.as<int64_t>(),
          c->nzrec.as<uint32_t>(), c->rec_words, c->vals.as<float>(), c->keys_hi.as<uint64_t>());
    else
      keys_to_records_kernel<double, double><<<g, 256, 0, c->stream>>>(
          c->keys.as<uint64_t>(), dv.as<double>(), n, d, c->dims_dev.as<int64_t>(),
          c->nzrec.as<uint32_t>(), c->rec_words, c->vals.as<double>(), c->keys_hi.as<uint64_t>());
    CK(cudaGetLastError());
    c->sync();
  }
  c->nz_begin = 0;
  c->nz_end = n;
  apply_nz_shard(c);
}

void normalize_on_device(gcpb_ctx* c, int64_t nnz, const int64_t* coords, const double* values) {
  const int d = c->d;
  if (nnz == 0) {
    std::vector<uint64_t> k;
    std::vector<double> v;
    set_sparse_normalized(c, k, v);
    return;
  }
  DBuf keys_in, keys_out, vals_in, vals_out, sums, keep, stage, bad, tmp, nsel;
  keys_in.alloc(nnz * 8);
  keys_out.alloc(nnz * 8);
  vals_in.alloc(nnz * 8);
  vals_out.alloc(nnz * 8);
  bad.alloc(8);
  CK(cudaMemsetAsync(bad.p, 0xff, 8, c->stream));
  CK(cudaMemcpyAsync(vals_in.p, values, nnz * 8, cudaMemcpyHostToDevice, c->stream));
  const int64_t chunk = std::min<int64_t>(nnz, std::max<int64_t>(1, (int64_t{256} << 20) / (8 * d)));
  stage.alloc(chunk * d * 8);
  for (int64_t b = 0; b < nnz; b += chunk) {
    const int64_t m = std::min(chunk, nnz - b);
    CK(cudaMemcpyAsync(stage.p, coords + b * d, m * d * 8, cudaMemcpyHostToDevice, c->stream));
    coords_to_keys_kernel<<<grid_for(m, 256, c->num_sms, 16), 256, 0, c->stream>>>(
        stage.as<int64_t>(), m, d, c->dims_dev.as<int64_t>(), b, keys_in.as<uint64_t>() + b,
        bad.as<unsigned long long>());
    CK(cudaGetLastError());
    c->sync();  // the staging buffer is reused
  }
  unsigned long long first_bad = 0;
  CK(cudaMemcpyAsync(&first_bad, bad.p, 8, cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  if (first_bad != ~0ull) {
    check_index_host(c, coords + static_cast<int64_t>(first_bad) * d);  // throws (tensor.cpp:21)
    throw std::out_of_range("sparse tensor: index out of range");
  }
  int end_bit = 1;
  while (end_bit < 64 && (c->total - 1) >> end_bit) ++end_bit;
  cub_call(tmp, [&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortPairs(t, b, keys_in.as<uint64_t>(), keys_out.as<uint64_t>(),
                                           vals_in.as<double>(), vals_out.as<double>(), nnz, 0,
                                           end_bit, c->stream);
  });
  sums.alloc(nnz * 8);
  keep.alloc(nnz);
  run_sum_kernel<<<grid_for(nnz, 256, c->num_sms, 16), 256, 0, c->stream>>>(
      keys_out.as<uint64_t>(), vals_out.as<double>(), nnz, sums.as<double>(), keep.as<uint8_t>());
  CK(cudaGetLastError());
  nsel.alloc(8);
  int64_t n_unique = 0;
  cub_call(tmp, [&](void* t, size_t& b) {
    return cub::DeviceSelect::Flagged(t, b, keys_out.as<uint64_t>(), keep.as<uint8_t>(),
                                      keys_in.as<uint64_t>(), nsel.as<int64_t>(), nnz, c->stream);
  });
  cub_call(tmp, [&](void* t, size_t& b) {
    return cub::DeviceSelect::Flagged(t, b, sums.as<double>(), keep.as<uint8_t>(),
                                      vals_in.as<double>(), nsel.as<int64_t>(), nnz, c->stream);
  });
  CK(cudaMemcpyAsync(&n_unique, nsel.p, 8, cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  set_sparse_normalized_device(c, keys_in.as<uint64_t>(), vals_in.as<double>(), n_unique);
}


}  // namespace

namespace gcpb {
// Shared with gcpb_io.cpp: context-free calls report through gcpb_last_error(NULL).
void set_global_error(const std::string& msg) { g_global_err = msg; }
}  // namespace gcpb

// ===========================================================================
// C-ABI
// ===========================================================================
// ---- peer-mapped tables (NVLink / NVSwitch peer memory) ---------------------
namespace {
struct PeerBlob {  // gcpb_peer_handle's export: one rank's table, mappable anywhere
  uint32_t magic;
  int32_t pid, device, il, dtype, rp, pitch, pad;
  int64_t nelem;
  cudaIpcMemHandle_t ha, hg;  // allocations holding the factor / gradient rows
  uint64_t raw_a, raw_g;      // row bases (same-process peers use them as is)
  uint64_t base_a, base_g;    // allocation bases (row base = base + offset)
};
constexpr uint32_t kPeerMagic = 0x47435042u;  // "GCPB"
static_assert(sizeof(PeerBlob) <= GCPB_PEER_HANDLE_BYTES, "peer blob size");

template <typename T>
void peer_tables(gcpb_ctx* c, void** a, void** g, int* pitch) {
  if (c->il_enabled) {  // the interleaved table: factor rows at +0, gradient rows at +rp
    ag_prepare<T>(c);
    *a = c->AG.p;
    *g = c->AG.as<T>() + c->rp;
    *pitch = static_cast<int>(2 * c->rp);
  } else {
    a_current(c);
    *a = c->A.p;
    *g = c->Gr.p;
    *pitch = static_cast<int>(c->rp);
  }
}
}  // namespace

extern "C" {

const char* gcpb_version(void) { return "gcpb 0.1 (sm_100a)"; }

const char* gcpb_last_error(const gcpb_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_global_err.c_str();
}

int gcpb_create(int device, int dtype, int ndims, const int64_t* dims, int64_t rank,
                gcpb_ctx** out) {
  return guard(nullptr, [&] {
    if (!out) throw std::invalid_argument("gcpb_create: null output");
    *out = nullptr;
    if (dtype != GCPB_F32 && dtype != GCPB_F64) throw std::invalid_argument("dtype must be F32 or F64");
    if (ndims < 1) throw std::invalid_argument("Shape: need at least one mode");
    if (ndims > kMaxModes) throw std::invalid_argument("Shape: at most 16 modes supported");
    if (rank < 1) throw std::invalid_argument("kruskal model: rank must be >= 1");
    auto c = std::make_unique<gcpb_ctx>();
    c->device = device;
    c->dtype = dtype;
    c->tsize = dtype == GCPB_F32 ? 4 : 8;
    c->vw = dtype == GCPB_F32 ? 4 : 2;
    c->d = ndims;
    c->r = rank;
    const int64_t pad = dtype == GCPB_F32 ? 8 : 4;  // 32-byte rows
    c->rp = (rank + pad - 1) / pad * pad;
    if (c->rp / c->vw > 32 * 8) throw std::invalid_argument("rank too large for the device path (r <= 1024 fp32 / 512 fp64)");
    unsigned __int128 total = 1;
    const unsigned __int128 maxv = ~static_cast<unsigned __int128>(0);
    for (int k = 0; k < ndims; ++k) {
      if (dims[k] < 1) throw std::invalid_argument("Shape: every extent must be positive");
      if (dims[k] >= (int64_t{1} << 31))
        throw std::invalid_argument("device path supports extents < 2^31");
      if (total > maxv / static_cast<unsigned __int128>(dims[k]))
        throw std::invalid_argument("Shape: total entry count overflows 128 bits");
      total *= static_cast<unsigned __int128>(dims[k]);
      c->dims[k] = dims[k];
    }
    c->total128 = total;
    c->total_fits = total <= static_cast<unsigned __int128>(UINT64_MAX);
    c->wide = !c->total_fits;
    if (total >> 127)  // keys stay below 2^127 (the wide hash's empty marker)
      throw std::invalid_argument("device path supports N < 2^127 entries");
    {
      unsigned __int128 st = 1;
      for (int k = 0; k < ndims; ++k) {
        c->stride_lo[k] = static_cast<uint64_t>(st);
        c->stride_hi[k] = static_cast<uint64_t>(st >> 64);
        st *= static_cast<unsigned __int128>(dims[k]);
      }
    }
    c->total = c->total_fits ? static_cast<uint64_t>(total) : 0;
    c->total_d = static_cast<double>(total);
    int64_t o = 0;
    for (int k = 0; k < ndims; ++k) {
      c->off[k] = o;
      o += c->dims[k] * c->rp;
    }
    c->off[ndims] = o;
    c->nelem = o;
    // beyond 2^31 padded elements (2^32 in the interleaved table) the fused
    // kernel needs 64-bit row offsets: its OFF64 instantiations (d = 3, 4;
    // rows of at most 32 chunks)
    c->off64 = o >= (int64_t{1} << 31);
    CK(cudaSetDevice(device));
    CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    CK(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
    c->stream = c->own_stream;
    {
      int lo = 0, hi = 0;  // the ordering's few blocks go ahead of the fused kernel's
      CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      CK(cudaStreamCreateWithPriority(&c->side_stream, cudaStreamNonBlocking, hi));
      CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->ev_ahead, cudaEventDisableTiming));
    }
    const size_t bytes = static_cast<size_t>(c->nelem) * c->tsize;
    DBuf* bufs[4] = {&c->A, &c->Gr, &c->B, &c->C};
    for (DBuf* b : bufs) {
      b->alloc(bytes);
      CK(cudaMemsetAsync(b->p, 0, bytes, c->stream));
    }
    c->grad_zero = true;
    c->tune.read_env();
    // Interleaved factor/gradient rows when the tables exceed L2 (GCPB_IL=0/1 forces)
    c->il_enabled = c->tune.il >= 0 ? c->tune.il != 0 : bytes > (size_t{64} << 20);
    // Privatized gradient replicas: the scatter of a small gradient (e.g. C2's
    // 51 KB) otherwise funnels every red.global into a few hundred L2 sectors,
    // where the L2 atomic units serialise per address.  Up to 32 replicas are
    // allocated when they fit in 16 MB of L2; each call uses as many as its
    // contention warrants (replicas_for()).
    {
      const int64_t rs = (c->nelem + 63) / 64 * 64;
      int64_t cap = static_cast<int64_t>(16) * 1024 * 1024 / std::max<int64_t>(1, rs * c->tsize);
      cap = std::min<int64_t>(cap, 32);
      if (c->tune.replicas > 0) cap = c->tune.replicas;
      if (cap >= 2) {
        c->nrep_cap = static_cast<int>(cap);
        c->rep_stride = rs;
        c->Grep.alloc(static_cast<size_t>(rs) * cap * c->tsize);
        CK(cudaMemsetAsync(c->Grep.p, 0, static_cast<size_t>(rs) * cap * c->tsize, c->stream));
      }
    }
    c->dstate.alloc(sizeof(DevState));
    CK(cudaMallocHost(reinterpret_cast<void**>(&c->pinned_params), 16 * sizeof(double)));
    std::memset(&c->host_state, 0, sizeof(DevState));
    c->host_state.lr = 1e-3;
    c->host_state.beta1 = 0.9;
    c->host_state.beta2 = 0.999;
    c->host_state.eps = 1e-8;
    c->push_state();
    c->dims_dev.alloc(kMaxModes * sizeof(int64_t));
    CK(cudaMemcpyAsync(c->dims_dev.p, c->dims, kMaxModes * sizeof(int64_t), cudaMemcpyHostToDevice,
                       c->stream));
    c->sync();
    *out = c.release();
  });
}

void gcpb_destroy(gcpb_ctx* ctx) { delete ctx; }

int gcpb_set_stream(gcpb_ctx* ctx, void* stream) {
  return guard(ctx, [&] {
    ctx->sync();
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
  });
}

void* gcpb_get_stream(gcpb_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

// ---- tensor data -------------------------------------------------------------------
int gcpb_set_sparse(gcpb_ctx* ctx, int64_t nnz, const int64_t* coords, const double* values) {
  return guard(ctx, [&] {
    NvtxRange nvtx_("gcpb_set_sparse");
    if (nnz < 0) throw std::invalid_argument("sparse tensor: negative nnz");
    if (nnz > 0 && (!coords || !values)) throw std::invalid_argument("sparse tensor: null buffers");
    if (ctx->wide)
      normalize_wide(ctx, nnz, coords, values);
    else
      normalize_on_device(ctx, nnz, coords, values);
  });
}

int gcpb_set_sparse_device(gcpb_ctx* ctx, int64_t nnz, const uint64_t* d_keys_sorted,
                           const void* d_values, int value_dtype) {
  return guard(ctx, [&] {
    if (nnz < 0) throw std::invalid_argument("sparse tensor: negative nnz");
    if (!ctx->total_fits)
      throw std::invalid_argument("device ingest takes u64 keys: N >= 2^64 needs gcpb_set_sparse");
    if (value_dtype != GCPB_F32 && value_dtype != GCPB_F64)
      throw std::invalid_argument("value dtype must be F32 or F64");
    // the caller's buffers may still be written by work on other streams
    // (e.g. a generator on torch's stream): wait for the device first
    CK(cudaDeviceSynchronize());
    ctx->nnz = nnz;
    ctx->tensor_kind = 2;
    ctx->tensor_version += 1;
    ctx->hash_ready = false;
    ctx->domain_flags = -1;
    ctx->dense.reset();
    const size_t nn = static_cast<size_t>(std::max<int64_t>(nnz, 1));
    ctx->rec_words = record_words(ctx->d, ctx->tsize);
    ctx->keys.alloc(nn * sizeof(uint64_t));
    ctx->nzrec.alloc(nn * ctx->rec_words * sizeof(uint32_t));
    ctx->vals.alloc(nn * ctx->tsize);
    if (nnz > 0) {
      CK(cudaMemcpyAsync(ctx->keys.p, d_keys_sorted, nnz * sizeof(uint64_t),
                         cudaMemcpyDeviceToDevice, ctx->stream));
      ctx->s_aux.alloc(16);
      CK(cudaMemsetAsync(ctx->s_aux.p, 0, 4, ctx->stream));
      const int g = grid_for(nnz, 256, ctx->num_sms);
      if (value_dtype == GCPB_F32)
        check_keys_kernel<float><<<g, 256, 0, ctx->stream>>>(
            ctx->keys.as<uint64_t>(), static_cast<const float*>(d_values), nnz, ctx->total,
            ctx->s_aux.as<unsigned>());
      else
        check_keys_kernel<double><<<g, 256, 0, ctx->stream>>>(
            ctx->keys.as<uint64_t>(), static_cast<const double*>(d_values), nnz, ctx->total,
            ctx->s_aux.as<unsigned>());
      unsigned flags = 0;
      CK(cudaMemcpyAsync(&flags, ctx->s_aux.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
      if (flags & 1u) throw std::out_of_range("sparse tensor: linear key out of range");
      if (flags & 2u) throw std::invalid_argument("device ingest requires strictly increasing keys");
      if (flags & 4u) throw std::invalid_argument("device ingest requires nonzero values");
      const int64_t* dd = ctx->dims_dev.as<int64_t>();
      uint32_t* rec = ctx->nzrec.as<uint32_t>();
      const uint64_t* kk = ctx->keys.as<uint64_t>();
      if (ctx->dtype == GCPB_F32) {
        if (value_dtype == GCPB_F32)
          keys_to_records_kernel<float, float><<<g, 256, 0, ctx->stream>>>(
              kk, static_cast<const float*>(d_values), nnz, ctx->d, dd, rec, ctx->rec_words,
              ctx->vals.as<float>());
        else
          keys_to_records_kernel<double, float><<<g, 256, 0, ctx->stream>>>(
              kk, static_cast<const double*>(d_values), nnz, ctx->d, dd, rec, ctx->rec_words,
              ctx->vals.as<float>());
      } else {
        if (value_dtype == GCPB_F32)
          keys_to_records_kernel<float, double><<<g, 256, 0, ctx->stream>>>(
              kk, static_cast<const float*>(d_values), nnz, ctx->d, dd, rec, ctx->rec_words,
              ctx->vals.as<double>());
        else
          keys_to_records_kernel<double, double><<<g, 256, 0, ctx->stream>>>(
              kk, static_cast<const double*>(d_values), nnz, ctx->d, dd, rec, ctx->rec_words,
              ctx->vals.as<double>());
      }
      CK(cudaGetLastError());
    }
    ctx->sync();
    ctx->nz_begin = 0;
    ctx->nz_end = nnz;
    apply_nz_shard(ctx);
  });
}

int64_t gcpb_nnz(const gcpb_ctx* ctx) { return ctx ? ctx->nnz : 0; }

int gcpb_get_sparse(gcpb_ctx* ctx, int64_t* coords_out, double* values_out) {
  return guard(ctx, [&] {
    if (ctx->tensor_kind != 2) throw std::invalid_argument("no sparse tensor set");
    const int64_t n = ctx->nnz;
    std::vector<uint64_t> keys(static_cast<size_t>(n)), keys_hi(static_cast<size_t>(n), 0);
    if (n > 0)
      CK(cudaMemcpyAsync(keys.data(), ctx->keys.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    if (n > 0 && ctx->wide)
      CK(cudaMemcpyAsync(keys_hi.data(), ctx->keys_hi.p, n * 8, cudaMemcpyDeviceToHost,
                         ctx->stream));
    std::vector<double> v(static_cast<size_t>(n));
    if (ctx->dtype == GCPB_F32) {
      std::vector<float> f(static_cast<size_t>(n));
      if (n > 0)
        CK(cudaMemcpyAsync(f.data(), ctx->vals.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
      for (int64_t e = 0; e < n; ++e) v[e] = f[e];
    } else {
      if (n > 0)
        CK(cudaMemcpyAsync(v.data(), ctx->vals.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
    }
    ctx->sync();
    for (int64_t e = 0; e < n; ++e) {
      unsigned __int128 rem = (static_cast<unsigned __int128>(keys_hi[e]) << 64) | keys[e];
      for (int k = 0; k < ctx->d; ++k) {
        const unsigned __int128 nk = static_cast<unsigned __int128>(ctx->dims[k]);
        coords_out[e * ctx->d + k] = static_cast<int64_t>(rem % nk);
        rem /= nk;
      }
      values_out[e] = v[e];
    }
  });
}

int gcpb_set_dense(gcpb_ctx* ctx, const double* values, int storage) {
  return guard(ctx, [&] {
    NvtxRange nvtx_("gcpb_set_dense");
    if (!ctx->total_fits || ctx->total > (uint64_t{1} << 40))
      throw std::invalid_argument("dense tensor too large to materialize");
    const uint64_t n = ctx->total;
    const size_t bytes = dense_bytes(storage, n);
    std::vector<unsigned char> host(bytes, 0);
    for (uint64_t i = 0; i < n; ++i) {
      const double v = values[i];
      switch (storage) {
        case GCPB_STORE_U8:
          if (!(v >= 0.0 && v <= 255.0 && v == std::floor(v)))
            throw std::invalid_argument("U8 dense storage needs integers in [0, 255]");
          host[i] = static_cast<unsigned char>(v);
          break;
        case GCPB_STORE_BIT:
          if (v != 0.0 && v != 1.0) throw std::invalid_argument("BIT dense storage needs 0/1 data");
          if (v == 1.0) host[i >> 3] |= static_cast<unsigned char>(1u << (i & 7));
          break;
        case GCPB_STORE_F32: {
          const float f = static_cast<float>(v);
          std::memcpy(&host[i * 4], &f, 4);
          break;
        }
        default:
          std::memcpy(&host[i * 8], &v, 8);
      }
    }
    ctx->dense.alloc(bytes);
    CK(cudaMemcpyAsync(ctx->dense.p, host.data(), bytes, cudaMemcpyHostToDevice, ctx->stream));
    ctx->sync();
    ctx->dense_storage = storage;
    ctx->tensor_kind = 1;
    ctx->tensor_version += 1;
    ctx->nnz = 0;
    ctx->domain_flags = -1;
  });
}

int gcpb_set_dense_device(gcpb_ctx* ctx, const void* d_values, int storage) {
  return guard(ctx, [&] {
    if (!ctx->total_fits) throw std::invalid_argument("dense tensor too large to materialize");
    const size_t bytes = dense_bytes(storage, ctx->total);
    ctx->dense.alloc(bytes);
    CK(cudaDeviceSynchronize());  // the source may be written on another stream
    CK(cudaMemcpyAsync(ctx->dense.p, d_values, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    ctx->sync();
    ctx->dense_storage = storage;
    ctx->tensor_kind = 1;
    ctx->tensor_version += 1;
    ctx->nnz = 0;
    ctx->domain_flags = -1;
  });
}

int gcpb_generate_dense_bernoulli(gcpb_ctx* ctx, int64_t true_rank, const double* true_factors,
                                  uint64_t seed, int storage) {
  return guard(ctx, [&] {
    if (!ctx->total_fits) throw std::invalid_argument("dense tensor too large to materialize");
    if (true_rank < 1 || true_rank > 1024) throw std::invalid_argument("true rank out of range");
    if (storage != GCPB_STORE_U8 && storage != GCPB_STORE_BIT)
      throw std::invalid_argument("binary generator stores U8 or BIT");
    int64_t foff[kMaxModes] = {};
    int64_t tot = 0;
    for (int k = 0; k < ctx->d; ++k) {
      foff[k] = tot;
      tot += ctx->dims[k] * true_rank;
    }
    DBuf F, fo;
    F.alloc(tot * sizeof(double));
    fo.alloc(kMaxModes * sizeof(int64_t));
    CK(cudaMemcpyAsync(F.p, true_factors, tot * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(fo.p, foff, sizeof(foff), cudaMemcpyHostToDevice, ctx->stream));
    ctx->dense.alloc(dense_bytes(storage, ctx->total));
    if (storage == GCPB_STORE_U8) {
      const int64_t nfibers = static_cast<int64_t>(ctx->total / static_cast<uint64_t>(ctx->dims[0]));
      const size_t smem = 8 * true_rank * sizeof(double);
      gen_bernoulli_kernel<<<grid_for(nfibers * 32, 256, ctx->num_sms, 8), 256, smem,
                             ctx->stream>>>(ctx->dense.as<uint8_t>(), ctx->d,
                                            ctx->dims_dev.as<int64_t>(), fo.as<int64_t>(),
                                            static_cast<int>(true_rank), F.as<double>(), seed,
                                            nfibers);
    } else {
      const int64_t nwords = static_cast<int64_t>((ctx->total + 31) / 32);
      gen_bernoulli_bits_kernel<<<grid_for(nwords, 256, ctx->num_sms, 16), 256, 0, ctx->stream>>>(
          ctx->dense.as<uint32_t>(), ctx->d, ctx->dims_dev.as<int64_t>(), fo.as<int64_t>(),
          static_cast<int>(true_rank), F.as<double>(), seed, ctx->total);
    }
    CK(cudaGetLastError());
    ctx->sync();
    ctx->dense_storage = storage;
    ctx->tensor_kind = 1;
    ctx->tensor_version += 1;
    ctx->nnz = 0;
    ctx->domain_flags = -1;
  });
}

int gcpb_tensor_norm(gcpb_ctx* ctx, double* out) {
  return guard(ctx, [&] {
    if (ctx->tensor_kind == 0) throw std::invalid_argument("no tensor set");
    constexpr int kGrid = 592;
    ctx->est_partials.alloc(kGrid * sizeof(double));
    ctx->est_out.alloc(sizeof(double));
    double* parts = ctx->est_partials.as<double>();
    if (ctx->tensor_kind == 2) {
      if (ctx->dtype == GCPB_F32)
        sumsq_kernel<float><<<kGrid, 256, 0, ctx->stream>>>(ctx->vals.as<float>(), ctx->nnz, parts);
      else
        sumsq_kernel<double><<<kGrid, 256, 0, ctx->stream>>>(ctx->vals.as<double>(), ctx->nnz, parts);
    } else {
      const int64_t n = static_cast<int64_t>(ctx->total);
      if (ctx->dense_storage == GCPB_STORE_BIT)
        popcount_kernel<<<kGrid, 256, 0, ctx->stream>>>(ctx->dense.as<uint32_t>(), (n + 31) / 32,
                                                        parts);
      else if (ctx->dense_storage == GCPB_STORE_U8)
        sumsq_kernel<uint8_t><<<kGrid, 256, 0, ctx->stream>>>(ctx->dense.as<uint8_t>(), n, parts);
      else if (ctx->dense_storage == GCPB_STORE_F32)
        sumsq_kernel<float><<<kGrid, 256, 0, ctx->stream>>>(ctx->dense.as<float>(), n, parts);
      else
        sumsq_kernel<double><<<kGrid, 256, 0, ctx->stream>>>(ctx->dense.as<double>(), n, parts);
    }
    sum_partials_kernel<<<1, 32, 0, ctx->stream>>>(parts, kGrid, ctx->est_out.as<double>());
    CK(cudaGetLastError());
    double ss = 0.0;
    CK(cudaMemcpyAsync(&ss, ctx->est_out.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    *out = std::sqrt(ss);
  });
}

int gcpb_value_at(gcpb_ctx* ctx, int64_t n, const int64_t* idx, double* x_out) {
  return guard(ctx, [&] {
    if (ctx->tensor_kind == 0) throw std::invalid_argument("no tensor set");
    for (int64_t e = 0; e < n; ++e) check_index_host(ctx, idx + e * ctx->d);
    if (n == 0) return;
    if (ctx->tensor_kind == 2) ensure_hash(ctx);
    std::vector<uint64_t> lin(static_cast<size_t>(n)), lin_hi(static_cast<size_t>(n));
    for (int64_t e = 0; e < n; ++e) {  // linear_index (shape.cpp:87-96), 128-bit
      unsigned __int128 l = 0;
      for (int k = 0; k < ctx->d; ++k)
        l += static_cast<unsigned __int128>(idx[e * ctx->d + k]) *
             ((static_cast<unsigned __int128>(ctx->stride_hi[k]) << 64) | ctx->stride_lo[k]);
      lin[e] = static_cast<uint64_t>(l);
      lin_hi[e] = static_cast<uint64_t>(l >> 64);
    }
    DBuf dl, dlh, dx;
    dl.alloc(n * 8);
    dx.alloc(n * 8);
    CK(cudaMemcpyAsync(dl.p, lin.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream));
    if (ctx->wide) {
      dlh.alloc(n * 8);
      CK(cudaMemcpyAsync(dlh.p, lin_hi.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream));
    }
    int xkind = X_SPARSE;
    if (ctx->tensor_kind == 1)
      xkind = ctx->dense_storage == GCPB_STORE_BIT
                  ? X_DENSE_BIT
                  : (ctx->dense_storage == GCPB_STORE_U8
                         ? X_DENSE_U8
                         : (ctx->dense_storage == GCPB_STORE_F32 ? X_DENSE_F32 : X_DENSE_F64));
    if (ctx->dtype == GCPB_F32)
      value_at_kernel<float><<<grid_for(n, 256, ctx->num_sms), 256, 0, ctx->stream>>>(
          dl.as<uint64_t>(), n, xkind, ctx->dense.p, ctx->vals.as<float>(),
          ctx->hash_ready ? ctx->hkeys.as<uint64_t>() : nullptr, ctx->hvals.as<uint32_t>(),
          ctx->hmask, dx.as<double>(), ctx->wide ? dlh.as<uint64_t>() : nullptr,
          ctx->hkeys_hi.as<uint64_t>());
    else
      value_at_kernel<double><<<grid_for(n, 256, ctx->num_sms), 256, 0, ctx->stream>>>(
          dl.as<uint64_t>(), n, xkind, ctx->dense.p, ctx->vals.as<double>(),
          ctx->hash_ready ? ctx->hkeys.as<uint64_t>() : nullptr, ctx->hvals.as<uint32_t>(),
          ctx->hmask, dx.as<double>(), ctx->wide ? dlh.as<uint64_t>() : nullptr,
          ctx->hkeys_hi.as<uint64_t>());
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(x_out, dx.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
  });
}

// ---- factors / gradient / moments -----------------------------------------------------
int gcpb_set_factors(gcpb_ctx* ctx, int mode, const double* values) {
  return guard(ctx, [&] {
    NvtxRange nvtx_("gcpb_set_factors");
    ctx->check_mode(mode);
    upload(ctx, ctx->A, mode, values);
  });
}
int gcpb_get_factors(gcpb_ctx* ctx, int mode, double* out) {
  return guard(ctx, [&] {
    NvtxRange nvtx_("gcpb_get_factors");
    ctx->check_mode(mode);
    download(ctx, ctx->A, mode, out);
  });
}
int gcpb_get_grad(gcpb_ctx* ctx, int mode, double* out) {
  return guard(ctx, [&] {
    ctx->check_mode(mode);
    download(ctx, ctx->Gr, mode, out);
  });
}
int gcpb_set_grad(gcpb_ctx* ctx, int mode, const double* values) {
  return guard(ctx, [&] {
    ctx->check_mode(mode);
    upload(ctx, ctx->Gr, mode, values);
    ctx->grad_zero = false;
  });
}
int gcpb_get_moment(gcpb_ctx* ctx, int which, int mode, double* out) {
  return guard(ctx, [&] {
    ctx->check_mode(mode);
    if (which != 0 && which != 1) throw std::invalid_argument("moment must be 0 or 1");
    download(ctx, which == 0 ? ctx->B : ctx->C, mode, out);
  });
}
int gcpb_set_moment(gcpb_ctx* ctx, int which, int mode, const double* values) {
  return guard(ctx, [&] {
    ctx->check_mode(mode);
    if (which != 0 && which != 1) throw std::invalid_argument("moment must be 0 or 1");
    upload(ctx, which == 0 ? ctx->B : ctx->C, mode, values);
  });
}

// ---- hot path ---------------------------------------------------------------------------
int gcpb_stoch_grad(gcpb_ctx* ctx, const gcpb_sampler* sampler, const gcpb_loss* loss,
                    uint64_t seed, uint64_t iter, gcpb_stats* stats) {
  return guard(ctx, [&] {
    NvtxRange nvtx_("gcpb_stoch_grad");
    validate_sampler(sampler);
    validate_loss(loss);
    if (ctx->tensor_kind == 0) throw std::invalid_argument("no tensor set");
    if (sampler->strategy != GCPB_UNIFORM && ctx->tensor_kind != 2)
      throw std::invalid_argument(sampler->strategy == GCPB_STRATIFIED
                                      ? "stratified sampling requires a sparse tensor"
                                      : "semi-stratified sampling requires a sparse tensor");
    check_data_domain(ctx, loss->kind);
    ensure_grad_zero(ctx);
    const bool want_stats = stats != nullptr;
    SampleResult res;
    if (ctx->dtype == GCPB_F32)
      res = stoch_grad_impl<float>(ctx, sampler, loss, seed, iter, true, false, want_stats, false, -1);
    else
      res = stoch_grad_impl<double>(ctx, sampler, loss, seed, iter, true, false, want_stats, false, -1);
    ctx->grad_zero = false;
    if (want_stats) {
      *stats = res.stats;
      ctx->sync();
    }
  });
}

int gcpb_draw_samples(gcpb_ctx* ctx, const gcpb_sampler* sampler, const gcpb_loss* loss,
                      uint64_t seed, uint64_t iter, int64_t cap, int64_t* idx_out,
                      double* x_out, double* w_out, int32_t* flag_out, double* m_out,
                      double* y_out, int64_t* n_out, gcpb_stats* stats) {
  return guard(ctx, [&] {
    NvtxRange nvtx_("gcpb_draw_samples");
    validate_sampler(sampler);
    validate_loss(loss);
    if (ctx->tensor_kind == 0) throw std::invalid_argument("no tensor set");
    if (sampler->strategy != GCPB_UNIFORM && ctx->tensor_kind != 2)
      throw std::invalid_argument("stratified sampling requires a sparse tensor");
    check_data_domain(ctx, loss->kind);
    const int64_t n = expected_samples(ctx, sampler);
    if (n_out) *n_out = n;
    if (n > cap) throw std::length_error("gcpb_draw_samples: capacity too small");
    alloc_record(ctx, n);
    SampleResult res;
    if (ctx->dtype == GCPB_F32)
      res = stoch_grad_impl<float>(ctx, sampler, loss, seed, iter, false, true, true, false, -1);
    else
      res = stoch_grad_impl<double>(ctx, sampler, loss, seed, iter, false, true, true, false, -1);
    if (n > 0) {
      if (idx_out) CK(cudaMemcpyAsync(idx_out, ctx->s_idx.p, n * ctx->d * 8, cudaMemcpyDeviceToHost, ctx->stream));
      if (x_out) CK(cudaMemcpyAsync(x_out, ctx->s_x.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
      if (w_out) CK(cudaMemcpyAsync(w_out, ctx->s_w.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
      if (flag_out) CK(cudaMemcpyAsync(flag_out, ctx->s_flag.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
      if (m_out) CK(cudaMemcpyAsync(m_out, ctx->s_m.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
      if (y_out) CK(cudaMemcpyAsync(y_out, ctx->s_y.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    }
    ctx->sync();
    if (stats) *stats = res.stats;
  });
}


int gcpb_eval_deriv(gcpb_ctx* ctx, int64_t n, const int64_t* idx, const double* x,
                    const double* w, const int32_t* flags, const gcpb_loss* loss,
                    double* m_out, double* y_out) {
  return guard(ctx, [&] {
    validate_loss(loss);
    if (n < 0) throw std::invalid_argument("negative sample count");
    for (int64_t e = 0; e < n; ++e) {
      check_index_host(ctx, idx + e * ctx->d);
      check_domain_value(loss->kind, x[e]);
    }
    if (n == 0) return;
    alloc_record(ctx, n);
    ctx->s_aux.alloc(static_cast<size_t>(n) * sizeof(double));
    std::vector<int32_t> f(static_cast<size_t>(n), 0);
    if (flags) std::copy(flags, flags + n, f.begin());
    CK(cudaMemcpyAsync(ctx->s_idx.p, idx, n * ctx->d * 8, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->s_x.p, x, n * 8, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->s_w.p, w, n * 8, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->s_flag.p, f.data(), n * 4, cudaMemcpyHostToDevice, ctx->stream));
    if (ctx->dtype == GCPB_F32)
      given_launch<float>(ctx, n, loss, false, true, false);
    else
      given_launch<double>(ctx, n, loss, false, true, false);
    if (m_out) CK(cudaMemcpyAsync(m_out, ctx->s_m.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    if (y_out) CK(cudaMemcpyAsync(y_out, ctx->s_aux.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
  });
}

int gcpb_mttkrp_samples(gcpb_ctx* ctx, int64_t n, const int64_t* idx, const double* y) {
  return guard(ctx, [&] {
    if (n < 0) throw std::invalid_argument("negative sample count");
    for (int64_t e = 0; e < n; ++e) check_index_host(ctx, idx + e * ctx->d);
    CK(cudaMemsetAsync(ctx->Gr.p, 0, ctx->nelem * ctx->tsize, ctx->stream));
    ctx->grad_zero = true;
    if (n == 0) {
      ctx->sync();
      return;
    }
    alloc_record(ctx, n);
    CK(cudaMemcpyAsync(ctx->s_idx.p, idx, n * ctx->d * 8, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->s_y.p, y, n * 8, cudaMemcpyHostToDevice, ctx->stream));
    gcpb_loss l{GCPB_LOSS_GAUSSIAN, 0.0};
    if (ctx->dtype == GCPB_F32)
      given_launch<float>(ctx, n, &l, true, false, true);
    else
      given_launch<double>(ctx, n, &l, true, false, true);
    ctx->grad_zero = false;
    ctx->sync();
  });
}

// ---- optimizer -------------------------------------------------------------------------------
int gcpb_adam_step(gcpb_ctx* ctx, const gcpb_adam* adam) {
  return guard(ctx, [&] {
    NvtxRange nvtx_("gcpb_adam_step");
    set_adam_params(ctx, adam);
    if (ctx->dtype == GCPB_F32)
      adam_launch<float>(ctx);
    else
      adam_launch<double>(ctx);
    ctx->grad_zero = true;
  });
}

int gcpb_adam_reset(gcpb_ctx* ctx) {
  return guard(ctx, [&] {
    const size_t bytes = ctx->nelem * ctx->tsize;
    CK(cudaMemsetAsync(ctx->B.p, 0, bytes, ctx->stream));
    CK(cudaMemsetAsync(ctx->C.p, 0, bytes, ctx->stream));
    const int64_t zero = 0;
    CK(cudaMemcpyAsync(&ctx->dst()->t, &zero, 8, cudaMemcpyHostToDevice, ctx->stream));
    ctx->sync();
    ctx->moments_sharded = false;
  });
}

int gcpb_get_iterations(gcpb_ctx* ctx, int64_t* out) {
  return guard(ctx, [&] {
    CK(cudaMemcpyAsync(out, &ctx->dst()->t, 8, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
  });
}

int gcpb_set_iterations(gcpb_ctx* ctx, int64_t iterations) {
  return guard(ctx, [&] {
    CK(cudaMemcpyAsync(&ctx->dst()->t, &iterations, 8, cudaMemcpyHostToDevice, ctx->stream));
    ctx->sync();
  });
}

int gcpb_step(gcpb_ctx* ctx, const gcpb_sampler* sampler, const gcpb_loss* loss, uint64_t seed,
              uint64_t iter, const gcpb_adam* adam) {
  return guard(ctx, [&] {
    NvtxRange nvtx_("gcpb_step");
    check_step_args(ctx, sampler, loss);
    set_adam_params(ctx, adam);
    ensure_grad_zero(ctx);
    if (ctx->dtype == GCPB_F32)
      step_impl<float>(ctx, sampler, loss, seed, iter, nullptr, ZERO_HOST_CHECK);
    else
      step_impl<double>(ctx, sampler, loss, seed, iter, nullptr, ZERO_HOST_CHECK);
  });
}

int gcpb_step_host(gcpb_ctx* ctx, const gcpb_sampler* sampler, const gcpb_loss* loss,
                   uint64_t seed, uint64_t iter, const gcpb_adam* adam, const double* model_in,
                   double* model_out) {
  return guard(ctx, [&] {
    NvtxRange nvtx_("gcpb_step_host");
    check_step_args(ctx, sampler, loss);
    // Small problems on page-locked buffers: one cluster launch reads the
    // model from host memory, runs the iteration and writes it back (no
    // copies or pack kernels: C1's step is launch/latency-bound).
    if (model_in && model_out) {
      const void* din = host_device_alias(model_in);
      void* dout = din ? const_cast<void*>(host_device_alias(model_out)) : nullptr;
      const bool small = ctx->dtype == GCPB_F32 ? small_eligible<float>(ctx, sampler)
                                                : small_eligible<double>(ctx, sampler);
      if (din && dout && small) {
        set_adam_params(ctx, adam);
        if (ctx->dtype == GCPB_F32)
          small_launch<float>(ctx, sampler, loss, seed, 1, static_cast<const double*>(din),
                              static_cast<double*>(dout), &iter);
        else
          small_launch<double>(ctx, sampler, loss, seed, 1, static_cast<const double*>(din),
                               static_cast<double*>(dout), &iter);
        ctx->last_steps_path = 1;
        CK(cudaStreamSynchronize(ctx->stream));
        return;
      }
    }
    // pinned buffers are transferred in place: the call synchronises on the
    // download before returning (without model_out, on the stream)
    ctx->last_h2d_bytes = ctx->last_d2h_bytes = 0;
    if (model_in) upload(ctx, ctx->A, -1, model_in, is_pinned(model_in));
    set_adam_params(ctx, adam);
    ensure_grad_zero(ctx);
    if (ctx->dtype == GCPB_F32)
      step_impl<float>(ctx, sampler, loss, seed, iter, nullptr, ZERO_HOST_CHECK);
    else
      step_impl<double>(ctx, sampler, loss, seed, iter, nullptr, ZERO_HOST_CHECK);
    if (model_out)
      download(ctx, ctx->A, -1, model_out, is_pinned(model_out));
    else if (model_in)
      CK(cudaStreamSynchronize(ctx->stream));
  });
}

int gcpb_last_transfer_bytes(const gcpb_ctx* ctx, int64_t* h2d, int64_t* d2h) {
  if (!ctx || !h2d || !d2h) return GCPB_ERR_USAGE;
  *h2d = ctx->last_h2d_bytes;
  *d2h = ctx->last_d2h_bytes;
  return GCPB_OK;
}

int gcpb_run_steps(gcpb_ctx* ctx, const gcpb_sampler* sampler, const gcpb_loss* loss,
                   uint64_t seed, uint64_t iter0, int64_t n, const gcpb_adam* adam) {
  return guard(ctx, [&] {
    NvtxRange nvtx_("gcpb_run_steps");
    check_step_args(ctx, sampler, loss);
    if (n < 0) throw std::invalid_argument("negative step count");
    if (n == 0) return;
    if (ctx->dtype == GCPB_F32)
      run_steps_impl<float>(ctx, sampler, loss, seed, iter0, n, adam);
    else
      run_steps_impl<double>(ctx, sampler, loss, seed, iter0, n, adam);
  });
}

int gcpb_kernel_timing(gcpb_ctx* ctx, int enable) {
  return guard(ctx, [&] {
    ctx->sync();
    ctx->timing = enable != 0;
    if (enable) ctx->tevents_used = 0;
  });
}

int gcpb_kernel_time(gcpb_ctx* ctx, double* total_ms, int64_t* launches) {
  return guard(ctx, [&] {
    ctx->sync();
    double tot = 0.0;
    for (size_t i = 0; i < ctx->tevents_used; ++i) {
      float ms = 0.0f;
      CK(cudaEventElapsedTime(&ms, ctx->tevents[i].first, ctx->tevents[i].second));
      tot += ms;
    }
    *total_ms = tot;
    *launches = static_cast<int64_t>(ctx->tevents_used);
  });
}

int gcpb_set_draw_stream(gcpb_ctx* ctx, int kind, uint64_t counter) {
  return guard(ctx, [&] {
    if (kind != 0 && kind != 1) throw std::invalid_argument("draw stream must be 0 or 1");
    ctx->sync();
    ctx->draw_stream = kind;
    const uint32_t zero = 0;
    CK(cudaMemcpyAsync(&ctx->dst()->ref_ctr, &counter, 8, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(&ctx->dst()->ref_flag, &zero, 4, cudaMemcpyHostToDevice, ctx->stream));
    ctx->sync();
  });
}

int gcpb_get_draw_counter(gcpb_ctx* ctx, uint64_t* counter) {
  return guard(ctx, [&] {
    CK(cudaMemcpyAsync(counter, &ctx->dst()->ref_ctr, 8, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
  });
}

int gcpb_steps_path(const gcpb_ctx* ctx) { return ctx ? ctx->last_steps_path : -1; }

int64_t gcpb_debug_check_failures(int64_t* first_site, int64_t* first_value) {
#ifdef GCPB_CHECKED
  unsigned long long h[4] = {0, 0, 0, 0};
  if (cudaDeviceSynchronize() != cudaSuccess) return -2;
  if (cudaMemcpyFromSymbol(h, g_chk_dev, sizeof(h)) != cudaSuccess) return -2;
  if (first_site) *first_site = static_cast<int64_t>(h[1]);
  if (first_value) *first_value = static_cast<int64_t>(h[2]);
  return static_cast<int64_t>(h[0]);
#else
  if (first_site) *first_site = 0;
  if (first_value) *first_value = 0;
  return -1;
#endif
}

int64_t gcpb_debug_guard_failures(int64_t* buffers_checked) {
  if (buffers_checked) *buffers_checked = g_guard_checked.load(std::memory_order_relaxed);
  return g_guard_on ? g_guard_bad.load(std::memory_order_relaxed) : -1;
}

int gcpb_run_steps_launches(const gcpb_ctx* ctx, int64_t* kernels) {
  if (!ctx || !kernels) return GCPB_ERR_USAGE;
  *kernels = ctx->last_steps_path == 1 ? 1 : ctx->graph_kernels;
  return GCPB_OK;
}

int gcpb_hot_rows(const gcpb_ctx* ctx, int* rows, int* copies) {
  if (!ctx) return GCPB_ERR_USAGE;
  if (rows) *rows = ctx->hot_version == ctx->tensor_version ? ctx->hot_n : 0;
  if (copies) *copies = ctx->hot_last;
  return GCPB_OK;
}

int gcpb_interleaved(const gcpb_ctx* ctx, int* enabled, int* last) {
  if (!ctx) return GCPB_ERR_USAGE;
  if (enabled) *enabled = ctx->il_enabled ? 1 : 0;
  if (last) *last = ctx->il_last ? 1 : 0;
  return GCPB_OK;
}

int gcpb_synchronize(gcpb_ctx* ctx) {
  return guard(ctx, [&] { sync_and_check(ctx); });
}

int gcpb_gradient_full(gcpb_ctx* ctx, const gcpb_loss* loss) {
  return guard(ctx, [&] {
    NvtxRange nvtx_("gcpb_gradient_full");
    validate_loss(loss);
    if (ctx->dtype == GCPB_F32)
      gradient_full_impl<float>(ctx, loss);
    else
      gradient_full_impl<double>(ctx, loss);
    ctx->sync();
  });
}

int gcpb_gradient_poisson_implicit(gcpb_ctx* ctx, const gcpb_loss* loss) {
  return guard(ctx, [&] {
    NvtxRange nvtx_("gcpb_gradient_poisson_implicit");
    validate_loss(loss);
    no_nz_shard(ctx, "gradient_poisson_implicit");
    if (ctx->dtype == GCPB_F32)
      poisson_implicit_impl<float>(ctx, loss);
    else
      poisson_implicit_impl<double>(ctx, loss);
  });
}

int gcpb_gradient_moments(gcpb_ctx* ctx, const gcpb_sampler* sampler, const gcpb_loss* loss,
                          int64_t trials, uint64_t seed, double* mean, double* variance) {
  return guard(ctx, [&] {
    check_step_args(ctx, sampler, loss);
    no_nz_shard(ctx, "gradient_moments");
    if (ctx->dtype == GCPB_F32)
      gradient_moments_impl<float>(ctx, sampler, loss, trials, seed, mean, variance);
    else
      gradient_moments_impl<double>(ctx, sampler, loss, trials, seed, mean, variance);
  });
}

int gcpb_bias_variance(gcpb_ctx* ctx, const gcpb_sampler* sampler, const gcpb_loss* loss,
                       int64_t trials, uint64_t seed, const double* exact, double* bias,
                       double* variance) {
  return guard(ctx, [&] {
    NvtxRange nvtx_("gcpb_bias_variance");
    check_step_args(ctx, sampler, loss);
    no_nz_shard(ctx, "empirical_bias_variance");
    if (ctx->dtype == GCPB_F32)
      bias_variance_impl<float>(ctx, sampler, loss, trials, seed, exact, bias, variance);
    else
      bias_variance_impl<double>(ctx, sampler, loss, trials, seed, exact, bias, variance);
  });
}

int gcpb_rng_seed(uint64_t seed, gcpb_rng* out) {
  return guard(nullptr, [&] {
    if (!out) throw std::invalid_argument("gcpb_rng_seed: null output");
    rng_out(HostRngStream(seed), out);
  });
}

int gcpb_rng_split(const gcpb_rng* in, uint64_t label, gcpb_rng* out) {
  return guard(nullptr, [&] {
    if (!in || !out) throw std::invalid_argument("gcpb_rng_split: null argument");
    rng_out(HostRngStream::from_key(in->key).split(label), out);
  });
}

int gcpb_gen_gamma_problem(gcpb_ctx* ctx, gcpb_rng* rng, int storage, double* truth_out) {
  return guard(ctx, [&] {
    if (!rng) throw std::invalid_argument("gen_gamma_problem: null rng");
    gen_gamma_impl(ctx, rng, storage, truth_out);
  });
}

int gcpb_gen_binary_problem(gcpb_ctx* ctx, const gcpb_binary_spec* spec, gcpb_rng* rng,
                            double* truth_out) {
  return guard(ctx, [&] {
    if (!rng || !spec) throw std::invalid_argument("gen_binary_problem: null argument");
    if (ctx->wide) throw std::invalid_argument("gen_binary_problem: N >= 2^64 not supported");
    gen_binary_impl(ctx, spec, rng, truth_out);
  });
}

int gcpb_fit_gcp_adam(gcpb_ctx* ctx, const gcpb_loss* loss, const gcpb_fit_config* cfg,
                      gcpb_trace_record* trace, int64_t trace_cap, int64_t* n_trace,
                      double* final_estimate) {
  return guard(ctx, [&] {
    NvtxRange nvtx_("gcpb_fit_gcp_adam");
    using clock = std::chrono::steady_clock;
    const auto start = clock::now();
    auto secs = [](clock::time_point a) {
      return std::chrono::duration<double>(clock::now() - a).count();
    };
    if (!cfg) throw std::invalid_argument("fit: null config");
    validate_loss(loss);
    // FitConfig::validate (optimizer.cpp:31-45)
    validate_sampler(&cfg->sampler);
    if (!(cfg->learning_rate > 0.0)) throw std::invalid_argument("fit: learning rate must be > 0");
    if (!(cfg->beta1 >= 0.0 && cfg->beta1 < 1.0) || !(cfg->beta2 >= 0.0 && cfg->beta2 < 1.0))
      throw std::invalid_argument("fit: moment decays must satisfy 0 <= beta < 1");
    if (!(cfg->epsilon > 0.0)) throw std::invalid_argument("fit: epsilon must be > 0");
    if (cfg->epoch_iters < 1) throw std::invalid_argument("fit: iterations per epoch must be >= 1");
    if (cfg->max_bad_epochs < 0) throw std::invalid_argument("fit: max bad epochs must be >= 0");
    if (!(cfg->decay > 0.0 && cfg->decay < 1.0))
      throw std::invalid_argument("fit: decay must be in (0, 1)");
    if (cfg->estimator_samples < 0) throw std::invalid_argument("fit: estimator count must be >= 0");
    if (cfg->max_epochs < 0) throw std::invalid_argument("fit: max epochs must be >= 0");
    check_step_args(ctx, &cfg->sampler, loss);

    // lower bound (optimizer.cpp:74)
    gcpb_adam ad{cfg->learning_rate, cfg->beta1, cfg->beta2, cfg->epsilon, 0, 0.0};
    if (cfg->lower_bound_mode == 1) {
      ad.has_lower_bound = 1;
      ad.lower_bound = cfg->lower_bound;
    } else if (cfg->lower_bound_mode == 0) {
      const int k = loss->kind;
      if (k == GCPB_LOSS_POISSON || k == GCPB_LOSS_BERNOULLI_ODDS || k == GCPB_LOSS_GAMMA ||
          k == GCPB_LOSS_BETA_HALF) {
        ad.has_lower_bound = 1;
        ad.lower_bound = 0.0;
      }
    }

    // streams (optimizer.cpp:76-78)
    const HostRngStream root(cfg->seed);
    const uint64_t est_seed = root.split("estimator").key();
    const uint64_t grad_seed = root.split("gradients").key();
    {
      const int rc = gcpb_set_draw_stream(ctx, cfg->draw_stream == 1 ? 1 : 0, 0);
      if (rc != GCPB_OK) throw std::runtime_error(ctx->err);
    }

    // init (optimizer.cpp:80-82, kruskal.cpp:33-45,85-93)
    if (!cfg->keep_factors) {
      HostRngStream init = root.split("init");
      std::vector<std::vector<double>> F(static_cast<size_t>(ctx->d));
      for (int k = 0; k < ctx->d; ++k) {
        F[k].resize(static_cast<size_t>(ctx->dims[k] * ctx->r));
        for (auto& v : F[k]) v = init.next_double();
      }
      double data_norm = 0.0;  // TensorView::norm
      if (gcpb_tensor_norm(ctx, &data_norm) != GCPB_OK) throw std::runtime_error(ctx->err);
      if (data_norm > 0.0) {
        const double current = model_norm_host(F, ctx->r);
        if (current == 0.0) throw std::invalid_argument("kruskal model: cannot rescale a zero model");
        const double ratio = std::pow(data_norm / current, 1.0 / ctx->d);
        for (auto& f : F)
          for (auto& v : f) v *= ratio;
      }
      std::vector<double> flat;
      for (auto& f : F) flat.insert(flat.end(), f.begin(), f.end());
      upload(ctx, ctx->A, -1, flat.data());
    }

    // estimator (optimizer.cpp:84-91)
    const int est_kind = cfg->estimator_kind >= 0
                             ? cfg->estimator_kind
                             : (ctx->tensor_kind == 2 ? GCPB_EST_STRATIFIED : GCPB_EST_UNIFORM);
    {
      const int rc = gcpb_estimator_draw(ctx, est_kind, cfg->estimator_samples, 1.1, est_seed);
      if (rc != GCPB_OK) throw std::runtime_error(ctx->err);
    }
    auto estimate = [&]() {
      double f = 0.0;
      const int rc = gcpb_estimate(ctx, loss, &f);
      if (rc != GCPB_OK) throw std::runtime_error(ctx->err);
      return f;
    };

    // AdamState::init (optimizer.cpp:93)
    const size_t bytes = ctx->nelem * ctx->tsize;
    CK(cudaMemsetAsync(ctx->B.p, 0, bytes, ctx->stream));
    CK(cudaMemsetAsync(ctx->C.p, 0, bytes, ctx->stream));
    {
      const int64_t zero = 0;
      CK(cudaMemcpyAsync(&ctx->dst()->t, &zero, 8, cudaMemcpyHostToDevice, ctx->stream));
      ctx->sync();
    }
    double lr = cfg->learning_rate;
    int64_t bad = 0;
    double best = estimate();
    if (!std::isfinite(best))
      throw std::runtime_error("fit: initial loss estimate is not finite (" +
                               std::to_string(best) + ")");
    {
      const int rc = gcpb_snapshot_save(ctx);
      if (rc != GCPB_OK) throw std::runtime_error(ctx->err);
    }
    int64_t nt = 0;
    auto record = [&](int64_t epoch, double f, double a, double sec, bool acc) {
      if (nt < trace_cap && trace) trace[nt] = gcpb_trace_record{epoch, f, a, sec, acc ? 1 : 0};
      ++nt;
    };
    record(0, best, lr, secs(start), true);
    // Small stratified budgets step with the host-checked sampler (exact for
    // any q); large ones replay a CUDA graph per epoch.
    const bool graph_ok = !(cfg->sampler.strategy == GCPB_STRATIFIED &&
                            cfg->sampler.zero_samples < 4096);
    uint64_t it = 0;  // gradient stream position, never rewound (optimizer.cpp:78)
    for (int64_t epoch = 1; epoch <= cfg->max_epochs; ++epoch) {
      const auto e0 = clock::now();
      const double alpha_used = lr;
      ad.learning_rate = lr;
      if (graph_ok) {
        if (ctx->dtype == GCPB_F32)
          run_steps_impl<float>(ctx, &cfg->sampler, loss, grad_seed, it, cfg->epoch_iters, &ad);
        else
          run_steps_impl<double>(ctx, &cfg->sampler, loss, grad_seed, it, cfg->epoch_iters, &ad);
        sync_and_check(ctx);
      } else {
        set_adam_params(ctx, &ad);
        ensure_grad_zero(ctx);
        for (int64_t i = 0; i < cfg->epoch_iters; ++i) {
          if (ctx->dtype == GCPB_F32)
            step_impl<float>(ctx, &cfg->sampler, loss, grad_seed, it + i, nullptr, ZERO_HOST_CHECK);
          else
            step_impl<double>(ctx, &cfg->sampler, loss, grad_seed, it + i, nullptr, ZERO_HOST_CHECK);
        }
      }
      it += static_cast<uint64_t>(cfg->epoch_iters);
      const double fnew = estimate();
      if (!std::isfinite(fnew))
        throw std::runtime_error("fit: loss estimate became non-finite at epoch " +
                                 std::to_string(epoch));
      const double sec = secs(e0);
      if (fnew <= best) {  // optimizer.cpp:128-135
        best = fnew;
        const int rc = gcpb_snapshot_save(ctx);
        if (rc != GCPB_OK) throw std::runtime_error(ctx->err);
        record(epoch, fnew, alpha_used, sec, true);
      } else {  // optimizer.cpp:136-146
        const int rc = gcpb_snapshot_restore(ctx);
        if (rc != GCPB_OK) throw std::runtime_error(ctx->err);
        lr *= cfg->decay;
        ++bad;
        record(epoch, fnew, alpha_used, sec, false);
        if (bad > cfg->max_bad_epochs) break;
      }
    }
    if (n_trace) *n_trace = nt;
    if (final_estimate) *final_estimate = best;
  });
}

// ---- estimator -----------------------------------------------------------------------------------
int gcpb_estimator_set(gcpb_ctx* ctx, int64_t n, const int64_t* idx, const double* x,
                       const double* w) {
  return guard(ctx, [&] {
    if (n < 0) throw std::invalid_argument("estimator: count must be >= 0");
    for (int64_t e = 0; e < n; ++e) check_index_host(ctx, idx + e * ctx->d);
    const size_t nn = static_cast<size_t>(std::max<int64_t>(n, 1));
    ctx->est_idx.alloc(nn * ctx->d * 8);
    ctx->est_x.alloc(nn * 8);
    ctx->est_w.alloc(nn * 8);
    if (n > 0) {
      CK(cudaMemcpyAsync(ctx->est_idx.p, idx, n * ctx->d * 8, cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaMemcpyAsync(ctx->est_x.p, x, n * 8, cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaMemcpyAsync(ctx->est_w.p, w, n * 8, cudaMemcpyHostToDevice, ctx->stream));
    }
    ctx->est_n = n;
    ctx->sync();
  });
}

int gcpb_estimator_draw(gcpb_ctx* ctx, int kind, int64_t count, double rho, uint64_t seed) {
  return guard(ctx, [&] {
    NvtxRange nvtx_("gcpb_estimator_draw");
    if (count < 0) throw std::invalid_argument("estimator: count must be >= 0");
    if (kind != GCPB_EST_UNIFORM && kind != GCPB_EST_STRATIFIED)
      throw std::invalid_argument("unknown estimator kind");
    if (ctx->tensor_kind == 0) throw std::invalid_argument("no tensor set");
    if (kind == GCPB_EST_STRATIFIED && ctx->tensor_kind != 2)
      throw std::invalid_argument("stratified estimator requires a sparse tensor");
    gcpb_sampler sk{};
    if (kind == GCPB_EST_UNIFORM) {
      sk.strategy = GCPB_UNIFORM;
      sk.num_samples = count;
    } else {
      sk.strategy = GCPB_STRATIFIED;
      sk.nonzero_samples = count / 2;
      sk.zero_samples = count - count / 2;
      sk.oversample = rho;
      if (!(rho > 1.0)) throw std::invalid_argument("sample_zeros_rejection: rho must be > 1");
    }
    const int64_t n = count;
    alloc_record(ctx, n);
    gcpb_loss l{GCPB_LOSS_GAUSSIAN, 0.0};
    // RefStream: the estimator has its own stream (split "estimator"), drawn
    // from counter 0; the gradient stream's counter is preserved.
    uint64_t saved_ctr = 0;
    if (ctx->draw_stream == 1) {
      CK(cudaMemcpyAsync(&saved_ctr, &ctx->dst()->ref_ctr, 8, cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
      const uint64_t zero = 0;
      CK(cudaMemcpyAsync(&ctx->dst()->ref_ctr, &zero, 8, cudaMemcpyHostToDevice, ctx->stream));
    }
    if (n > 0) {
      if (kind == GCPB_EST_UNIFORM) {
        if (ctx->dtype == GCPB_F32)
          stoch_grad_impl<float>(ctx, &sk, &l, seed, 0, false, true, true, true, kind);
        else
          stoch_grad_impl<double>(ctx, &sk, &l, seed, 0, false, true, true, true, kind);
      } else {
        if (ctx->dtype == GCPB_F32)
          stoch_grad_impl<float>(ctx, &sk, &l, seed, 0, false, true, true, true, kind);
        else
          stoch_grad_impl<double>(ctx, &sk, &l, seed, 0, false, true, true, true, kind);
      }
    }
    const size_t nn = static_cast<size_t>(std::max<int64_t>(n, 1));
    ctx->est_idx.alloc(nn * ctx->d * 8);
    ctx->est_x.alloc(nn * 8);
    ctx->est_w.alloc(nn * 8);
    if (n > 0) {
      CK(cudaMemcpyAsync(ctx->est_idx.p, ctx->s_idx.p, n * ctx->d * 8, cudaMemcpyDeviceToDevice, ctx->stream));
      CK(cudaMemcpyAsync(ctx->est_x.p, ctx->s_x.p, n * 8, cudaMemcpyDeviceToDevice, ctx->stream));
      CK(cudaMemcpyAsync(ctx->est_w.p, ctx->s_w.p, n * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    ctx->est_n = n;
    if (ctx->draw_stream == 1) {
      CK(cudaMemcpyAsync(&ctx->dst()->ref_ctr, &saved_ctr, 8, cudaMemcpyHostToDevice, ctx->stream));
    }
    ctx->sync();
  });
}

int64_t gcpb_estimator_size(const gcpb_ctx* ctx) { return ctx ? ctx->est_n : 0; }

int gcpb_estimator_get(gcpb_ctx* ctx, int64_t* idx_out, double* x_out, double* w_out) {
  return guard(ctx, [&] {
    const int64_t n = ctx->est_n;
    if (n > 0) {
      if (idx_out) CK(cudaMemcpyAsync(idx_out, ctx->est_idx.p, n * ctx->d * 8, cudaMemcpyDeviceToHost, ctx->stream));
      if (x_out) CK(cudaMemcpyAsync(x_out, ctx->est_x.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
      if (w_out) CK(cudaMemcpyAsync(w_out, ctx->est_w.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    }
    ctx->sync();
  });
}

int gcpb_estimate(gcpb_ctx* ctx, const gcpb_loss* loss, double* out) {
  return guard(ctx, [&] {
    NvtxRange nvtx_("gcpb_estimate");
    validate_loss(loss);
    if (ctx->est_n == 0) {
      *out = 0.0;
      return;
    }
    if (ctx->dtype == GCPB_F32)
      estimate_launch<float>(ctx, loss);
    else
      estimate_launch<double>(ctx, loss);
    CK(cudaMemcpyAsync(out, ctx->est_out.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
  });
}

// ---- snapshots ----------------------------------------------------------------------------------
int gcpb_snapshot_save(gcpb_ctx* ctx) {
  return guard(ctx, [&] {
    const size_t bytes = ctx->nelem * ctx->tsize;
    a_current(ctx);
    for (auto pr : {std::make_pair(&ctx->As, &ctx->A), std::make_pair(&ctx->Bs, &ctx->B),
                    std::make_pair(&ctx->Cs, &ctx->C)}) {
      pr.first->alloc(bytes);
      CK(cudaMemcpyAsync(pr.first->p, pr.second->p, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    DevState* st = ctx->dst();
    CK(cudaMemcpyAsync(&st->t_saved, &st->t, 8, cudaMemcpyDeviceToDevice, ctx->stream));
    ctx->have_snapshot = true;
    ctx->sync();
  });
}

int gcpb_snapshot_restore(gcpb_ctx* ctx) {
  return guard(ctx, [&] {
    if (!ctx->have_snapshot) throw std::logic_error("no snapshot saved");
    ctx->ag_ok = false;
    ctx->a_stale = false;  // A is overwritten entirely
    const size_t bytes = ctx->nelem * ctx->tsize;
    for (auto pr : {std::make_pair(&ctx->A, &ctx->As), std::make_pair(&ctx->B, &ctx->Bs),
                    std::make_pair(&ctx->C, &ctx->Cs)})
      CK(cudaMemcpyAsync(pr.first->p, pr.second->p, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    DevState* st = ctx->dst();
    CK(cudaMemcpyAsync(&st->t, &st->t_saved, 8, cudaMemcpyDeviceToDevice, ctx->stream));
    ctx->sync();
  });
}

// ---- multi-GPU ------------------------------------------------------------------------------------
int gcpb_nccl_unique_id(char out[128]) {
  return guard(nullptr, [&] {
    ncclUniqueId id;
    nck(ncclGetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(out, &id, 128);
  });
}

int gcpb_comm_init(gcpb_ctx* ctx, const char unique_id[128], int rank, int nranks) {
  return guard(ctx, [&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("bad rank/nranks");
    ncclUniqueId id;
    std::memcpy(&id, unique_id, 128);
    CK(cudaSetDevice(ctx->device));
    if (ctx->comm) ncclCommDestroy(ctx->comm);
    nck(ncclCommInitRank(&ctx->comm, nranks, id, rank), "ncclCommInitRank");
    ctx->rank = rank;
    ctx->nranks = nranks;
    apply_nz_shard(ctx);
  });
}

int gcpb_peer_handle(gcpb_ctx* ctx, void* out) {
  return guard(ctx, [&] {
    if (!out) throw std::invalid_argument("peer handle: null output");
    PeerBlob b;
    std::memset(&b, 0, sizeof(b));
    void *a = nullptr, *g = nullptr;
    int pitch = 0;
    if (ctx->dtype == GCPB_F32)
      peer_tables<float>(ctx, &a, &g, &pitch);
    else
      peer_tables<double>(ctx, &a, &g, &pitch);
    ensure_grad_zero(ctx);
    ctx->sync();
    b.magic = kPeerMagic;
    b.pid = static_cast<int32_t>(getpid());
    b.device = ctx->device;
    b.il = ctx->il_enabled ? 1 : 0;
    b.dtype = ctx->dtype;
    b.rp = static_cast<int32_t>(ctx->rp);
    b.pitch = pitch;
    b.nelem = ctx->nelem;
    void* base_a = ctx->il_enabled ? ctx->AG.p : ctx->A.p;
    void* base_g = ctx->il_enabled ? ctx->AG.p : ctx->Gr.p;
    if (g_guard_on) {  // guarded allocations start one band earlier
      base_a = static_cast<unsigned char*>(base_a) - kGuardBytes;
      base_g = static_cast<unsigned char*>(base_g) - kGuardBytes;
    }
    CK(cudaIpcGetMemHandle(&b.ha, base_a));
    CK(cudaIpcGetMemHandle(&b.hg, base_g));
    b.raw_a = reinterpret_cast<uint64_t>(a);
    b.raw_g = reinterpret_cast<uint64_t>(g);
    b.base_a = reinterpret_cast<uint64_t>(base_a);
    b.base_g = reinterpret_cast<uint64_t>(base_g);
    std::memset(out, 0, GCPB_PEER_HANDLE_BYTES);
    std::memcpy(out, &b, sizeof(b));
  });
}

int gcpb_peer_open(gcpb_ctx* ctx, const void* handles, int nranks) {
  return guard(ctx, [&] {
    if (!handles) throw std::invalid_argument("peer open: null handles");
    if (nranks != ctx->nranks || nranks < 1 || nranks > kMaxPeers)
      throw std::invalid_argument("peer open: need one handle per rank of the communicator "
                                  "(<= 16 ranks)");
    for (void* pmap : ctx->peer_ipc) cudaIpcCloseMemHandle(pmap);
    ctx->peer_ipc.clear();
    ctx->peer_a.assign(static_cast<size_t>(nranks), nullptr);
    ctx->peer_g.assign(static_cast<size_t>(nranks), nullptr);
    ctx->peer_ok = false;
    const char* hb = static_cast<const char*>(handles);
    const int32_t me = static_cast<int32_t>(getpid());
    PeerBlob mine;
    std::memcpy(&mine, hb + static_cast<size_t>(ctx->rank) * GCPB_PEER_HANDLE_BYTES, sizeof(mine));
    for (int p = 0; p < nranks; ++p) {
      PeerBlob b;
      std::memcpy(&b, hb + static_cast<size_t>(p) * GCPB_PEER_HANDLE_BYTES, sizeof(b));
      if (b.magic != kPeerMagic) throw std::invalid_argument("peer open: not a gcpb peer handle");
      if (b.il != mine.il || b.dtype != mine.dtype || b.rp != mine.rp || b.pitch != mine.pitch ||
          b.nelem != mine.nelem)
        throw std::invalid_argument("peer open: ranks hold differently shaped tables");
      if (b.pid == me) {  // same process (threads / one-GPU emulation): raw pointers
        ctx->peer_a[static_cast<size_t>(p)] = reinterpret_cast<void*>(b.raw_a);
        ctx->peer_g[static_cast<size_t>(p)] = reinterpret_cast<void*>(b.raw_g);
        continue;
      }
      void *ma = nullptr, *mg = nullptr;
      CK(cudaIpcOpenMemHandle(&ma, b.ha, cudaIpcMemLazyEnablePeerAccess));
      ctx->peer_ipc.push_back(ma);
      if (b.base_g == b.base_a) {
        mg = ma;
      } else {
        CK(cudaIpcOpenMemHandle(&mg, b.hg, cudaIpcMemLazyEnablePeerAccess));
        ctx->peer_ipc.push_back(mg);
      }
      ctx->peer_a[static_cast<size_t>(p)] = static_cast<char*>(ma) + (b.raw_a - b.base_a);
      ctx->peer_g[static_cast<size_t>(p)] = static_cast<char*>(mg) + (b.raw_g - b.base_g);
    }
    ctx->peer_ok = nranks > 1;
  });
}

int gcpb_peer_close(gcpb_ctx* ctx) {
  return guard(ctx, [&] {
    if (ctx->moments_sharded)
      throw std::logic_error("peer close: the Adam moments are sharded over the ranks after peer "
                             "steps (each row's moments live on its owner); call gcpb_adam_reset "
                             "before returning to the replicated adam_step");
    ctx->sync();
    for (void* pmap : ctx->peer_ipc) cudaIpcCloseMemHandle(pmap);
    ctx->peer_ipc.clear();
    ctx->peer_a.clear();
    ctx->peer_g.clear();
    ctx->peer_ok = false;
  });
}

int gcpb_set_shard(gcpb_ctx* ctx, int rank, int nranks) {
  return guard(ctx, [&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("bad rank/nranks");
    ctx->rank = rank;
    ctx->nranks = nranks;
    apply_nz_shard(ctx);
  });
}

int gcpb_allreduce_grad(gcpb_ctx* ctx) {
  return guard(ctx, [&] {
    if (ctx->nranks == 1) return;
    if (!has_comm(ctx)) throw std::logic_error("allreduce without a communicator");
    if (ctx->dtype == GCPB_F32)
      comm_allreduce_grad<float>(ctx);
    else
      comm_allreduce_grad<double>(ctx);
  });
}

int gcpb_comm_init_host(gcpb_ctx* ctx, int rank, int nranks, gcpb_allgather_i64_fn allgather,
                        gcpb_allreduce_f64_fn allreduce, void* user) {
  return guard(ctx, [&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("bad rank/nranks");
    if (!allgather || !allreduce) throw std::invalid_argument("host communicator needs callbacks");
    ctx->host_allgather = allgather;
    ctx->host_allreduce = allreduce;
    ctx->host_user = user;
    ctx->rank = rank;
    ctx->nranks = nranks;
    apply_nz_shard(ctx);
  });
}

// ---- host-only helpers ------------------------------------------------------------------------------
uint64_t gcpb_philox_bounded(uint64_t seed, uint32_t tag, uint64_t iter, uint64_t t, int slot,
                             uint64_t n) {
  if (n == 0) return 0;
  return bounded_draw(seed, tag, iter, t, slot, n);
}

int64_t gcpb_zero_batch_size(double total, double zeta, double rho, int64_t shortfall) {
  return zero_batch_size_dev(total, zeta, rho, shortfall);
}

void gcpb_shard_range(int64_t n, int rank, int nranks, int64_t* begin, int64_t* end) {
  if (nranks < 1) nranks = 1;
  const int64_t base = n / nranks, rem = n % nranks;
  const int64_t b = rank * base + std::min<int64_t>(rank, rem);
  *begin = b;
  *end = b + base + (rank < rem ? 1 : 0);
}

void gcpb_stratified_keep(const int64_t* accepted_per_rank, int nranks, int rank, int64_t need,
                          int64_t* offset, int64_t* keep) {
  int64_t before = 0;
  for (int i = 0; i < rank && i < nranks; ++i) before += accepted_per_rank[i];
  *offset = before;
  const int64_t room = need - before;
  const int64_t mine = accepted_per_rank[rank];
  *keep = room <= 0 ? 0 : (mine < room ? mine : room);
}

double gcpb_loss_deriv(const gcpb_loss* loss, double x, double m) {
  const double eps = 1e-10;
  switch (loss->kind) {
    case GCPB_LOSS_GAUSSIAN: return 2.0 * (m - x);
    case GCPB_LOSS_POISSON: return 1.0 - x / (m + eps);
    case GCPB_LOSS_BERNOULLI_ODDS: return 1.0 / (m + 1.0) - x / (m + eps);
    case GCPB_LOSS_GAMMA: return 1.0 / (m + eps) - x / ((m + eps) * (m + eps));
    case GCPB_LOSS_BETA_HALF: {
      const double s = std::sqrt(m + eps);
      return 1.0 / s - x / (s * s * s);
    }
    default: {
      const double r = x - m;
      if (std::fabs(r) <= loss->delta) return -2.0 * r;
      return r > 0.0 ? -2.0 * loss->delta : 2.0 * loss->delta;
    }
  }
}

double gcpb_loss_value(const gcpb_loss* loss, double x, double m) {
  const double eps = 1e-10;
  switch (loss->kind) {
    case GCPB_LOSS_GAUSSIAN: return (x - m) * (x - m);
    case GCPB_LOSS_POISSON: return m - x * std::log(m + eps);
    case GCPB_LOSS_BERNOULLI_ODDS: return std::log(m + 1.0) - x * std::log(m + eps);
    case GCPB_LOSS_GAMMA: return x / (m + eps) + std::log(m + eps);
    case GCPB_LOSS_BETA_HALF: {
      const double s = std::sqrt(m + eps);
      return 2.0 * s + 2.0 * x / s;
    }
    default: {
      const double r = x - m;
      if (std::fabs(r) <= loss->delta) return r * r;
      return 2.0 * loss->delta * std::fabs(r) - loss->delta * loss->delta;
    }
  }
}

}  // extern "C"
