// gcpb_aux.cuh — the kernels around the hot path: stratified zero-candidate
// testing with order-preserving compaction, hash build, Adam, the fp64 loss
// estimate, data generation and small parity helpers.
#pragma once
#include "gcpb_kernels.cuh"

namespace gcpb {

// Device-resident scalar state (one per context).  Living in device memory
// lets whole iterations be captured in a CUDA graph and replayed.
struct DevState {
  // Adam (AdamState + the FitConfig fields adam_step reads)
  int64_t t;  // AdamState::iterations
  int64_t t_saved;
  double lr, beta1, beta2, eps, lb;
  int32_t has_lb;
  uint32_t adam_done;
  // stratified zero sampler (one call)
  int64_t z_q;
  int64_t z_tested, z_accepted, z_rejected;  // RejectionStats, cumulative
  int64_t z_acc_before;                      // accepted before the current batch
  int64_t z_batch_begin, z_batch_size, z_nchunks;
  unsigned long long z_ticket;
  uint32_t z_batch_tag;
  int32_t z_pad;
  double z_total, z_zeta, z_rho;
  int64_t z_status_cap;
  int32_t z_overflow;
  int32_t z_incomplete;  // graph-mode steps whose zero sampler fell short
  uint64_t rng_iter;     // draw-stream iteration base for graph-replayed steps
  uint64_t ref_ctr;      // RefStream counter (draws consumed so far)
  uint32_t ref_flag;     // RefStream: a draw hit the rejection region
  uint32_t ref_pad;
  // multi-rank stratified zero sampler (global state): the
  // z_* fields above then describe this rank's slice of the current batch
  int64_t zg_q, zg_tested, zg_accepted, zg_rejected;
  int64_t zg_kept;   // accepted candidates this rank keeps (its zero-list length)
  int64_t zg_batch;  // global size of the current batch
  int64_t pick_n;    // nonzero-sharded ranks: picks of the global stream in range
  int64_t pick_n2;   // ... of the second pick list (the next step's picks, compacted ahead)
  uint64_t rng_iter_next;  // rng_iter + 1, taken before the exchange kernel advances rng_iter
};

// The next graph-replayed step's iteration, for work queued beside the kernel
// that advances rng_iter (the next step's pick compaction under the exchange).
__global__ void iter_next_kernel(DevState* st) {
  pdl_begin();
  if (threadIdx.x == 0 && blockIdx.x == 0) st->rng_iter_next = st->rng_iter + 1;
}

// Contiguous shard [begin, end) of n items for `rank` of `nranks` -- the
// device twin of gcpb_shard_range (gcpb.cu).
__host__ __device__ __forceinline__ void shard_range_dev(int64_t n, int rank, int nranks,
                                                         int64_t* begin, int64_t* end) {
  const int64_t base = n / nranks, rem = n % nranks;
  const int64_t b = rank * base + (rank < rem ? rank : rem);
  *begin = b;
  *end = b + base + (rank < rem ? 1 : 0);
}


constexpr int kZcThreads = 256;
constexpr int kZcItems = 8;
constexpr int64_t kZcChunk = kZcThreads * kZcItems;

struct ZeroArgs {
  int d;
  uint32_t dims[kMaxModes];
  uint32_t thr[kMaxModes];
  uint64_t stride[kMaxModes];
  int wide;                          // N >= 2^64: 128-bit keys (stride_hi, hkeys_hi)
  uint64_t stride_hi[kMaxModes];
  const uint64_t* hkeys_hi;
  uint64_t seed;
  uint64_t iter;
  const uint64_t* iter_base;  // optional device-resident iteration base
  uint32_t tag;
  const uint64_t* hkeys;
  uint64_t hmask;
  const uint32_t* bloom;  // blocked Bloom prefilter of the keys (nullptr = none)
  uint64_t bmask;         // Bloom blocks - 1
  DevState* st;
  unsigned long long* status;  // per chunk: non-hit count
  uint32_t* tbits;             // per thread of a chunk: non-hit bits | offset << 8
  uint64_t* zero_list;
  int refstream;
  uint64_t ref_key;
  int64_t ref_off;  // draw index of candidate 0's first slot (= picks drawn before)
  uint64_t thr64[kMaxModes];
};

// Batch size of one rejection round, samplers.hpp:118-122, evaluated with
// explicit round-to-nearest ops so it equals the host formula bit for bit.
__host__ __device__ inline int64_t zero_batch_size_dev(double total, double zeta, double rho,
                                                       int64_t shortfall) {
#if defined(__CUDA_ARCH__)
  double b = ceil(__dmul_rn(__dmul_rn(rho, __ddiv_rn(total, zeta)), static_cast<double>(shortfall)));
#else
  double b = std::ceil(rho * (total / zeta) * static_cast<double>(shortfall));
#endif
  if (!(b >= 1.0)) b = 1.0;
  if (b > 9e15) b = 9e15;
  return static_cast<int64_t>(b);
}

// Plans the next rejection batch from the device-resident shortfall.
__global__ void zero_plan_kernel(DevState* st, int first) {
  pdl_begin();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (first) {
    st->z_tested = 0;
    st->z_accepted = 0;
    st->z_rejected = 0;
  }
  const int64_t kept = st->z_accepted < st->z_q ? st->z_accepted : st->z_q;
  const int64_t shortfall = st->z_q - kept;
  st->z_ticket = 0;
  st->z_batch_tag += 1;
  st->z_acc_before = st->z_accepted;
  st->z_batch_begin = st->z_tested;
  if (shortfall <= 0) {
    st->z_batch_size = 0;
    st->z_nchunks = 0;
    return;
  }
  const int64_t batch = zero_batch_size_dev(st->z_total, st->z_zeta, st->z_rho, shortfall);
  int64_t nchunks = (batch + kZcChunk - 1) / kZcChunk;
  if (nchunks > st->z_status_cap) {  // cannot happen: batch shrinks with the shortfall
    st->z_overflow = 1;
    nchunks = 0;
  }
  st->z_batch_size = batch;
  st->z_nchunks = nchunks;
}

// Multi-rank stratified: the host plans the batch; this rank tests the slice
// [begin, begin + size) and collects its accepts (local ranks) from 0.
__global__ void zero_plan_slice_kernel(DevState* st, int64_t begin, int64_t size,
                                       int64_t nchunks) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  st->z_tested = 0;
  st->z_accepted = 0;
  st->z_rejected = 0;
  st->z_acc_before = 0;
  st->z_q = size;
  st->z_ticket = 0;
  st->z_batch_tag += 1;
  st->z_batch_begin = begin;
  st->z_batch_size = size;
  st->z_nchunks = nchunks;
}

// ---- multi-rank stratified zero sampler, device-planned ------
// Every rank plans the same batch from the global shortfall (the reference's
// formula, samplers.hpp:119-121), tests its contiguous slice of the batch's
// candidate ordinals (zero_cand/zero_scatter into a local scratch list, all
// of the slice's accepts kept), then the ranks' accept counts are
// all-gathered (ncclAllGather inside a step graph, or the host communicator)
// and each rank keeps the accepts whose global rank -- candidate order, which
// is rank order since the slices are contiguous -- is below the remaining
// need: exactly the single-rank "first q non-hits" (samplers.hpp:123-132).
__global__ void zero_plan_mr_kernel(DevState* st, int first, int rank, int nranks) {
  pdl_begin();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (first) {
    st->zg_tested = 0;
    st->zg_accepted = 0;
    st->zg_rejected = 0;
    st->zg_kept = 0;
  }
  st->z_ticket = 0;
  st->z_batch_tag += 1;
  st->z_tested = 0;
  st->z_accepted = 0;
  st->z_rejected = 0;
  st->z_acc_before = 0;
  const int64_t kept = st->zg_accepted < st->zg_q ? st->zg_accepted : st->zg_q;
  const int64_t shortfall = st->zg_q - kept;
  st->z_batch_begin = st->zg_tested;
  if (shortfall <= 0) {
    st->zg_batch = 0;
    st->z_batch_size = 0;
    st->z_nchunks = 0;
    st->z_q = 0;
    return;
  }
  const int64_t batch = zero_batch_size_dev(st->z_total, st->z_zeta, st->z_rho, shortfall);
  int64_t lo = 0, hi = 0;
  shard_range_dev(batch, rank, nranks, &lo, &hi);
  int64_t nchunks = (hi - lo + kZcChunk - 1) / kZcChunk;
  if (nchunks > st->z_status_cap) {  // cannot happen: batches shrink with the shortfall
    st->z_overflow = 1;
    nchunks = 0;
  }
  st->zg_batch = batch;
  st->z_batch_begin = st->zg_tested + lo;
  st->z_batch_size = hi - lo;
  st->z_nchunks = nchunks;
  st->z_q = hi - lo;  // the slice's accepts all go to the scratch list
}

__device__ __forceinline__ int64_t zero_keep_mr(const DevState* st, const int64_t* counts,
                                                int rank) {
  int64_t off = 0;
  for (int r = 0; r < rank; ++r) off += counts[r];
  const int64_t need = st->zg_q - (st->zg_accepted < st->zg_q ? st->zg_accepted : st->zg_q);
  const int64_t room = need - off;
  return room <= 0 ? 0 : (counts[rank] < room ? counts[rank] : room);
}

__global__ void zero_keep_mr_kernel(const DevState* st, const int64_t* counts, int rank,
                                    const uint64_t* __restrict__ scratch,
                                    uint64_t* __restrict__ list) {
  pdl_begin();
  const int64_t keep = zero_keep_mr(st, counts, rank);
  const int64_t at = st->zg_kept;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < keep;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    list[at + i] = scratch[i];
}

__global__ void zero_commit_mr_kernel(DevState* st, const int64_t* counts, int rank, int nranks) {
  pdl_begin();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int64_t keep = zero_keep_mr(st, counts, rank);
  int64_t total = 0;
  for (int r = 0; r < nranks; ++r) total += counts[r];
  st->zg_kept += keep;
  st->zg_accepted += total;
  st->zg_tested += st->zg_batch;
  st->zg_rejected += st->zg_batch - total;
}

// Graph mode: counts steps whose device-planned batches fell short of q.
__global__ void zero_check_mr_kernel(DevState* st) {
  pdl_begin();
  if (threadIdx.x == 0 && blockIdx.x == 0 && st->zg_accepted < st->zg_q) st->z_incomplete += 1;
}

// ---- nonzero-sharded picks --------------------------------------------------
// A rank holding nonzero ordinals [nz_begin, nz_end) draws the whole global
// pick stream (the same draws phase_a makes for SEG_PICK, so the sample
// multiset is independent of the rank count) and keeps the picks in its
// range, appended to `list` (block-aggregated; the order only changes the
// gradient's summation order).
struct PickSpec {
  uint64_t seed, iter;
  const uint64_t* iter_base;
  uint32_t tag, thr_eta;
  int64_t p;
  uint64_t eta;
  int64_t nz_begin, nz_end;
  int refstream;
  uint64_t ref_key, thr64_eta;
  const uint64_t* ref_ctr;
  unsigned* ref_flag;
};

// One global pick of the stream (the draw phase_a makes for SEG_PICK).
__device__ __forceinline__ uint64_t pick_draw(const PickSpec& ps, uint64_t it, uint64_t tt) {
  if (ps.refstream)
    return refstream_below(ps.ref_key, *ps.ref_ctr + tt + 1, ps.eta, ps.thr64_eta, ps.ref_flag);
  if (ps.eta <= (1ull << 32)) {
    const U4 b = philox_block(ps.seed, ps.tag, 0u, 0u, it, tt);
    const uint64_t prod = static_cast<uint64_t>(b.x) * ps.eta;
    return (static_cast<uint32_t>(prod) >= ps.thr_eta)
               ? (prod >> 32)
               : bounded32_from(ps.seed, ps.tag, it, tt, 0, ps.eta, ps.thr_eta, 1u);
  }
  return bounded64(ps.seed, ps.tag, it, tt, 0, ps.eta);
}

// Block-aggregated append: a block takes chunks of 256 x kPickItems picks,
// every thread draws kPickItems of them, the kept ones are ranked with a warp
// scan + the warps' totals, and ONE atomic per chunk reserves the block's
// slice of the list.  (A warp-aggregated append made 4e6 atomics on the one
// counter for the 1.28e8 global picks of C5 at 8 ranks: 2.85 ms, bound by the
// same-address atomic rate; the block form is bound by the Philox draws.)
constexpr int kPickItems = 8;  // 4 and 16 measured slower (C5 at 8 ranks: 5.01 / 4.97 / 5.11 ms per step)
__global__ void __launch_bounds__(256) pick_compact_kernel(const PickSpec ps, uint64_t* list,
                                                           int64_t* count) {
  pdl_begin();
  __shared__ unsigned s_warp[8];
  __shared__ unsigned long long s_base;
  const uint64_t it = ps.iter + (ps.iter_base ? *ps.iter_base : 0ull);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int64_t kChunk = 256 * kPickItems;
  for (int64_t c0 = blockIdx.x * kChunk; c0 < ps.p; c0 += static_cast<int64_t>(gridDim.x) * kChunk) {
    uint64_t e[kPickItems];
    unsigned km = 0;
#pragma unroll
    for (int j = 0; j < kPickItems; ++j) {
      const int64_t t = c0 + j * 256 + threadIdx.x;
      e[j] = 0;
      if (t < ps.p) {
        e[j] = pick_draw(ps, it, static_cast<uint64_t>(t));
        if (static_cast<int64_t>(e[j]) >= ps.nz_begin && static_cast<int64_t>(e[j]) < ps.nz_end)
          km |= 1u << j;
      }
    }
    const unsigned cnt = __popc(km);
    unsigned incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned tot = 0;
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        const unsigned v = s_warp[w];
        s_warp[w] = tot;  // exclusive prefix over the warps
        tot += v;
      }
      s_base = tot ? atomicAdd(reinterpret_cast<unsigned long long*>(count),
                               static_cast<unsigned long long>(tot))
                   : 0ull;
    }
    __syncthreads();
    unsigned long long at = s_base + s_warp[warp] + (incl - cnt);
#pragma unroll
    for (int j = 0; j < kPickItems; ++j)
      if (km & (1u << j)) list[at++] = e[j];
    __syncthreads();  // s_warp / s_base are rewritten by the next chunk
  }
}

// Column sums of every factor in fp64 (gradient_poisson_implicit's all-ones
// part, kernels.cpp:213-216): one block per (mode, column).
template <typename T>
__global__ void colsum_kernel(const T* __restrict__ A, const int64_t* off, const int64_t* dims,
                              int rp, int r, double* out) {
  const int k = blockIdx.x / r, j = blockIdx.x % r;
  __shared__ double s[256];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < dims[k]; i += blockDim.x) acc += A[off[k] + i * rp + j];
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[k * r + j] = s[0];
}

// G_k(i, :) += c_k(:) for every row i of every mode (rowwise() +=).
template <typename T>
__global__ void add_rowconst_kernel(T* __restrict__ G, const double* __restrict__ c,
                                    int64_t n, int rp, int r, const int64_t* off, int d) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int col = static_cast<int>(e % rp);
    if (col >= r) continue;
    int k = 0;
    while (k + 1 < d && e >= off[k + 1]) ++k;
    G[e] += static_cast<T>(c[k * r + col]);
  }
}

// Element-wise Welford over trials: mean, M2 (fp64), trial count n (1-based).
template <typename T>
__global__ void welford_kernel(const T* __restrict__ g, double* mean, double* m2, int64_t n_elem,
                               double n) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n_elem;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double x = static_cast<double>(g[e]);
    const double d1 = x - mean[e];
    const double mu = mean[e] + d1 / n;
    m2[e] += d1 * (x - mu);
    mean[e] = mu;
  }
}

// Per-block partial sums of (a - b)^2 and of v (fixed grid).
__global__ void sqdiff_sum_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                  const double* __restrict__ v, int64_t n, double* partials) {
  __shared__ double s1[256], s2[256];
  double x1 = 0.0, x2 = 0.0;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double dd = a[e] - b[e];
    x1 += dd * dd;
    x2 += v[e];
  }
  s1[threadIdx.x] = x1;
  s2[threadIdx.x] = x2;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      s1[threadIdx.x] += s1[threadIdx.x + o];
      s2[threadIdx.x] += s2[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = s1[0];
    partials[2 * blockIdx.x + 1] = s2[0];
  }
}

template <typename T>
__global__ void to_double_kernel(const T* __restrict__ in, double* out, int64_t n) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[e] = static_cast<double>(in[e]);
}

// RefStream: advance the counter by the draws one sampler call consumed:
// fixed + (per_tested ? tested * d : 0)  (stratified: p + tested * d; 2 = the
// multi-rank global tested count).
__global__ void ref_advance_kernel(DevState* st, uint64_t fixed, int per_tested, int d) {
  pdl_begin();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int64_t tested = per_tested == 2 ? st->zg_tested : st->z_tested;
  st->ref_ctr += fixed + (per_tested ? static_cast<uint64_t>(tested) * d : 0ull);
}

// Graph mode: counts steps whose device-planned batches did not yield q zeros.
__global__ void zero_check_kernel(DevState* st) {
  pdl_begin();
  if (threadIdx.x == 0 && blockIdx.x == 0 && st->z_accepted < st->z_q) st->z_incomplete += 1;
}

// Blocked Bloom filter over the nonzero keys (one 32-byte block per key, 3
// bits inside it): a zero candidate — almost every candidate at C3's density
// of 1e-5 — is rejected from one L2-resident sector instead of a random HBM
// probe of the 4-way hash; the ~1 % false positives and the true hits fall
// through to the exact hash lookup.
GCPB_HD uint64_t bloom_hash(uint64_t key) {
  return mix64(key ^ 0x5bd1e9955bd1e995ull);
}
__global__ void bloom_build_kernel(const uint64_t* __restrict__ keys, int64_t n, uint32_t* bloom,
                                   uint64_t bmask) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t h = bloom_hash(keys[e]);
    uint32_t* blk = bloom + (h & bmask) * 8;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const uint32_t pos = static_cast<uint32_t>(h >> (40 + 8 * b)) & 255u;
      atomicOr(blk + (pos >> 5), 1u << (pos & 31u));
    }
  }
}
__device__ __forceinline__ bool bloom_maybe(const uint32_t* __restrict__ bloom, uint64_t bmask,
                                            uint64_t key) {
  const uint64_t h = bloom_hash(key);
  const uint32_t* blk = bloom + (h & bmask) * 8;
  bool all = true;
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    const uint32_t pos = static_cast<uint32_t>(h >> (40 + 8 * b)) & 255u;
    all = all && ((__ldg(blk + (pos >> 5)) >> (pos & 31u)) & 1u);
  }
  return all;
}

// Tests one batch of zero candidates against the nonzero keys (Bloom
// prefilter, then the exact hash) — the reference's "test the whole batch,
// keep the first q non-hits" (samplers.hpp:117-133) in two kernels without an
// inter-block dependency: zero_cand_kernel writes each chunk's non-hit count
// and, per thread, its non-hit bits and offset inside the chunk;
// zero_scatter_kernel ranks them (prefix over the chunk counts) and appends
// the accepted ordinals, in candidate order, to zero_list (ranks < q only).
// DM > 0: the mode count is a compile-time constant (d = 3, 4: every config),
// so the per-mode loops unroll over constant-bank parameters.
template <int DM>
__global__ void __launch_bounds__(kZcThreads) zero_cand_kernel(const ZeroArgs a) {
  pdl_begin();
  const int d = DM > 0 ? DM : a.d;
  __shared__ int s_warp_sum[kZcThreads / 32];
  __shared__ int s_warp_valid[kZcThreads / 32];
  DevState* st = a.st;
  const int64_t nchunks = st->z_nchunks;
  const int64_t bbeg = st->z_batch_begin;
  const int64_t bend = bbeg + st->z_batch_size;
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const uint64_t iter = a.iter + (a.iter_base ? *a.iter_base : 0ull);
  const uint64_t rbase = a.refstream ? st->ref_ctr : 0ull;
  for (int64_t chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
    const int64_t cbeg = bbeg + chunk * kZcChunk + static_cast<int64_t>(threadIdx.x) * kZcItems;
    uint32_t bits = 0;
    int nvalid = 0;
#pragma unroll 1
    for (int j = 0; j < kZcItems; ++j) {
      const int64_t c = cbeg + j;
      if (c >= bend) break;
      ++nvalid;
      uint64_t lin = 0;
      uint32_t ikw[DM > 0 ? DM : kMaxModes];  // per-mode indices (128-bit keys only)
      if (a.refstream) {
        for (int k = 0; k < d; ++k) {
          const uint64_t jj = static_cast<uint64_t>(a.ref_off + c * d + k);
          const uint64_t ik =
              refstream_below(a.ref_key, rbase + jj + 1, a.dims[k], a.thr64[k], &st->ref_flag);
          lin += ik * a.stride[k];
          if (DM == 0) ikw[k] = static_cast<uint32_t>(ik);
        }
      }
#pragma unroll
      for (int g4 = 0; g4 < (DM > 0 ? (DM + 3) / 4 : (kMaxModes + 3) / 4); ++g4) {
        if (a.refstream || g4 * 4 >= d) break;
        const U4 b = philox_block(a.seed, a.tag, static_cast<uint32_t>(g4), 0u, iter,
                                  static_cast<uint64_t>(c));
#pragma unroll
        for (int sl = 0; sl < 4; ++sl) {
          const int k = g4 * 4 + sl;
          if (k >= d) break;
          const uint64_t prod = static_cast<uint64_t>(word_of(b, sl)) * a.dims[k];
          uint32_t ik = (static_cast<uint32_t>(prod) >= a.thr[k])
                            ? static_cast<uint32_t>(prod >> 32)
                            : bounded32_from(a.seed, a.tag, iter, static_cast<uint64_t>(c), k,
                                             a.dims[k], a.thr[k], 1u);
          lin += static_cast<uint64_t>(ik) * a.stride[k];
          if (DM == 0) ikw[k] = ik;
        }
      }
      bool hit;
      if (DM == 0 && a.wide) {  // N >= 2^64 (general-d instantiation only)
        const unsigned __int128 l = wide_lin(ikw, a.stride, a.stride_hi, d);
        const uint64_t lo = static_cast<uint64_t>(l), hi = static_cast<uint64_t>(l >> 64);
        hit = a.hkeys != nullptr &&
              (a.bloom == nullptr || bloom_maybe(a.bloom, a.bmask, wide_digest(lo, hi))) &&
              hash_find_wide(a.hkeys, a.hkeys_hi, a.hmask, lo, hi) >= 0;
      } else {
        hit = a.hkeys != nullptr &&
              (a.bloom == nullptr || bloom_maybe(a.bloom, a.bmask, lin)) &&
              hash_find(a.hkeys, a.hmask, lin) >= 0;
      }
      if (!hit) bits |= 1u << j;
    }
    const int cnt = __popc(bits);
    // block exclusive scan of cnt
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    int vsum = nvalid;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) vsum += __shfl_xor_sync(0xffffffffu, vsum, o);
    if (lane == 31) s_warp_sum[wid] = incl;
    if (lane == 0) s_warp_valid[wid] = vsum;
    __syncthreads();
    int warp_excl = 0, block_total = 0, block_valid = 0;
    for (int w = 0; w < kZcThreads / 32; ++w) {
      if (w < wid) warp_excl += s_warp_sum[w];
      block_total += s_warp_sum[w];
      block_valid += s_warp_valid[w];
    }
    const int thread_excl = warp_excl + incl - cnt;
    a.tbits[chunk * kZcThreads + threadIdx.x] = bits | (static_cast<uint32_t>(thread_excl) << 8);
    if (threadIdx.x == 0) {
      a.status[chunk] = static_cast<unsigned long long>(block_total);
      atomicAdd(reinterpret_cast<unsigned long long*>(&st->z_tested),
                static_cast<unsigned long long>(block_valid));
      atomicAdd(reinterpret_cast<unsigned long long*>(&st->z_accepted),
                static_cast<unsigned long long>(block_total));
      atomicAdd(reinterpret_cast<unsigned long long*>(&st->z_rejected),
                static_cast<unsigned long long>(block_valid - block_total));
    }
    __syncthreads();  // s_warp_* reused by the next chunk
  }
}

__global__ void __launch_bounds__(kZcThreads) zero_scatter_kernel(const ZeroArgs a) {
  pdl_begin();
  __shared__ unsigned long long s_part[kZcThreads / 32];
  DevState* st = a.st;
  const int64_t nchunks = st->z_nchunks;
  const int64_t bbeg = st->z_batch_begin;
  const int64_t acc_before = st->z_acc_before;
  const int64_t q = st->z_q;
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  for (int64_t chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
    unsigned long long part = 0;  // non-hits of the chunks before this one
    for (int64_t i = threadIdx.x; i < chunk; i += kZcThreads) part += a.status[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) s_part[wid] = part;
    __syncthreads();
    unsigned long long excl = 0;
    for (int w = 0; w < kZcThreads / 32; ++w) excl += s_part[w];
    const uint32_t tb = a.tbits[chunk * kZcThreads + threadIdx.x];
    const int64_t cbeg = bbeg + chunk * kZcChunk + static_cast<int64_t>(threadIdx.x) * kZcItems;
    int64_t rank = acc_before + static_cast<int64_t>(excl) + static_cast<int64_t>(tb >> 8);
    for (int j = 0; j < kZcItems; ++j) {
      if ((tb >> j) & 1u) {
        if (rank < q) a.zero_list[rank] = static_cast<uint64_t>(cbeg + j);
        ++rank;
      }
    }
    __syncthreads();  // s_part reused by the next chunk
  }
}

// Open-addressing build (keys unique).
__global__ void hash_build_kernel(const uint64_t* __restrict__ keys, int64_t n,
                                  unsigned long long* tkeys, uint32_t* tvals, uint64_t mask) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const unsigned long long key = keys[e];
    uint64_t b = mix64(key) & mask;
    for (;;) {
      bool done = false;
      for (int s = 0; s < 4; ++s) {
        const unsigned long long prev = atomicCAS(&tkeys[b * 4 + s], ~0ull, key);
        if (prev == ~0ull) {
          tvals[b * 4 + s] = static_cast<uint32_t>(e);
          done = true;
          break;
        }
      }
      if (done) break;
      b = (b + 1) & mask;
    }
  }
}

// Read-then-zero of gradient replicas / hot copies: L2-coherent loads
// (ld.global.cg).  A read-only (.nc) load is NOT ordered against a later
// store to the same address — ptxas schedules it past the store (seen in the
// SASS) — so the re-zeroing pattern must not use __ldg.
__device__ __forceinline__ void load_chunk_cg(const float* p, Vec<float>& out) {
  const float4 q = __ldcg(reinterpret_cast<const float4*>(p));
  out.v[0] = q.x, out.v[1] = q.y, out.v[2] = q.z, out.v[3] = q.w;
}
__device__ __forceinline__ void load_chunk_cg(const double* p, Vec<double>& out) {
  const double2 q = __ldcg(reinterpret_cast<const double2*>(p));
  out.v[0] = q.x, out.v[1] = q.y;
}

// Hot-row copies folded inside the Adam launch (FusedArgs::Ghot): block
// main_blocks + s sums the rh copies of hot slot s and the row's gradient
// replicas in parallel and updates that row; the main blocks skip hot rows.
template <typename T>
struct HotAdam {
  const uint8_t* hslot;
  T* Ghot;
  const int64_t* hot_off;  // element offset of each slot's row
  int rh, n, d;
  uint32_t rowbase[4];
  int64_t off[4];
};

template <typename T>
__device__ __forceinline__ bool hot_chunk(const HotAdam<T>& h, int64_t i0, int rp) {
  int64_t base = h.off[0];
  uint32_t rb = h.rowbase[0];
#pragma unroll
  for (int k = 1; k < 4; ++k)  // static indices keep the parameter arrays in the constant bank
    if (k < h.d && i0 >= h.off[k]) {
      base = h.off[k];
      rb = h.rowbase[k];
    }
  const uint32_t row = static_cast<uint32_t>((i0 - base) / rp);
  return __ldg(h.hslot + rb + row) != 0xFFu;
}

// Sum over the rh copies of hot slot `slot` (and, with reps, the row's nrep
// gradient replicas) of 16-byte chunk c = threadIdx % (rp / VW), re-zeroing
// them: thread (j, c) takes sources j, j + J, ..., four loads in flight, then
// a shared-memory tree combines the J partials.  Valid in threads < rp / VW.
template <typename T>
__device__ __forceinline__ Vec<T> hot_rows_sum(T* __restrict__ Ghot, int slot, int rh, int rp,
                                               T* __restrict__ reps, int nrep,
                                               int64_t rep_stride, int64_t row_off) {
  constexpr int VW = Vec<T>::W;
  __shared__ Vec<T> part[256];
  const int ch = rp / VW;
  const int J = blockDim.x / ch;
  const int c = threadIdx.x % ch;
  const int j0 = threadIdx.x / ch;
  Vec<T> acc;
#pragma unroll
  for (int e = 0; e < VW; ++e) acc.v[e] = static_cast<T>(0);
  const int nsrc = rh + nrep;
  auto src = [&](int j) -> T* {
    return j < rh ? Ghot + (static_cast<int64_t>(slot) * rh + j) * rp + c * VW
                  : reps + (j - rh) * rep_stride + row_off + c * VW;
  };
  if (j0 < J) {
    for (int j = j0; j < nsrc; j += 4 * J) {  // up to four sources' loads in flight
      Vec<T> x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (j + u * J < nsrc) {
          load_chunk_cg(src(j + u * J), x[u]);
        } else {
#pragma unroll
          for (int e = 0; e < VW; ++e) x[u].v[e] = static_cast<T>(0);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (j + u * J < nsrc) {
#pragma unroll
          for (int e = 0; e < VW; ++e) acc.v[e] += x[u].v[e];
          store_chunk(src(j + u * J), Vec<T>{});
        }
      }
    }
  }
  part[threadIdx.x] = acc;
  __syncthreads();
  int Jp = 1;
  while (Jp < J) Jp <<= 1;
  for (int h = Jp >> 1; h > 0; h >>= 1) {
    if (j0 < h && j0 + h < J) {
#pragma unroll
      for (int e = 0; e < VW; ++e) part[threadIdx.x].v[e] += part[threadIdx.x + h * ch].v[e];
    }
    __syncthreads();
  }
  return part[threadIdx.x % (ch > 0 ? ch : 1)];
}

// adam_step (optimizer.cpp:47-66) fused with zeroing the gradient; padding
// columns (j >= r) are left untouched.  With nrep > 0 the gradient is read
// as the sum of the privatized replicas (folding grad_reduce_kernel into the
// update) and the replicas are re-zeroed.  Vectorised: each thread owns one
// 16-byte chunk per array per iteration (rows are padded to 32 bytes, so a
// chunk never straddles rows), two chunks in flight.  The last block advances
// t (and the draw-stream base when advance_rng).
// Interleaved factor/gradient table (AG, rows [A row | G row], pitch 2 rp):
// element i0 of the contiguous layout (column col0 of its row) sits at
// AG + 2 i0 - col0 (factor) and + rp (gradient).
template <typename T>
struct ILTab {
  T* ag;  // null: no interleaved table
  int rp;
  int gcontig;  // 1: the gradient was packed into the contiguous Gr (sharded steps)
};

template <typename T, bool EXTRA = false, bool IL = false>
__device__ __forceinline__ void adam_chunk(T* __restrict__ A, T* __restrict__ Gr,
                                           T* __restrict__ B, T* __restrict__ C, int64_t i0,
                                           int col0, int r, T* __restrict__ reps, int nrep,
                                           int64_t rep_stride, T c1, T c2, T lr, T b1, T b2,
                                           T ob1, T ob2, T eps, bool has_lb, T lb,
                                           Vec<T> extra = Vec<T>{}, ILTab<T> il = ILTab<T>{}) {
  constexpr int VW = Vec<T>::W;
  Vec<T> a, g, b, c;
  // IL: the factors live in AG (A is refreshed from it on demand)
  T* const ila = IL ? il.ag + 2 * i0 - col0 : nullptr;  // this chunk's factor slot in AG
  if (IL) {
    if (!il.gcontig) Gr = ila + il.rp - i0;  // so that Gr + i0 is the chunk's gradient slot
    A = ila - i0;                            // and A + i0 its factor slot
  }
  load_chunk(A + i0, a);
  load_chunk(B + i0, b);
  load_chunk(C + i0, c);
  if (nrep > 0) {
#pragma unroll
    for (int e = 0; e < VW; ++e) g.v[e] = static_cast<T>(0);
    for (int q = 0; q < nrep; q += 4) {  // up to four replicas' loads in flight
      Vec<T> x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (q + u < nrep) {
          load_chunk_cg(reps + (q + u) * rep_stride + i0, x[u]);
        } else {
#pragma unroll
          for (int e = 0; e < VW; ++e) x[u].v[e] = static_cast<T>(0);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (q + u < nrep) {
#pragma unroll
          for (int e = 0; e < VW; ++e) g.v[e] += x[u].v[e];
          store_chunk(reps + (q + u) * rep_stride + i0, Vec<T>{});
        }
      }
    }
  } else {
    load_chunk_cg(Gr + i0, g);
    store_chunk(Gr + i0, Vec<T>{});
  }
  if (EXTRA) {
#pragma unroll
    for (int e = 0; e < VW; ++e) g.v[e] += extra.v[e];
  }
  Vec<T> ao = a, bo = b, co = c;  // padding columns keep their (zero) values
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    if (col0 + e < r) {
      const T gv = g.v[e];
      const T bv = b1 * b.v[e] + ob1 * gv;
      const T cv = b2 * c.v[e] + ob2 * (gv * gv);
      bo.v[e] = bv;
      co.v[e] = cv;
      T av = a.v[e] - lr * (bv / c1) / sqrt((cv / c2) + eps);
      if (has_lb) av = av > lb ? av : lb;
      ao.v[e] = av;
    }
  }
  store_chunk(A + i0, ao);
  store_chunk(B + i0, bo);
  store_chunk(C + i0, co);
}

// IL: factors and gradient are read from the interleaved table il.ag, the
// gradient re-zeroed there and the updated factors written there only (the
// host refreshes A from it when something else needs A).
template <typename T, bool IL = false>
__global__ void __launch_bounds__(256) adam_kernel(T* __restrict__ A, T* __restrict__ Gr,
                                                   T* __restrict__ B, T* __restrict__ C,
                                                   int64_t n, int rp, int r, DevState* st,
                                                   T* __restrict__ reps, int nrep,
                                                   int64_t rep_stride, int advance_rng,
                                                   const HotAdam<T> hot,
                                                   const ILTab<T> il = ILTab<T>{}, int lp = 1) {
  pdl_begin();
  constexpr int VW = Vec<T>::W;
  __shared__ double s_c1, s_c2;
  if (threadIdx.x == 0) {
    const double te = static_cast<double>(st->t + 1);
    s_c1 = 1.0 - pow(st->beta1, te);
    s_c2 = 1.0 - pow(st->beta2, te);
  }
  __syncthreads();
  const T c1 = static_cast<T>(s_c1), c2 = static_cast<T>(s_c2);
  const T lr = static_cast<T>(st->lr);
  const T b1 = static_cast<T>(st->beta1), b2 = static_cast<T>(st->beta2);
  const T ob1 = static_cast<T>(1.0 - st->beta1), ob2 = static_cast<T>(1.0 - st->beta2);
  const T eps = static_cast<T>(st->eps);
  const bool has_lb = st->has_lb != 0;
  const T lb = static_cast<T>(st->lb);
  const uint32_t nchunk = static_cast<uint32_t>(n / VW);  // n < 2^31, multiple of VW
  const int main_blocks = static_cast<int>(gridDim.x) - hot.n;
  const uint32_t stride = static_cast<uint32_t>(main_blocks) * blockDim.x;
  if (static_cast<int>(blockIdx.x) >= main_blocks) {  // one hot row per extra block
    const int slot = static_cast<int>(blockIdx.x) - main_blocks;
    const int64_t row_off = hot.hot_off[slot];
    const Vec<T> hs = hot_rows_sum(hot.Ghot, slot, hot.rh, rp, reps, nrep, rep_stride, row_off);
    if (static_cast<int>(threadIdx.x) < rp / VW)  // gradient = copies + replicas (+ Gr)
      adam_chunk<T, true, IL>(A, Gr, B, C, row_off + threadIdx.x * VW,
                              static_cast<int>(threadIdx.x) * VW, r, nullptr, 0, 0, c1, c2, lr,
                              b1, b2, ob1, ob2, eps, has_lb, lb, hs, il);
  } else if (nrep > 0) {
    // Small problems: the replicas are folded here.  lp lanes share a chunk,
    // each summing (and re-zeroing) replicas j, j + lp, ... with up to four
    // loads in flight, so the fold is one or two L2 round trips instead of
    // nrep / 4 (C2: 32 replicas); a fixed xor-shuffle tree combines them and
    // lane 0 applies the update.
    const uint32_t total = nchunk * static_cast<uint32_t>(lp);
    for (uint32_t t0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; t0 < total; t0 += stride) {
      const uint32_t t = t0 + (threadIdx.x & 31u);
      const bool in = t < total;
      const uint32_t q = t / static_cast<uint32_t>(lp);
      const int j = static_cast<int>(t % static_cast<uint32_t>(lp));
      const int64_t i0 = static_cast<int64_t>(in ? q : 0u) * VW;
      Vec<T> g;
#pragma unroll
      for (int e = 0; e < VW; ++e) g.v[e] = static_cast<T>(0);
      for (int rr = j; in && rr < nrep; rr += 4 * lp) {
        Vec<T> x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (rr + u * lp < nrep) {
            load_chunk_cg(reps + (rr + u * lp) * rep_stride + i0, x[u]);
          } else {
#pragma unroll
            for (int e = 0; e < VW; ++e) x[u].v[e] = static_cast<T>(0);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (rr + u * lp < nrep) {
#pragma unroll
            for (int e = 0; e < VW; ++e) g.v[e] += x[u].v[e];
            store_chunk(reps + (rr + u * lp) * rep_stride + i0, Vec<T>{});
          }
        }
      }
      for (int o = lp / 2; o > 0; o >>= 1) {
#pragma unroll
        for (int e = 0; e < VW; ++e) g.v[e] += __shfl_xor_sync(0xffffffffu, g.v[e], o);
      }
      if (in && j == 0 && (hot.n == 0 || !hot_chunk(hot, i0, rp)))
        adam_chunk<T, true, IL>(A, Gr, B, C, i0, static_cast<int>(i0 % rp), r, nullptr, 0, 0, c1,
                                c2, lr, b1, b2, ob1, ob2, eps, has_lb, lb, g, il);
    }
  } else {
    // Streaming path: U chunks per thread with all 4U loads issued before any
    // use, so enough bytes are in flight to cover HBM latency.
    constexpr int U = 4;
    for (uint32_t q0 = blockIdx.x * blockDim.x + threadIdx.x; q0 < nchunk; q0 += U * stride) {
      Vec<T> a[U], g[U], b[U], c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        uint32_t q = q0 + u * stride;
        q = q < nchunk ? q : nchunk - 1;
        const int64_t i0 = static_cast<int64_t>(q) * VW;
        if (IL) {
          const int64_t col = static_cast<int64_t>((q * VW) % static_cast<uint32_t>(rp));
          load_chunk(il.ag + 2 * i0 - col, a[u]);
          load_chunk_cg(il.gcontig ? Gr + i0 : il.ag + 2 * i0 - col + rp, g[u]);
        } else {
          load_chunk(A + i0, a[u]);
          load_chunk_cg(Gr + i0, g[u]);
        }
        load_chunk(B + i0, b[u]);
        load_chunk(C + i0, c[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t q = q0 + u * stride;
        if (q >= nchunk) break;
        const int64_t i0 = static_cast<int64_t>(q) * VW;
        if (hot.n > 0 && hot_chunk(hot, i0, rp)) continue;  // its hot block updates it
        const int col0 = static_cast<int>((q * VW) % static_cast<uint32_t>(rp));
        Vec<T> ao = a[u], bo = b[u], co = c[u];
#pragma unroll
        for (int e = 0; e < VW; ++e) {
          if (col0 + e < r) {
            const T gv = g[u].v[e];
            const T bv = b1 * b[u].v[e] + ob1 * gv;
            const T cv = b2 * c[u].v[e] + ob2 * (gv * gv);
            bo.v[e] = bv;
            co.v[e] = cv;
            T av = a[u].v[e] - lr * (bv / c1) / sqrt((cv / c2) + eps);
            if (has_lb) av = av > lb ? av : lb;
            ao.v[e] = av;
          }
        }
        if (IL) {
          T* ila = il.ag + 2 * i0 - col0;
          store_chunk(il.gcontig ? Gr + i0 : ila + rp, Vec<T>{});
          store_chunk(ila, ao);
        } else {
          store_chunk(Gr + i0, Vec<T>{});
          store_chunk(A + i0, ao);
        }
        store_chunk(B + i0, bo);
        store_chunk(C + i0, co);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&st->adam_done, 1u);
    if (prev == gridDim.x - 1) {
      st->t += 1;
      if (advance_rng) st->rng_iter += 1;
      st->adam_done = 0;
    }
  }
}

// Streaming adam_step for factor tables in HBM (no gradient replicas; C5):
// the same update as adam_kernel's streaming path, with
// * the per-chunk row arithmetic in 32 bits (cpr = rp / VW chunks per row,
//   a power of two: shifts), the hot-row test one byte of hslot per row;
// * FAST (fp32 only): the bias corrections folded into two scalars and one
//   MUFU reciprocal square root per element,
//     A -= (lr / c1) * B * rsqrt(C * (1 / c2) + eps)
//   (optimizer.cpp:58-62 with its division and sqrt reassociated; fp32
//   contexts are held to 1e-4 against the fp64 reference);
// * NOPAD (r == rp): no padding-column test;
// * U chunks per thread with all loads issued before any use.
// Extra blocks fold the hot rows' copies exactly as adam_kernel does.
template <typename T, bool IL, bool FAST, bool NOPAD, int U, int MINB>
__global__ void __launch_bounds__(256, MINB)
    adam_stream_kernel(T* __restrict__ A, T* __restrict__ Gr, T* __restrict__ B,
                       T* __restrict__ C, int64_t n, int rp, int cpr_shift, int r,
                       DevState* st, int advance_rng, const HotAdam<T> hot,
                       const ILTab<T> il) {
  pdl_begin();
  constexpr int VW = Vec<T>::W;
  __shared__ double s_c1, s_c2;
  if (threadIdx.x == 0) {
    const double te = static_cast<double>(st->t + 1);
    s_c1 = 1.0 - pow(st->beta1, te);
    s_c2 = 1.0 - pow(st->beta2, te);
  }
  __syncthreads();
  const T c1 = static_cast<T>(s_c1), c2 = static_cast<T>(s_c2);
  const T lr = static_cast<T>(st->lr);
  const T b1 = static_cast<T>(st->beta1), b2 = static_cast<T>(st->beta2);
  const T ob1 = static_cast<T>(1.0 - st->beta1), ob2 = static_cast<T>(1.0 - st->beta2);
  const T eps = static_cast<T>(st->eps);
  const bool has_lb = st->has_lb != 0;
  const T lb = static_cast<T>(st->lb);
  const T step = static_cast<T>(st->lr / s_c1);  // FAST: lr / c1
  const T ic2 = static_cast<T>(1.0 / s_c2);       // FAST: 1 / c2
  const uint32_t nchunk = static_cast<uint32_t>(n / VW);
  const int main_blocks = static_cast<int>(gridDim.x) - hot.n;
  const uint32_t stride = static_cast<uint32_t>(main_blocks) * blockDim.x;
  const uint32_t cmask = (1u << cpr_shift) - 1u;
  if (static_cast<int>(blockIdx.x) >= main_blocks) {  // one hot row per extra block
    const int slot = static_cast<int>(blockIdx.x) - main_blocks;
    const int64_t row_off = hot.hot_off[slot];
    const Vec<T> hs = hot_rows_sum(hot.Ghot, slot, hot.rh, rp, static_cast<T*>(nullptr), 0, 0,
                                   row_off);
    if (static_cast<int>(threadIdx.x) < rp / VW)
      adam_chunk<T, true, IL>(A, Gr, B, C, row_off + threadIdx.x * VW,
                              static_cast<int>(threadIdx.x) * VW, r, nullptr, 0, 0, c1, c2, lr,
                              b1, b2, ob1, ob2, eps, has_lb, lb, hs, il);
  } else {
    for (uint32_t q0 = blockIdx.x * blockDim.x + threadIdx.x; q0 < nchunk; q0 += U * stride) {
      Vec<T> a[U], g[U], b[U], c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        uint32_t q = q0 + u * stride;
        q = q < nchunk ? q : nchunk - 1;
        const uint32_t col = (q & cmask) * VW;
        const int64_t i0 = static_cast<int64_t>(q) * VW;
        if (IL) {
          T* ila = il.ag + 2 * i0 - col;
          load_chunk_stream(ila, a[u]);
          load_chunk_stream(il.gcontig ? Gr + i0 : ila + rp, g[u]);
        } else {
          load_chunk_stream(A + i0, a[u]);
          load_chunk_stream(Gr + i0, g[u]);
        }
        load_chunk_stream(B + i0, b[u]);
        load_chunk_stream(C + i0, c[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t q = q0 + u * stride;
        if (q >= nchunk) break;
        if (hot.n > 0 && __ldg(hot.hslot + (q >> cpr_shift)) != 0xFFu) continue;  // hot block
        const uint32_t col = (q & cmask) * VW;
        const int64_t i0 = static_cast<int64_t>(q) * VW;
        Vec<T> ao = a[u], bo = b[u], co = c[u];
#pragma unroll
        for (int e = 0; e < VW; ++e) {
          if (NOPAD || static_cast<int>(col) + e < r) {
            const T gv = g[u].v[e];
            const T bv = b1 * b[u].v[e] + ob1 * gv;
            const T cv = b2 * c[u].v[e] + ob2 * (gv * gv);
            bo.v[e] = bv;
            co.v[e] = cv;
            T av;
            if constexpr (FAST)
              av = a[u].v[e] - step * bv * rsqrtf(cv * ic2 + eps);
            else
              av = a[u].v[e] - lr * (bv / c1) / sqrt((cv / c2) + eps);
            if (has_lb) av = av > lb ? av : lb;
            ao.v[e] = av;
          }
        }
        if (IL) {
          T* ila = il.ag + 2 * i0 - col;
          store_chunk_stream(il.gcontig ? Gr + i0 : ila + rp, Vec<T>{});
          store_chunk_stream(ila, ao);
        } else {
          store_chunk_stream(Gr + i0, Vec<T>{});
          store_chunk_stream(A + i0, ao);
        }
        store_chunk_stream(B + i0, bo);
        store_chunk_stream(C + i0, co);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&st->adam_done, 1u);
    if (prev == gridDim.x - 1) {
      st->t += 1;
      if (advance_rng) st->rng_iter += 1;
      st->adam_done = 0;
    }
  }
}

// ---- multi-GPU: reduce-scatter + sharded Adam + all-gather in one kernel ----
// (the reference's per-worker partial reduction,
// kernels.cpp:148-166, and adam_step, optimizer.cpp:47-66).  Every rank's
// factor/gradient table is mapped into every rank (CUDA IPC over NVLink /
// NVSwitch peer memory, gcpb_peer_open).  Rank `self` owns the global rows
// [row0, row1) (all modes' rows are contiguous: global row i at element
// i * rp of the contiguous layout, i * pitch of the table).  For each chunk
// of its rows it loads the gradient chunk from every peer's table (P2P
// loads), sums them in rank order, re-zeroes them there (P2P stores; only the
// owner touches those addresses in this phase), applies the Adam update with
// its local moments (ZeRO-1: only the owner's moment rows are used), and
// writes the new factor chunk into every peer's table (P2P stores) -- so the
// reduce-scatter, the optimizer and the all-gather are one pass, the
// incoming (gradient) and outgoing (factor) NVLink traffic overlap, and no
// contiguous staging copy of the interleaved table is needed.  The ranks
// synchronise before (all scatters complete) and after (all factor writes
// complete) through the communicator; no kernel waits on another.
constexpr int kMaxPeers = 16;
template <typename T>
struct PeerTabs {
  T* a[kMaxPeers];  // factor row base (row 0) of each rank's table
  T* g[kMaxPeers];  // gradient row base of each rank's table
  int npeers, self;
  int pitch;        // elements between rows of the tables
};

template <typename T, bool FAST>
__global__ void __launch_bounds__(256) peer_adam_kernel(const PeerTabs<T> pt, T* __restrict__ B,
                                                        T* __restrict__ C, int64_t row0,
                                                        int64_t row1, int rp, int cpr_shift,
                                                        int r, DevState* st, int advance_rng) {
  pdl_begin();
  constexpr int VW = Vec<T>::W;
  constexpr int U = 2;  // chunks per thread per pass: U * npeers P2P loads in flight
  __shared__ double s_c1, s_c2;
  if (threadIdx.x == 0) {
    const double te = static_cast<double>(st->t + 1);
    s_c1 = 1.0 - pow(st->beta1, te);
    s_c2 = 1.0 - pow(st->beta2, te);
  }
  __syncthreads();
  const T c1 = static_cast<T>(s_c1), c2 = static_cast<T>(s_c2);
  const T lr = static_cast<T>(st->lr);
  const T b1 = static_cast<T>(st->beta1), b2 = static_cast<T>(st->beta2);
  const T ob1 = static_cast<T>(1.0 - st->beta1), ob2 = static_cast<T>(1.0 - st->beta2);
  const T eps = static_cast<T>(st->eps);
  const bool has_lb = st->has_lb != 0;
  const T lb = static_cast<T>(st->lb);
  const T step = static_cast<T>(st->lr / s_c1);
  const T ic2 = static_cast<T>(1.0 / s_c2);
  const int64_t nch = (row1 - row0) << cpr_shift;
  const int64_t cmask = (int64_t{1} << cpr_shift) - 1;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t q0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q0 < nch;
       q0 += U * stride) {
    Vec<T> g[U];
    int64_t toff[U], coff[U];
    int col[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = q0 + u * stride < nch ? q0 + u * stride : nch - 1;
      const int64_t row = row0 + (q >> cpr_shift);
      col[u] = static_cast<int>(q & cmask) * VW;
      toff[u] = row * pt.pitch + col[u];
      coff[u] = row * rp + col[u];
#pragma unroll
      for (int e = 0; e < VW; ++e) g[u].v[e] = static_cast<T>(0);
    }
    for (int p = 0; p < pt.npeers; ++p) {  // rank order: every replica sees the same sum
      Vec<T> x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) load_chunk_cg(pt.g[p] + toff[u], x[u]);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int e = 0; e < VW; ++e) g[u].v[e] += x[u].v[e];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (q0 + u * stride >= nch) break;
      Vec<T> a, b, c;
      load_chunk_cg(pt.a[pt.self] + toff[u], a);
      load_chunk_cg(B + coff[u], b);
      load_chunk_cg(C + coff[u], c);
      Vec<T> ao = a, bo = b, co = c;
#pragma unroll
      for (int e = 0; e < VW; ++e) {
        if (col[u] + e < r) {
          const T gv = g[u].v[e];
          const T bv = b1 * b.v[e] + ob1 * gv;
          const T cv = b2 * c.v[e] + ob2 * (gv * gv);
          bo.v[e] = bv;
          co.v[e] = cv;
          T av;
          if constexpr (FAST)
            av = a.v[e] - step * bv * rsqrtf(cv * ic2 + eps);
          else
            av = a.v[e] - lr * (bv / c1) / sqrt((cv / c2) + eps);
          if (has_lb) av = av > lb ? av : lb;
          ao.v[e] = av;
        }
      }
      store_chunk(B + coff[u], bo);
      store_chunk(C + coff[u], co);
      for (int p = 0; p < pt.npeers; ++p) {
        store_chunk(pt.g[p] + toff[u], Vec<T>{});
        store_chunk(pt.a[p] + toff[u], ao);
      }
    }
  }
  __threadfence_system();  // peer stores visible before the ranks' barrier
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(&st->adam_done, 1u);
    if (prev == gridDim.x - 1) {
      st->t += 1;
      if (advance_rng) st->rng_iter += 1;
      st->adam_done = 0;
    }
  }
}

// AG <- [A row | 0]: (re)builds the interleaved factor/gradient table from
// the contiguous factors (after any factor write other than the IL Adam).
template <typename T>
__global__ void ag_sync_kernel(const T* __restrict__ A, T* __restrict__ AG, int64_t nchunk,
                               int rp) {
  constexpr int VW = Vec<T>::W;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < nchunk;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i0 = q * VW;
    const int64_t col = i0 % rp;
    Vec<T> a;
    load_chunk(A + i0, a);
    store_chunk(AG + 2 * i0 - col, a);
    store_chunk(AG + 2 * i0 - col + rp, Vec<T>{});
  }
}

// Gr <- AG's gradient rows, which are re-zeroed (sharded steps: the
// all-reduce needs the gradient contiguous).
template <typename T>
__global__ void ag_pack_kernel(T* __restrict__ AG, T* __restrict__ Gr, int64_t nchunk, int rp) {
  pdl_begin();
  constexpr int VW = Vec<T>::W;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < nchunk;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i0 = q * VW;
    T* g = AG + 2 * i0 - i0 % rp + rp;
    Vec<T> v;
    load_chunk_cg(g, v);
    store_chunk(g, Vec<T>{});
    store_chunk(Gr + i0, v);
  }
}

// A <- AG's factor rows (A is stale after interleaved Adam updates).
template <typename T>
__global__ void ag_unsync_kernel(const T* __restrict__ AG, T* __restrict__ A, int64_t nchunk,
                                 int rp) {
  constexpr int VW = Vec<T>::W;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < nchunk;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i0 = q * VW;
    Vec<T> a;
    load_chunk(AG + 2 * i0 - i0 % rp, a);
    store_chunk(A + i0, a);
  }
}

// G = sum of the nrep privatized gradient replicas; replicas re-zeroed.
// Eight lanes per 16-byte chunk, each taking every eighth replica: a lane
// issues all its loads (L2-coherent: the read-then-zero rule above) before the
// zero stores, then the lanes' partial sums meet in a shuffle tree.  (The
// element-per-thread loop this replaces walked the replicas one dependent
// load + store at a time: 115 us for C3's 32 x 512 KB, now a few.)
template <typename T>
__global__ void __launch_bounds__(256) grad_reduce_kernel(T* __restrict__ G, T* __restrict__ reps,
                                                          int64_t nchunks, int nrep,
                                                          int64_t stride) {
  pdl_begin();
  constexpr int VW = Vec<T>::W;
  constexpr int kLanes = 8, kMaxPer = 4;  // up to 32 replicas per pass
  const int sub = threadIdx.x & (kLanes - 1);
  for (int64_t q = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / kLanes;
       q < ((nchunks + 3) & ~int64_t{3});  // whole warps (4 chunks) stay in the shuffles
       q += static_cast<int64_t>(gridDim.x) * blockDim.x / kLanes) {
    const bool live = q < nchunks;
    T acc[VW];
#pragma unroll
    for (int e = 0; e < VW; ++e) acc[e] = static_cast<T>(0);
    for (int r0 = 0; r0 < nrep; r0 += kLanes * kMaxPer) {
      Vec<T> v[kMaxPer];
#pragma unroll
      for (int j = 0; j < kMaxPer; ++j) {
        const int r = r0 + j * kLanes + sub;
        if (live && r < nrep) {
          load_chunk_cg(reps + r * stride + q * VW, v[j]);
        } else {
#pragma unroll
          for (int e = 0; e < VW; ++e) v[j].v[e] = static_cast<T>(0);
        }
      }
      Vec<T> z;
#pragma unroll
      for (int e = 0; e < VW; ++e) z.v[e] = static_cast<T>(0);
#pragma unroll
      for (int j = 0; j < kMaxPer; ++j) {
        const int r = r0 + j * kLanes + sub;
        if (live && r < nrep) store_chunk(reps + r * stride + q * VW, z);
#pragma unroll
        for (int e = 0; e < VW; ++e) acc[e] += v[j].v[e];
      }
    }
#pragma unroll
    for (int o = kLanes / 2; o > 0; o >>= 1)
#pragma unroll
      for (int e = 0; e < VW; ++e) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
    if (live && sub == 0) {
      Vec<T> out;
#pragma unroll
      for (int e = 0; e < VW; ++e) out.v[e] = acc[e];
      store_chunk(G + q * VW, out);
    }
  }
}

// ---------------------------------------------------------------------------
// Hot rows (FusedArgs::hslot / Ghot)
// ---------------------------------------------------------------------------
struct RowBase {
  uint32_t v[kMaxModes];
};

// Per-mode row counts of the stored nonzeros (hist[rowbase[k] + i_k]).  Lanes
// holding the same row are merged with match.any first, so a Zipf-hot row
// costs one atomic per warp instead of up to 32.
__global__ void row_hist_kernel(const uint32_t* __restrict__ rec, int rec_words, int vwd,
                                int64_t n, int d, RowBase rb, uint32_t* __restrict__ hist) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += stride) {
    const uint32_t* r = rec + e * rec_words + vwd;
    for (int k = 0; k < d; ++k) {
      const uint32_t key = rb.v[k] + __ldg(r + k);
      const unsigned peers = __match_any_sync(__activemask(), key);
      if ((threadIdx.x & 31) == static_cast<unsigned>(__ffs(peers) - 1))
        atomicAdd(hist + key, static_cast<uint32_t>(__popc(peers)));
    }
  }
}

// G[row of slot] += sum of the slot's rh copies; copies re-zeroed (the
// gradient consumers other than the fused Adam: stoch_grad, the all-reduce).
template <typename T>
__global__ void __launch_bounds__(256) hot_fold_kernel(T* __restrict__ Ghot, int rh, int rp,
                                                       const int64_t* __restrict__ hot_off,
                                                       T* __restrict__ G, int il = 0) {
  pdl_begin();
  constexpr int VW = Vec<T>::W;
  const Vec<T> acc =
      hot_rows_sum<T>(Ghot, static_cast<int>(blockIdx.x), rh, rp, nullptr, 0, 0, 0);
  if (static_cast<int>(threadIdx.x) < rp / VW) {
    // G: the contiguous gradient, or (il) the interleaved table's gradient rows
    const int64_t ro = il ? 2 * hot_off[blockIdx.x] + rp : hot_off[blockIdx.x];
    T* g = G + ro + threadIdx.x * VW;
#pragma unroll
    for (int e = 0; e < VW; ++e) g[e] += acc.v[e];
  }
}

template <typename T>
struct ModelDesc {
  const T* A;
  int d, rp, r;
  int64_t off[kMaxModes];
};

template <typename T>
__device__ __forceinline__ double model_entry(const ModelDesc<T>& md, const int64_t* idx) {
  T sum = static_cast<T>(0);
  for (int j = 0; j < md.r; ++j) {
    T prod = static_cast<T>(1);
    for (int k = 0; k < md.d; ++k) prod *= md.A[md.off[k] + idx[k] * md.rp + j];
    sum += prod;
  }
  return static_cast<double>(sum);
}

// Fixed-order fp64 partial sums of w * f(x, m) (samplers.cpp:114-124): block
// b owns a fixed contiguous range; deterministic for a fixed grid.
template <typename T>
__global__ void estimate_partial_kernel(const ModelDesc<T> md, const int64_t* __restrict__ idx,
                                        const double* __restrict__ x,
                                        const double* __restrict__ w, int64_t n, int loss,
                                        double delta, double* partials) {
  __shared__ double s[256];
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t beg = static_cast<int64_t>(blockIdx.x) * per;
  const int64_t end = beg + per < n ? beg + per : n;
  double acc = 0.0;
  for (int64_t i = beg + threadIdx.x; i < end; i += blockDim.x) {
    const double m = model_entry(md, idx + i * md.d);
    acc += w[i] * loss_value(loss, delta, x[i], m);
  }
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = s[0];
}

__global__ void sum_partials_kernel(const double* partials, int n, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += partials[i];
    *out = s;
  }
}

// Synthetic dense binary tensor (BASELINE configs[1]): one warp per mode-0
// fiber; x = [u < m/(1+m)], u from the Philox stream at the linear index.
__global__ void gen_bernoulli_kernel(uint8_t* __restrict__ out, int d, const int64_t* dims,
                                     const int64_t* foff, int R, const double* __restrict__ F,
                                     uint64_t seed, int64_t nfibers) {
  extern __shared__ double s_p[];  // [warps][R]
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  double* P = s_p + wid * R;
  const int64_t n0 = dims[0];
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t f = warp0; f < nfibers; f += nwarps) {
    for (int j = lane; j < R; j += 32) {
      double p = 1.0;
      int64_t rem = f;
      for (int k = 1; k < d; ++k) {
        const int64_t ik = rem % dims[k];
        rem /= dims[k];
        p *= F[foff[k] + ik * R + j];
      }
      P[j] = p;
    }
    __syncwarp();
    for (int64_t i0 = lane; i0 < n0; i0 += 32) {
      double m = 0.0;
      for (int j = 0; j < R; ++j) m += F[foff[0] + i0 * R + j] * P[j];
      const double pr = m / (1.0 + m);
      const uint64_t lin = static_cast<uint64_t>(f) * static_cast<uint64_t>(n0) + i0;
      const U4 b = philox_block(seed, TAG_GENERATE, 0u, 0u, 0ull, lin);
      const double u =
          static_cast<double>(((static_cast<uint64_t>(b.x) << 32) | b.y) >> 11) * 0x1.0p-53;
      out[lin] = u < pr ? 1 : 0;
    }
    __syncwarp();
  }
}

// Same tensor as gen_bernoulli_kernel, bit-packed: thread per 32-entry word.
__global__ void gen_bernoulli_bits_kernel(uint32_t* __restrict__ out, int d, const int64_t* dims,
                                          const int64_t* foff, int R,
                                          const double* __restrict__ F, uint64_t seed,
                                          uint64_t total) {
  const uint64_t nwords = (total + 31) / 32;
  for (uint64_t wi = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; wi < nwords;
       wi += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint32_t bits = 0;
    for (int j = 0; j < 32; ++j) {
      const uint64_t lin = wi * 32 + j;
      if (lin >= total) break;
      const int64_t n0 = dims[0];
      const int64_t i0 = static_cast<int64_t>(lin % static_cast<uint64_t>(n0));
      const int64_t f = static_cast<int64_t>(lin / static_cast<uint64_t>(n0));
      double m = 0.0;
      for (int r = 0; r < R; ++r) {
        double p = 1.0;
        int64_t rem = f;
        for (int k = 1; k < d; ++k) {
          const int64_t ik = rem % dims[k];
          rem /= dims[k];
          p *= F[foff[k] + ik * R + r];
        }
        m += F[foff[0] + i0 * R + r] * p;
      }
      const double pr = m / (1.0 + m);
      const U4 b = philox_block(seed, TAG_GENERATE, 0u, 0u, 0ull, lin);
      const double u =
          static_cast<double>(((static_cast<uint64_t>(b.x) << 32) | b.y) >> 11) * 0x1.0p-53;
      if (u < pr) bits |= 1u << j;
    }
    out[wi] = bits;
  }
}

__global__ void popcount_kernel(const uint32_t* __restrict__ w, int64_t n, double* partials) {
  __shared__ double s[256];
  double acc = 0.0;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    acc += __popc(w[e]);
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = s[0];
}

// TensorView::value_at on the device copy (parity helper).
template <typename T>
__global__ void value_at_kernel(const uint64_t* __restrict__ lin, int64_t n, int xkind,
                                const void* dense, const T* vals, const uint64_t* hkeys,
                                const uint32_t* hvals, uint64_t hmask, double* out,
                                const uint64_t* lin_hi = nullptr,
                                const uint64_t* hkeys_hi = nullptr) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t l = lin[e];
    double x = 0.0;
    switch (xkind) {
      case X_DENSE_BIT:
        x = (static_cast<const uint32_t*>(dense)[l >> 5] >> (l & 31u)) & 1u;
        break;
      case X_DENSE_U8:
        x = static_cast<const uint8_t*>(dense)[l];
        break;
      case X_DENSE_F32:
        x = static_cast<const float*>(dense)[l];
        break;
      case X_DENSE_F64:
        x = static_cast<const double*>(dense)[l];
        break;
      default: {
        if (hkeys) {
          const int64_t slot = lin_hi ? hash_find_wide(hkeys, hkeys_hi, hmask, l, lin_hi[e])
                                      : hash_find(hkeys, hmask, l);
          if (slot >= 0) x = static_cast<double>(vals[hvals[slot]]);
        }
      }
    }
    out[e] = x;
  }
}

// Nonzero records from sorted linear keys (multi_index, shape.cpp:98-109) and
// values: [value (T) | coords u32 x d | zero pad] of rec_words words each.
template <typename V, typename T>
__global__ void keys_to_records_kernel(const uint64_t* __restrict__ keys,
                                       const V* __restrict__ vals_in, int64_t n, int d,
                                       const int64_t* dims, uint32_t* rec, int rec_words,
                                       T* vals_out, const uint64_t* __restrict__ keys_hi = nullptr) {
  constexpr int VWD = sizeof(T) / 4;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint32_t* r = rec + e * rec_words;
    const T v = static_cast<T>(vals_in[e]);
    vals_out[e] = v;
    uint32_t vw[2] = {0u, 0u};
    memcpy(vw, &v, sizeof(T));
    for (int w = 0; w < VWD; ++w) r[w] = vw[w];
    if (keys_hi) {  // 128-bit keys (N >= 2^64)
      unsigned __int128 rem = (static_cast<unsigned __int128>(keys_hi[e]) << 64) | keys[e];
      for (int k = 0; k < d; ++k) {
        const unsigned __int128 nk = static_cast<unsigned __int128>(dims[k]);
        r[VWD + k] = static_cast<uint32_t>(rem % nk);
        rem /= nk;
      }
    } else {
      uint64_t rem = keys[e];
      for (int k = 0; k < d; ++k) {
        const uint64_t nk = static_cast<uint64_t>(dims[k]);
        r[VWD + k] = static_cast<uint32_t>(rem % nk);
        rem /= nk;
      }
    }
    for (int w = VWD + d; w < rec_words; ++w) r[w] = 0u;
  }
}

// Validation of device ingest: keys strictly increasing and < N, values != 0.
template <typename V>
__global__ void check_keys_kernel(const uint64_t* __restrict__ keys, const V* __restrict__ vals,
                                  int64_t n, uint64_t total, unsigned* flags) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (keys[e] >= total) atomicOr(flags, 1u);
    if (e > 0 && keys[e - 1] >= keys[e]) atomicOr(flags, 2u);
    if (vals[e] == static_cast<V>(0)) atomicOr(flags, 4u);
  }
}

template <typename V, typename T>
__global__ void convert_kernel(const V* __restrict__ in, T* __restrict__ out, int64_t n) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[e] = static_cast<T>(in[e]);
}

// Sum of squares in fp64 (fixed grid, deterministic per launch geometry).
template <typename V>
__global__ void sumsq_kernel(const V* __restrict__ v, int64_t n, double* partials) {
  __shared__ double s[256];
  double acc = 0.0;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double x = static_cast<double>(v[e]);
    acc += x * x;
  }
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = s[0];
}

// Loss-domain scan of the stored data (loss.cpp:42-62): bit 0 = some x < 0,
// bit 1 = some x not in {0, 1}, bit 2 = NaN.
template <typename V>
__global__ void domain_scan_kernel(const V* __restrict__ v, int64_t n, unsigned* flags) {
  unsigned f = 0;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double x = static_cast<double>(v[e]);
    if (x < 0.0) f |= 1u;
    if (x != 0.0 && x != 1.0) f |= 2u;
    if (x != x) f |= 4u;
  }
  if (f) atomicOr(flags, f);
}

// Factor transfers: unpadded fp64 rows <-> padded device rows (padding
// columns written as zero, so the "padding stays zero" invariant holds).
template <typename T, typename S = double>
__global__ void unpack_rows_kernel(const S* __restrict__ src, T* __restrict__ dst,
                                   int64_t total, int r, int rp) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = i / rp;
    const int col = static_cast<int>(i - row * rp);
    dst[i] = col < r ? static_cast<T>(src[row * r + col]) : static_cast<T>(0);
  }
}

template <typename T, typename S = double>
__global__ void pack_rows_kernel(const T* __restrict__ src, S* __restrict__ dst, int64_t n,
                                 int r, int rp) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = i / r;
    dst[i] = static_cast<S>(src[row * rp + (i - row * r)]);
  }
}

}  // namespace gcpb
