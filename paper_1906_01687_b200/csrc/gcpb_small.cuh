// gcpb_small.cuh — persistent kernel for small problems (C1-class): many
// iterations of the hot path (uniform draws -> entry -> weighted derivative ->
// MTTKRP -> adam_step, src/optimizer.cpp:116-119) in ONE launch on one cluster.
//
// For small problems (C1: 300 samples, 300 x 5 fp64 factors) a step of the
// graph path is a chain of launches whose gaps dominate (~10 us for 300
// samples).  Here one thread-block cluster runs the whole call: per
// iteration the samples are drawn from the same Philox stream as the fused
// kernel (identical indices), the gradient goes to L2 with red.global, one
// hardware cluster barrier, the Adam update (the adam_kernel arithmetic) on
// every CTA's shared-memory replica of the model.  The tensor gather of the
// NEXT iteration's sample is issued before the barrier, so its latency
// overlaps the Adam phase.
// Results equal the graph path up to floating-point summation order.
// (A one-CTA variant with the model in shared memory was measured slower:
// shared-memory fp64 atomics are CAS loops at ~2 cycles/lane on one SM.)
#pragma once
#include "gcpb_aux.cuh"
#include "gcpb_kernels.cuh"

namespace gcpb {

template <typename T>
struct SmallArgs {
  T* A;
  T* B;
  T* C;
  int64_t nelem;
  int d, r, rp;
  int64_t off[kMaxModes];
  uint32_t dims[kMaxModes];
  uint32_t thr[kMaxModes];
  uint64_t stride[kMaxModes];
  int xkind;
  const void* dense;
  const uint64_t* hkeys;
  const uint32_t* hvals;
  uint64_t hmask;
  const T* vals;
  int loss;
  T delta;
  int64_t s;
  double w;
  uint64_t seed;
  uint32_t tag;
  int64_t n_steps;
  DevState* st;
  // Host-model step (gcpb_step_host on page-locked buffers): the model is
  // read from / written to host memory directly (unpadded fp64 rows, mapped
  // into the device address space) instead of separate copies and pack
  // kernels; the iteration is given (iter_given) rather than device-resident.
  const double* host_in;
  double* host_out;
  int iter_given;
  uint64_t iter;
};

template <typename T, int DM>
__device__ __forceinline__ void small_draw(const SmallArgs<T>& a, uint64_t iter, int64_t t,
                                           uint32_t (&ik)[DM]) {
#pragma unroll
  for (int g4 = 0; g4 < (DM + 3) / 4; ++g4) {
    const U4 b = philox_block(a.seed, a.tag, static_cast<uint32_t>(g4), 0u, iter,
                              static_cast<uint64_t>(t));
#pragma unroll
    for (int sl = 0; sl < 4; ++sl) {
      const int k = g4 * 4 + sl;
      if (k < DM) {
        const uint64_t prod = static_cast<uint64_t>(word_of(b, sl)) * a.dims[k];
        ik[k] = (static_cast<uint32_t>(prod) >= a.thr[k])
                    ? static_cast<uint32_t>(prod >> 32)
                    : bounded32_from(a.seed, a.tag, iter, static_cast<uint64_t>(t), k, a.dims[k],
                                     a.thr[k], 1u);
      }
    }
  }
}

template <typename T, int DM>
__device__ __forceinline__ T small_x(const SmallArgs<T>& a, const uint32_t (&ik)[DM]) {
  uint64_t lin = 0;
#pragma unroll
  for (int k = 0; k < DM; ++k) lin += static_cast<uint64_t>(ik[k]) * a.stride[k];
  switch (a.xkind) {
    case X_DENSE_BIT:
      return static_cast<T>((__ldg(static_cast<const uint32_t*>(a.dense) + (lin >> 5)) >>
                             (lin & 31u)) & 1u);
    case X_DENSE_U8:
      return static_cast<T>(__ldg(static_cast<const uint8_t*>(a.dense) + lin));
    case X_DENSE_F32:
      return static_cast<T>(__ldg(static_cast<const float*>(a.dense) + lin));
    case X_DENSE_F64:
      return static_cast<T>(__ldg(static_cast<const double*>(a.dense) + lin));
    case X_SPARSE: {
      const int64_t slot = hash_find(a.hkeys, a.hmask, lin);
      return slot < 0 ? static_cast<T>(0) : a.vals[a.hvals[slot]];
    }
    default:
      return static_cast<T>(0);
  }
}

__device__ __forceinline__ void cluster_sync_release_acquire() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// One thread-block cluster runs every iteration.  Each CTA keeps a replica
// of A, B, C in shared memory; samples are spread over the cluster's
// threads and their MTTKRP contributions go to L2 with red.global into a
// gradient buffer; ONE hardware cluster barrier (release/acquire) per
// iteration; then every CTA reads the whole gradient and applies the same
// Adam update to its replica (identical inputs and arithmetic -> identical
// replicas), so no second barrier is needed to publish the model.  The
// gradient is triple-buffered: buffer k%3 collects iteration k, and after
// barrier k the cluster zeroes buffer (k+2)%3 (read at k-1, before barrier
// k; next written at k+2, after barrier k+1).
constexpr int kSmallCluster = 8;
constexpr int kSmallThreads = 1024;

template <typename T, int DM>
__global__ void __launch_bounds__(kSmallThreads, 1) small_steps_kernel(const SmallArgs<T> a,
                                                                      T* __restrict__ G3) {
  extern __shared__ __align__(16) unsigned char small_smem[];
  T* sA = reinterpret_cast<T*>(small_smem);
  T* sB = sA + a.nelem;
  T* sC = sB + a.nelem;
  __shared__ double s_corr[4];  // Adam bias corrections, double-buffered by step parity
  const int cta = blockIdx.x, ncta = gridDim.x;  // grid == one cluster
  int64_t nreal = 0;  // real (non-padding) elements: rows x r
  for (int k = 0; k < a.d; ++k) nreal += static_cast<int64_t>(a.dims[k]) * a.r;
  // sample ordinals interleaved over the CTAs, so a few hundred samples
  // still spread over every SM of the cluster
  const int64_t tid = static_cast<int64_t>(threadIdx.x) * ncta + cta;
  const int64_t nth = static_cast<int64_t>(ncta) * blockDim.x;
  if (a.host_in) {
    // padded element e <- host row e / rp, column e % rp; four host reads in
    // flight per thread (each is a round trip over the host link)
    for (int64_t e0 = threadIdx.x; e0 < a.nelem; e0 += 4 * static_cast<int64_t>(blockDim.x)) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t e = e0 + u * static_cast<int64_t>(blockDim.x);
        const int64_t row = e / a.rp, col = e - row * a.rp;
        v[u] = (e < a.nelem && col < a.r) ? a.host_in[row * a.r + col] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t e = e0 + u * static_cast<int64_t>(blockDim.x);
        if (e < a.nelem) sA[e] = static_cast<T>(v[u]);
      }
    }
  }
  for (int64_t e = threadIdx.x; e < a.nelem; e += blockDim.x) {
    if (!a.host_in) sA[e] = a.A[e];
    sB[e] = a.B[e];
    sC[e] = a.C[e];
  }
  const DevState* st = a.st;
  const uint64_t iter0 = a.iter_given ? a.iter : st->rng_iter;
  const int64_t t0 = st->t;
  const T lr = static_cast<T>(st->lr);
  const double beta1 = st->beta1, beta2 = st->beta2;
  const T b1 = static_cast<T>(beta1), b2 = static_cast<T>(beta2);
  const T ob1 = static_cast<T>(1.0 - beta1), ob2 = static_cast<T>(1.0 - beta2);
  const T eps = static_cast<T>(st->eps);
  const bool has_lb = st->has_lb != 0;
  const T lb = static_cast<T>(st->lb);
  const T wv = static_cast<T>(a.w);
  const int64_t zslice = (a.nelem + ncta - 1) / ncta;
  const int64_t z0 = cta * zslice, z1 = min(a.nelem, z0 + zslice);
  uint32_t nik[DM];
  T nx = static_cast<T>(0);
  if (tid < a.s) {
    small_draw<T, DM>(a, iter0, tid, nik);
    nx = small_x<T, DM>(a, nik);
  }
  __syncthreads();
  for (int64_t step = 0; step < a.n_steps; ++step) {
    const uint64_t iter = iter0 + static_cast<uint64_t>(step);
    T* G = G3 + (step % 3) * a.nelem;
    if (threadIdx.x == blockDim.x - 1) {  // a thread with no sample when s is small
      const double te = static_cast<double>(t0 + step + 1);
      s_corr[(step & 1) * 2] = 1.0 - pow(beta1, te);
      s_corr[(step & 1) * 2 + 1] = 1.0 - pow(beta2, te);
    }
    for (int64_t t = tid; t < a.s; t += nth) {
      uint32_t ik[DM];
      T x;
      if (t == tid) {
#pragma unroll
        for (int k = 0; k < DM; ++k) ik[k] = nik[k];
        x = nx;
      } else {
        small_draw<T, DM>(a, iter, t, ik);
        x = small_x<T, DM>(a, ik);
      }
      const T* row[DM];
#pragma unroll
      for (int k = 0; k < DM; ++k) row[k] = sA + a.off[k] + static_cast<int64_t>(ik[k]) * a.rp;
      T m = static_cast<T>(0);  // entry (kruskal.cpp:50-57)
      for (int j = 0; j < a.r; ++j) {
        T p = row[0][j];
#pragma unroll
        for (int k = 1; k < DM; ++k) p = p * row[k][j];
        m += p;
      }
      const T y = wv * loss_deriv_fast(a.loss, a.delta, x, m);
      for (int j = 0; j < a.r; ++j) {  // leave-one-out products (kernels.cpp:21-37)
        T pre[DM];
        T p = static_cast<T>(1);
#pragma unroll
        for (int k = 0; k < DM; ++k) {
          pre[k] = p;
          p = p * row[k][j];
        }
        T suf = static_cast<T>(1);
#pragma unroll
        for (int k = DM - 1; k >= 0; --k) {
          atomicAdd(G + a.off[k] + static_cast<int64_t>(ik[k]) * a.rp + j, y * (pre[k] * suf));
          suf = suf * row[k][j];
        }
      }
    }
    // the next iteration's first sample is model-independent: gather it now
    if (step + 1 < a.n_steps && tid < a.s) {
      small_draw<T, DM>(a, iter + 1, tid, nik);
      nx = small_x<T, DM>(a, nik);
    }
    cluster_sync_release_acquire();
    // adam_step (optimizer.cpp:47-66) on this CTA's replica, t_eff = t + 1;
    // the bias corrections were computed during the sampling phase
    const T c1 = static_cast<T>(s_corr[(step & 1) * 2]), c2 = static_cast<T>(s_corr[(step & 1) * 2 + 1]);
    // real (non-padding) elements q -> (row, col); all gradient loads of a
    // thread are issued before any use (one L2 round trip per iteration)
    constexpr int U = 4;
    for (int64_t q0 = threadIdx.x; q0 < nreal; q0 += U * static_cast<int64_t>(blockDim.x)) {
      T gv[U];
      int64_t ev[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t q = q0 + u * static_cast<int64_t>(blockDim.x);
        const int64_t row = q / a.r;
        ev[u] = row * a.rp + (q - row * a.r);
        gv[u] = q < nreal ? __ldcg(G + ev[u]) : static_cast<T>(0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (q0 + u * static_cast<int64_t>(blockDim.x) >= nreal) break;
        const int64_t e = ev[u];
        const T bv = b1 * sB[e] + ob1 * gv[u];
        const T cv = b2 * sC[e] + ob2 * (gv[u] * gv[u]);
        T av = sA[e] - lr * (bv / c1) / sqrt((cv / c2) + eps);
        if (has_lb) av = av > lb ? av : lb;
        sA[e] = av;
        sB[e] = bv;
        sC[e] = cv;
      }
    }
    T* Gz = G3 + ((step + 2) % 3) * a.nelem;
    for (int64_t e = z0 + threadIdx.x; e < z1; e += blockDim.x) __stcg(Gz + e, static_cast<T>(0));
    __syncthreads();
  }
  cluster_sync_release_acquire();  // every CTA has read the last gradient buffer
  if (a.n_steps > 0) {
    T* Gl = G3 + ((a.n_steps - 1) % 3) * a.nelem;
    for (int64_t e = z0 + threadIdx.x; e < z1; e += blockDim.x) Gl[e] = static_cast<T>(0);
  }
  if (cta == 0) {
    for (int64_t e = threadIdx.x; e < a.nelem; e += blockDim.x) {
      a.A[e] = sA[e];
      a.B[e] = sB[e];
      a.C[e] = sC[e];
    }
    if (a.host_out)
      for (int64_t q = threadIdx.x; q < nreal; q += blockDim.x) {
        const int64_t row = q / a.r;
        a.host_out[q] = static_cast<double>(sA[row * a.rp + (q - row * a.r)]);
      }
    if (threadIdx.x == 0) {
      a.st->t = t0 + a.n_steps;
      if (!a.iter_given) a.st->rng_iter = iter0 + static_cast<uint64_t>(a.n_steps);
    }
  }
}

}  // namespace gcpb
