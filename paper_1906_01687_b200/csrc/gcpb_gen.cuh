// gcpb_gen.cuh — device side of the synthetic problem generators
// (src/synthetic.cpp:26-146), drawing the reference's own RngStream values:
// draw c of a stream is mix64(key + phi * c), so every draw whose counter is
// known in advance is computed in parallel.  Model entries use explicitly
// rounded fp64 multiply/add (no FMA contraction) in the reference's order
// (kruskal.cpp:47-58: j outer, k inner, product from 1.0), so accept/reject
// decisions are bit-identical to the reference.
#pragma once
#include <cstdint>

#include "gcpb_kernels.cuh"

namespace gcpb {

constexpr uint64_t kPhi = 0x9e3779b97f4a7c15ull;

__device__ __forceinline__ double ref_double(uint64_t key, uint64_t ctr) {
  return static_cast<double>(mix64(key + kPhi * ctr) >> 11) * 0x1.0p-53;
}

// truth.entry(idx) over unpadded fp64 factors F (mode k at foff[k], n_k x r).
__device__ __forceinline__ double gen_entry(const int64_t* idx, int d, const int64_t* foff, int r,
                                            const double* __restrict__ F) {
  double sum = 0.0;
  for (int j = 0; j < r; ++j) {
    double prod = 1.0;
    for (int k = 0; k < d; ++k) prod = __dmul_rn(prod, F[foff[k] + idx[k] * r + j]);
    sum = __dadd_rn(sum, prod);
  }
  return sum;
}

// gen_gamma_problem data (synthetic.cpp:33-40): x[lin] = -m * log1p(-u) with
// u the draw at counter c_base + lin + 1, lin first-mode-fastest.
template <typename S>
__global__ void gen_gamma_kernel(S* __restrict__ out, int d, const int64_t* __restrict__ dims,
                                 const int64_t* __restrict__ foff, int r,
                                 const double* __restrict__ F, uint64_t key, uint64_t c_base,
                                 int64_t n) {
  int64_t dm[kMaxModes], fo[kMaxModes];
  for (int k = 0; k < d; ++k) {
    dm[k] = dims[k];
    fo[k] = foff[k];
  }
  for (int64_t lin = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; lin < n;
       lin += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t idx[kMaxModes];
    uint64_t rest = static_cast<uint64_t>(lin);
    for (int k = 0; k < d; ++k) {
      idx[k] = static_cast<int64_t>(rest % static_cast<uint64_t>(dm[k]));
      rest /= static_cast<uint64_t>(dm[k]);
    }
    const double m = gen_entry(idx, d, fo, r, F);
    const double u = ref_double(key, c_base + static_cast<uint64_t>(lin) + 1);
    out[lin] = static_cast<S>(__dmul_rn(-m, log1p(-u)));
  }
}

// True when idx lies in the structural support of some column j' < jmax
// (every mode's factor entry in that column is positive).
__device__ __forceinline__ bool in_support(const int64_t* idx, int d, const int64_t* foff, int r,
                                           const double* __restrict__ F, int jmax) {
  for (int j = 0; j < jmax; ++j) {
    bool all = true;
    for (int k = 0; k < d && all; ++k) all = F[foff[k] + idx[k] * r + j] > 0.0;
    if (all) return true;
  }
  return false;
}

struct BinaryColumnArgs {
  int d, r, j;
  int64_t ssize[kMaxModes];   // support sizes
  int64_t soff[kMaxModes];    // offsets into sup[]
  int64_t foff[kMaxModes];
  int64_t stride[kMaxModes];  // linear-key strides
  int64_t total;              // column_total
};

// Candidate c of column j: mixed radix over the supports, mode 0 fastest
// (synthetic.cpp:98-122).  flags[c] = 1 when c was not a candidate of an
// earlier column (the reference's candidate_set.insert(...).second).
__device__ __forceinline__ void column_candidate(const BinaryColumnArgs& a, const int64_t* sup,
                                                 int64_t c, int64_t* idx) {
  uint64_t rest = static_cast<uint64_t>(c);
  for (int k = 0; k < a.d; ++k) {
    const uint64_t s = static_cast<uint64_t>(a.ssize[k]);
    idx[k] = sup[a.soff[k] + static_cast<int64_t>(rest % s)];
    rest /= s;
  }
}

__global__ void binary_new_kernel(BinaryColumnArgs a, const int64_t* __restrict__ sup,
                                  const double* __restrict__ F, uint32_t* __restrict__ flags) {
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < a.total;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t idx[kMaxModes];
    column_candidate(a, sup, c, idx);
    flags[c] = in_support(idx, a.d, a.foff, a.r, F, a.j) ? 0u : 1u;
  }
}

// New candidates draw u at counter c_base + rank + 1 and become ones when
// u < m / (1 + m) (synthetic.cpp:110-114).
__global__ void binary_accept_kernel(BinaryColumnArgs a, const int64_t* __restrict__ sup,
                                     const double* __restrict__ F,
                                     const uint32_t* __restrict__ flags,
                                     const uint64_t* __restrict__ rank, uint64_t key,
                                     uint64_t c_base, uint64_t* __restrict__ out_keys,
                                     unsigned long long* __restrict__ out_n) {
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < a.total;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (!flags[c]) continue;
    int64_t idx[kMaxModes];
    column_candidate(a, sup, c, idx);
    const double m = gen_entry(idx, a.d, a.foff, a.r, F);
    const double u = ref_double(key, c_base + rank[c] + 1);
    if (u < m / __dadd_rn(1.0, m)) {
      uint64_t lin = 0;
      for (int k = 0; k < a.d; ++k) lin += static_cast<uint64_t>(idx[k] * a.stride[k]);
      out_keys[atomicAdd(out_n, 1ull)] = lin;
    }
  }
}

// Noise placement (synthetic.cpp:129-140): raw draw g (counter c_base + g +
// 1) is a placement attempt when it passes next_below's rejection; it
// places a one unless its key is a structural candidate or an earlier
// attempt took the same key.  First occurrence wins: every attempt records
// its ordinal with atomicMin in an open-addressing table keyed by the
// linear key.
struct NoiseArgs {
  int d, r;
  int64_t dims[kMaxModes];
  int64_t foff[kMaxModes];
  uint64_t n;          // N
  uint64_t threshold;  // (2^64 - N) % N
  uint64_t key, c_base;
  int64_t g0, count;   // attempt ordinals [g0, g0 + count)
  uint64_t mask;       // table capacity - 1
};


__global__ void noise_insert_kernel(NoiseArgs a, const double* __restrict__ F,
                                    uint64_t* __restrict__ tkeys, unsigned long long* __restrict__ tpos,
                                    uint64_t* __restrict__ dkey, uint8_t* __restrict__ ok) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < a.count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t g = static_cast<uint64_t>(a.g0 + i);
    const uint64_t raw = mix64(a.key + kPhi * (a.c_base + g + 1));
    uint8_t st = 0;
    uint64_t lin = 0;
    if (raw >= a.threshold) {
      lin = raw % a.n;
      int64_t idx[kMaxModes];
      uint64_t rest = lin;
      for (int k = 0; k < a.d; ++k) {
        idx[k] = static_cast<int64_t>(rest % static_cast<uint64_t>(a.dims[k]));
        rest /= static_cast<uint64_t>(a.dims[k]);
      }
      if (!in_support(idx, a.d, a.foff, a.r, F, a.r - 1)) {
        st = 1;
        uint64_t s = mix64(lin) & a.mask;
        for (;;) {
          const unsigned long long prev = atomicCAS(reinterpret_cast<unsigned long long*>(tkeys + s),
                                                    static_cast<unsigned long long>(kEmptyKey),
                                                    static_cast<unsigned long long>(lin));
          if (prev == kEmptyKey || prev == lin) break;
          s = (s + 1) & a.mask;
        }
        atomicMin(tpos + s, static_cast<unsigned long long>(g));
      }
    }
    dkey[i] = lin;
    ok[i] = st;
  }
}

__global__ void noise_first_kernel(NoiseArgs a, const uint64_t* __restrict__ tkeys,
                                   const unsigned long long* __restrict__ tpos,
                                   const uint64_t* __restrict__ dkey, const uint8_t* __restrict__ ok,
                                   uint32_t* __restrict__ first) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < a.count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint32_t f = 0;
    if (ok[i]) {
      const uint64_t lin = dkey[i];
      uint64_t s = mix64(lin) & a.mask;
      while (tkeys[s] != lin) s = (s + 1) & a.mask;
      f = tpos[s] == static_cast<unsigned long long>(a.g0 + i) ? 1u : 0u;
    }
    first[i] = f;
  }
}

// Keep the first `need` placements of this batch; report the ordinal of the
// last one kept (the draw that ends the loop) through *last.
__global__ void noise_keep_kernel(int64_t count, const uint32_t* __restrict__ first,
                                  const uint64_t* __restrict__ rank, const uint64_t* __restrict__ dkey,
                                  int64_t need, uint64_t* __restrict__ out_keys,
                                  unsigned long long* __restrict__ out_n,
                                  long long* __restrict__ last) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (!first[i]) continue;
    const int64_t k = static_cast<int64_t>(rank[i]);
    if (k >= need) continue;
    out_keys[atomicAdd(out_n, 1ull)] = dkey[i];
    if (k == need - 1) *last = i;
  }
}

__global__ void u32_to_u64_kernel(const uint32_t* __restrict__ in, uint64_t* __restrict__ out,
                                  int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = in[i];
}

__global__ void fill_f64_kernel(double* __restrict__ out, double v, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = v;
}

}  // namespace gcpb

namespace gcpb {

// ---- SparseTensor normalisation on the device (tensor.cpp:10-41) ----------
// Linear key of each entry (first-mode-fastest); the first out-of-range
// entry in input order is reported through atomicMin so the host can raise
// the reference's check_index message for exactly that entry.
__global__ void coords_to_keys_kernel(const int64_t* __restrict__ coords, int64_t n, int d,
                                      const int64_t* __restrict__ dims, int64_t base,
                                      uint64_t* __restrict__ keys,
                                      unsigned long long* __restrict__ first_bad) {
  int64_t dm[kMaxModes];
  for (int k = 0; k < d; ++k) dm[k] = dims[k];
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint64_t lin = 0, stride = 1;
    bool bad = false;
    for (int k = 0; k < d; ++k) {
      const int64_t v = coords[i * d + k];
      bad |= v < 0 || v >= dm[k];
      lin += static_cast<uint64_t>(v) * stride;
      stride *= static_cast<uint64_t>(dm[k]);
    }
    keys[i] = lin;
    if (bad) atomicMin(first_bad, static_cast<unsigned long long>(base + i));
  }
}

// After a stable sort by key: each run head sums its run left to right (the
// input order, as the host path's stable sort), flags nonzero sums.
__global__ void run_sum_kernel(const uint64_t* __restrict__ keys, const double* __restrict__ vals,
                               int64_t n, double* __restrict__ sums, uint8_t* __restrict__ keep) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = keys[i];
    uint8_t f = 0;
    double s = 0.0;
    if (i == 0 || keys[i - 1] != k) {
      s = vals[i];
      for (int64_t j = i + 1; j < n && keys[j] == k; ++j) s = __dadd_rn(s, vals[j]);
      f = s != 0.0 ? 1 : 0;
    }
    sums[i] = s;
    keep[i] = f;
  }
}

}  // namespace gcpb
