// gcpb_kernels.cuh — device code shared by the fused hot-path kernel and the
// context layer.  See DESIGN.md §4 for the data layout and §5 for the kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <utility>

#include "philox.cuh"

namespace gcpb {

// Programmatic dependent launch (PDL): kernels of one iteration are launched
// with programmatic stream serialisation (launch_k), so the next kernel's
// launch processing overlaps the current one's tail.  Every such kernel
// starts with pdl_begin(), which waits until its predecessor has completed
// and its writes are visible (a no-op when launched without the attribute).
// An explicit early trigger (griddepcontrol.launch_dependents at kernel start,
// GCPB_PDL_TRIGGER=1) was measured slower on every config (C4 step 36.2 ->
// 37.5 us, C2 0.844 -> 0.854 ms: waiting dependents hold SM slots); the
// implicit trigger at block exit gains ~0.6 us per step on C4.
#ifndef GCPB_PDL_TRIGGER
#define GCPB_PDL_TRIGGER 0
#endif
__device__ __forceinline__ void pdl_begin() {
#if GCPB_PDL_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// GCPB_PDL=0 turns programmatic serialisation off.
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("GCPB_PDL");
    return e == nullptr || atoi(e) != 0;
  }();
  return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

constexpr int kMaxModes = 16;
constexpr uint64_t kEmptyKey = ~0ull;

// Checked build (-DGCPB_CHECKED, tools/checked_build.sh): index assertions at
// the gather / scatter sites of the hot path.  A failed check does not trap
// (that would lose the context): it counts into chk[0] and keeps the first
// failing site and value in chk[1], chk[2]; gcpb_debug_check_failures reads
// them and tests/conftest.py asserts zero after every GPU test.
#ifdef GCPB_CHECKED
#define GCPB_CHECK(chk, cond, site, val)                                          \
  do {                                                                            \
    if ((chk) != nullptr && !(cond)) {                                            \
      if (atomicAdd((chk), 1ull) == 0ull) {                                       \
        (chk)[1] = static_cast<unsigned long long>(site);                         \
        (chk)[2] = static_cast<unsigned long long>(val);                          \
      }                                                                           \
    }                                                                             \
  } while (0)
#else
#define GCPB_CHECK(chk, cond, site, val) ((void)0)
#endif

// Data-access kinds for the tensor value x at a sampled index.
enum XKind : int {
  X_NONE = 0,
  X_DENSE_U8 = 1,
  X_DENSE_F32 = 2,
  X_DENSE_F64 = 3,
  X_SPARSE = 4,
  X_DENSE_BIT = 5
};

// Sample-segment kinds of one fused launch (in the reference's sample order).
enum SegKind : int {
  SEG_UNIFORM = 0,    // sample_uniform body (samplers.hpp:87-93): x looked up
  SEG_PICK = 1,       // nonzero picks (samplers.hpp:159-165 / 201-207)
  SEG_DRAW_ZERO = 2,  // semi-stratified unrestricted draws, x = 0 (samplers.hpp:211-216)
  SEG_ZERO_LIST = 3,  // stratified accepted zero candidates (samplers.hpp:169-172)
  SEG_GIVEN = 4,      // host-given samples (parity entry points)
  SEG_FULL = 5,       // every entry, t = linear index (gradient_full, kernels.cpp:170-198)
  SEG_NZ_ALL = 6,     // every stored nonzero, t = ordinal (gradient_poisson_implicit)
};

struct Seg {
  int kind;
  uint32_t tag;
  int flag;          // 1: y = w * (g(x,m) - g(0,m))  (semi nonzero term)
  int pad_;
  int64_t t_begin;   // first sample ordinal handled by this launch
  int64_t t_end;
  int64_t tiles_begin;  // first global tile of this segment
  int64_t out_offset;   // record position of ordinal t_begin
  double weight;
  int64_t ref_off;      // RefStream: draw index of this segment's first draw
  // Device-resident length (multi-rank lists whose length is known only on
  // the device): the segment ends at t_begin + min(t_end - t_begin, *len_dev).
  const int64_t* len_dev;
};

template <typename T>
struct FusedArgs {
  const T* A;  // factors, mode k at A + off[k], row i at + i * pitch
  T* G;        // gradient (or nrep privatized replicas), same layout
  int nrep;          // gradient replicas: block b accumulates into replica b % nrep
  int64_t rep_stride;  // elements between replicas
  int d;
  int rp;      // padded row length (elements)
  int pitch;   // elements between consecutive rows of A (and of G): rp, or 2 * rp
               // when factor and gradient rows are interleaved ([A row | G row])
  int nchunks; // 16-byte chunks holding real columns: ceil(r / VW)
  int loss;
  T delta;
  int64_t off[kMaxModes];
  uint32_t dims[kMaxModes];
  uint32_t thr[kMaxModes];  // Lemire thresholds (2^32 - n_k) mod n_k
  uint64_t stride[kMaxModes];
  // N >= 2^64 (sparse only): 128-bit linear keys, stride_hi the strides' high
  // words, hkeys_hi the membership hash's high words (hash_find_wide)
  int wide;
  uint64_t stride_hi[kMaxModes];
  const uint64_t* hkeys_hi;
  uint64_t seed;
  uint64_t iter;
  const uint64_t* iter_base;  // optional device-resident iteration base (graph replay)
  // tensor access
  int xkind;
  const void* dense;
  const uint32_t* nzrec;  // AoS nonzero records: [value (T) | coords (u32 x d) | pad]
  int rec_words;          // words per record: 4, 8, 16 or 32 (16..128 bytes)
  const T* vals;
  uint64_t eta;        // global nonzero count (pick range)
  uint32_t thr_eta;
  int64_t nz_begin, nz_end;  // global pick ordinals held by this context
  const uint64_t* hkeys;
  const uint32_t* hvals;
  uint64_t hmask;
  // segments
  int nseg;
  Seg seg[3];
  const uint64_t* zero_list;
  // ordered lists (order_build): 32-bit ordinals relative to zl_base, read
  // instead of zero_list when set (half the list traffic; the whole list of a
  // C5 step, 64 MB, stays in L2 between its scatter and its walk)
  const uint32_t* zero_list32;
  uint64_t zl_base;
  // checked builds (GCPB_CHECK): failure counters and the extents the indices
  // are checked against (elements of the factor / gradient table past A and G,
  // entries of the zero list, elements of Ghot); unused otherwise
  unsigned long long* chk;
  int64_t chk_tbl, chk_zl, chk_ghot;
  // optional: SEG_PICK reads its (global) nonzero ordinals from here instead
  // of drawing them (nonzero-sharded ranks: the picks of the global stream
  // that fall in this rank's range, compacted by pick_compact_kernel)
  const uint64_t* pick_list;
  // given samples
  const int64_t* g_idx;
  const double* g_x;
  const double* g_w;
  const int32_t* g_flag;
  const double* g_y;
  // record outputs (device pointers), written when non-null
  int64_t* r_idx;
  double* r_x;
  double* r_w;
  int32_t* r_flag;
  double* r_m;
  double* r_y;
  int scatter;
  int off64;  // host-side: tables beyond 2^31 padded elements -> 64-bit row offsets
  // RefStream mode: draws reproduce the reference's RngStream
  // (rng.cpp:43-61): u = mix64(key + phi * (counter + j + 1)), value u % n,
  // with j the draw's position in the reference's consumption order.
  int refstream;
  uint64_t ref_key;
  const uint64_t* ref_ctr;    // device counter base of this call
  uint64_t thr64[kMaxModes];  // (2^64 - n_k) mod n_k
  uint64_t thr64_eta;
  unsigned* ref_flag;         // set when a draw would have been rejected
  // Hot rows: the most frequent rows of each mode among the
  // nonzeros (C3-C5 draw Zipf-skewed coordinates, so one row can take 12 % of
  // all picks) receive their reductions in rh privatized copies instead of the
  // gradient, which the L2 atomic units would otherwise serialise per address.
  const uint8_t* hslot;         // per row: hot slot within its mode, 0xFF = not hot
  uint32_t rowbase[kMaxModes];  // mode k's rows start at hslot + rowbase[k]
  uint32_t hbase[kMaxModes];    // mode k's first slot in Ghot
  T* Ghot;                      // [slot][rh][rp]
  int rh;                       // copies per hot row (power of two); 0 = off
};

// ---------------------------------------------------------------------------
// Loss f(x,m) and g = df/dm (src/loss.cpp:64-110), eps = 1e-10 shift.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T loss_deriv(int kind, T delta, T x, T m) {
  const T eps = static_cast<T>(1e-10);
  const T one = static_cast<T>(1);
  const T two = static_cast<T>(2);
  switch (kind) {
    case 0:
      return two * (m - x);
    case 1:
      return one - x / (m + eps);
    case 2:
      return one / (m + one) - x / (m + eps);
    case 3:
      return one / (m + eps) - x / ((m + eps) * (m + eps));
    case 4: {
      const T s = sqrt(m + eps);
      return one / s - x / (s * s * s);
    }
    default: {
      const T r = x - m;
      if (fabs(r) <= delta) return -two * r;
      return r > static_cast<T>(0) ? -two * delta : two * delta;
    }
  }
}

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// fp32 derivative with one-MUFU reciprocals (<= 1 ulp); fp64 keeps IEEE
// division (the reference's arithmetic, loss.cpp:88-110).
__device__ __forceinline__ float loss_deriv_fast(int kind, float delta, float x, float m) {
  const float eps = 1e-10f;
  if (kind == 2) return rcp_approx(m + 1.0f) - x * rcp_approx(m + eps);  // bernoulli-odds
  if (kind == 0) return 2.0f * (m - x);                                  // gaussian
  if (kind == 1) return 1.0f - x * rcp_approx(m + eps);                  // poisson
  if (kind == 3) {                                                       // gamma
    const float r = rcp_approx(m + eps);
    return r - x * (r * r);
  }
  if (kind == 4) {  // beta-half
    const float r = rsqrtf(m + eps);
    return r - x * (r * r * r);
  }
  const float rr = x - m;  // huber
  if (fabsf(rr) <= delta) return -2.0f * rr;
  return rr > 0.0f ? -2.0f * delta : 2.0f * delta;
}
__device__ __forceinline__ double loss_deriv_fast(int kind, double delta, double x, double m) {
  return loss_deriv<double>(kind, delta, x, m);
}

__device__ __forceinline__ double loss_value(int kind, double delta, double x, double m) {
  const double eps = 1e-10;
  switch (kind) {
    case 0:
      return (x - m) * (x - m);
    case 1:
      return m - x * log(m + eps);
    case 2:
      return log(m + 1.0) - x * log(m + eps);
    case 3:
      return x / (m + eps) + log(m + eps);
    case 4: {
      const double s = sqrt(m + eps);
      return 2.0 * s + 2.0 * x / s;
    }
    default: {
      const double r = x - m;
      if (fabs(r) <= delta) return r * r;
      return 2.0 * delta * fabs(r) - delta * delta;
    }
  }
}

// ---------------------------------------------------------------------------
// Memory helpers
// ---------------------------------------------------------------------------
template <typename T>
struct Vec;  // one 16-byte chunk
template <>
struct Vec<float> {
  static constexpr int W = 4;
  float v[4];
};
template <>
struct Vec<double> {
  static constexpr int W = 2;
  double v[2];
};

__device__ __forceinline__ void load_chunk(const float* p, Vec<float>& out) {
  const float4 q = __ldg(reinterpret_cast<const float4*>(p));
  out.v[0] = q.x;
  out.v[1] = q.y;
  out.v[2] = q.z;
  out.v[3] = q.w;
}
__device__ __forceinline__ void load_chunk(const double* p, Vec<double>& out) {
  const double2 q = __ldg(reinterpret_cast<const double2*>(p));
  out.v[0] = q.x;
  out.v[1] = q.y;
}

// Streaming (touch-once) chunk loads and stores: no L1 allocation on loads,
// plain stores.
__device__ __forceinline__ void load_chunk_stream(const float* p, Vec<float>& out) {
  asm volatile("ld.global.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(out.v[0]), "=f"(out.v[1]), "=f"(out.v[2]), "=f"(out.v[3])
               : "l"(p));
}
__device__ __forceinline__ void load_chunk_stream(const double* p, Vec<double>& out) {
  asm volatile("ld.global.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(out.v[0]), "=d"(out.v[1])
               : "l"(p));
}
__device__ __forceinline__ void store_chunk_stream(float* p, const Vec<float>& v) {
  asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.v[0]), "f"(v.v[1]),
               "f"(v.v[2]), "f"(v.v[3])
               : "memory");
}
__device__ __forceinline__ void store_chunk_stream(double* p, const Vec<double>& v) {
  asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.v[0]), "d"(v.v[1]) : "memory");
}

__device__ __forceinline__ void store_chunk(float* p, const Vec<float>& v) {
  *reinterpret_cast<float4*>(p) = make_float4(v.v[0], v.v[1], v.v[2], v.v[3]);
}
__device__ __forceinline__ void store_chunk(double* p, const Vec<double>& v) {
  *reinterpret_cast<double2*>(p) = make_double2(v.v[0], v.v[1]);
}

// Scatter-add of one chunk: red.global.add.v4.f32 (one 16-byte vector
// reduction in L2) for fp32, two red.global.add.f64 for fp64.
__device__ __forceinline__ void red_chunk(float* p, const float (&v)[4]) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v[0]), "f"(v[1]),
               "f"(v[2]), "f"(v[3])
               : "memory");
}
__device__ __forceinline__ void red_chunk(double* p, const double (&v)[2]) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v[0]) : "memory");
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p + 1), "d"(v[1]) : "memory");
}

// One 16-byte word of a nonzero record at a random position of the record
// table: a 64-byte L2 fetch instead of the default ~128 bytes per miss
// (tools/fetchgran.cu: same miss rate, half the DRAM bytes; a neighbouring
// record is never wanted), evict-first in L1 and L2 (.cs: a record is used
// once; C5 step 3.548 -> 3.540 ms; .cv, .lu and evict-first cache policies
// measured no better than plain .nc).
__device__ __forceinline__ uint4 ld_record_u4(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.cs.L2::64B.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// Streaming loads of tensor data that should not displace factor rows in L1.
__device__ __forceinline__ uint32_t ld_stream_u8(const uint8_t* p) {
  uint16_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u8 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_stream_f32(const float* p) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_stream_f64(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ ulonglong2 ld_stream_u64x2(const uint64_t* p) {
  ulonglong2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];"
               : "=l"(v.x), "=l"(v.y)
               : "l"(p));
  return v;
}

// One RngStream draw (rng.cpp:43-61) at counter ctr, bounded by n.  The
// reference retries on u < thr (probability thr/2^64 <= n/2^64); this path
// reports it instead, since a retry would shift every later draw.
__device__ __forceinline__ uint64_t refstream_below(uint64_t key, uint64_t ctr, uint64_t n,
                                                   uint64_t thr, unsigned* flag) {
  const uint64_t u = mix64(key + 0x9e3779b97f4a7c15ull * ctr);
  if (u < thr) atomicOr(flag, 1u);
  return u % n;
}

// Open-addressing membership test: 2^b buckets of four u64 keys (one 32-byte
// sector per bucket), linear probing over buckets; slots fill left to right
// so an empty slot ends the probe.  Returns the slot or -1.
__device__ __forceinline__ int64_t hash_find(const uint64_t* __restrict__ keys, uint64_t mask,
                                             uint64_t key) {
  uint64_t b = mix64(key) & mask;
  for (;;) {
    const ulonglong2 q0 = ld_stream_u64x2(keys + b * 4);
    const ulonglong2 q1 = ld_stream_u64x2(keys + b * 4 + 2);
    if (q0.x == key) return static_cast<int64_t>(b * 4);
    if (q0.y == key) return static_cast<int64_t>(b * 4 + 1);
    if (q1.x == key) return static_cast<int64_t>(b * 4 + 2);
    if (q1.y == key) return static_cast<int64_t>(b * 4 + 3);
    if (q0.x == kEmptyKey || q0.y == kEmptyKey || q1.x == kEmptyKey || q1.y == kEmptyKey)
      return -1;
    b = (b + 1) & mask;
  }
}

// 128-bit linear keys (N >= 2^64; shape.hpp:12-14, shape.cpp:87-96).  The
// hash keeps the low words in `keys` (the layout above) and the high words in
// the parallel `keys_hi`; the bucket comes from a 64-bit digest of both.  A
// slot is empty when both words are ~0 (keys stay below 2^127), so a probe
// reads the high word only when the low word matches or is ~0.
GCPB_HD uint64_t wide_digest(uint64_t lo, uint64_t hi) {
  return lo ^ mix64(hi + 0x9e3779b97f4a7c15ull);
}
__device__ __forceinline__ int64_t hash_find_wide(const uint64_t* __restrict__ keys,
                                                  const uint64_t* __restrict__ keys_hi,
                                                  uint64_t mask, uint64_t lo, uint64_t hi) {
  uint64_t b = mix64(wide_digest(lo, hi)) & mask;
  for (;;) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const uint64_t v = keys[b * 4 + s];
      if (v == lo && keys_hi[b * 4 + s] == hi) return static_cast<int64_t>(b * 4 + s);
      if (v == kEmptyKey && keys_hi[b * 4 + s] == kEmptyKey) return -1;
    }
    b = (b + 1) & mask;
  }
}
// Sum_k ik[k] * stride_k in 128 bits (strides as low / high words).
__device__ __forceinline__ unsigned __int128 wide_lin(const uint32_t* ik, const uint64_t* stride,
                                                      const uint64_t* stride_hi, int d) {
  unsigned __int128 l = 0;
  for (int k = 0; k < d; ++k)
    l += static_cast<unsigned __int128>(ik[k]) *
         ((static_cast<unsigned __int128>(stride_hi[k]) << 64) | stride[k]);
  return l;
}

// ---------------------------------------------------------------------------
// Host-facing launcher (instantiated in gcpb_fused_f32.cu / gcpb_fused_f64.cu)
// ---------------------------------------------------------------------------
template <typename T>
cudaError_t launch_fused(const FusedArgs<T>& a, int64_t total_tiles, bool record,
                         cudaStream_t stream, int num_sms, bool* used_hot, int bps_cap = 0);

}  // namespace gcpb
