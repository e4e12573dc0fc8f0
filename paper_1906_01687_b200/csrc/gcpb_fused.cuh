// gcpb_fused.cuh — the hot path: one kernel that samples tensor entries,
// evaluates the Kruskal model at them, applies the weighted loss derivative
// and scatters the d-mode sparse MTTKRP.
//
// Replaces, per sample, the reference's
//   detail::draw_index / next_below       (samplers.hpp:62-68, rng.cpp:51-61)
//   KruskalModel::entry                   (kruskal.cpp:47-58)
//   TensorView::value_at / COO pick       (tensor.hpp:95-97, samplers.hpp:160-164)
//   weight * LossFunction::deriv          (samplers.hpp:83-91,158-172,200-216)
//   LeaveOneOut + accumulate_range        (kernels.cpp:12-57)
// and mttkrp_sampled_all's thread fan-out + partial reduction
// (kernels.cpp:137-168), which becomes red.global vector reductions in L2.
//
// Work decomposition: a warp owns tiles of 32 consecutive
// sample ordinals.  Phase A: lane L draws sample L of a tile (Philox block,
// Lemire bounded draws, tensor value / COO gather) — 32 independent gathers in
// flight per warp; Phase A of tile i+1 is issued before Phase B of tile i so
// its HBM latency overlaps compute.  Phase B: the warp splits into 32/G
// groups of G lanes; in G passes each group takes one sample (broadcast by
// shuffle); lane j owns VPL contiguous 16-byte chunks of every factor row,
// loads the d rows once (the reference gathers them twice: entry + LOO),
// forms prefix products, reduces m over the group with xor-shuffles,
// evaluates y, then walks the suffix products and issues one 16-byte vector
// reduction per (mode, chunk).  Phase B is branch-free around the shuffles
// (invalid samples are masked into zero contributions), so no collective
// re-convergence code is generated.
#pragma once
#include "gcpb_kernels.cuh"

// Minimum resident blocks per SM requested for the common (VPL = 1) kernels;
// caps registers at 65536 / (256 * GCPB_MINB).
#ifndef GCPB_MINB
#define GCPB_MINB 3
#endif

namespace gcpb {

// fp32 derivative with hardware reciprocals (MUFU.RCP + Newton step,
// correctly rounded); fp64 keeps IEEE division (the reference's arithmetic).
__device__ __forceinline__ float loss_deriv_fast(int kind, float delta, float x, float m) {
  const float eps = 1e-10f;
  switch (kind) {
    case 0:
      return 2.0f * (m - x);
    case 1:
      return 1.0f - x * __frcp_rn(m + eps);
    case 2:
      return __frcp_rn(m + 1.0f) - x * __frcp_rn(m + eps);
    case 3: {
      const float r = __frcp_rn(m + eps);
      return r - x * (r * r);
    }
    case 4: {
      const float r = rsqrtf(m + eps);
      return r - x * (r * r * r);
    }
    default: {
      const float rr = x - m;
      if (fabsf(rr) <= delta) return -2.0f * rr;
      return rr > 0.0f ? -2.0f * delta : 2.0f * delta;
    }
  }
}
__device__ __forceinline__ double loss_deriv_fast(int kind, double delta, double x, double m) {
  return loss_deriv<double>(kind, delta, x, m);
}

// Lane-owned slice of a factor row: VPL contiguous 16-byte chunks, of which
// the first `lim` hold real columns (the rest stay zero).  Pairs of chunks
// are fetched with one 256-bit load (LDG.E.256); rows are padded to 32 bytes
// so an even-aligned pair never leaves its row.
template <typename T, int VPL>
__device__ __forceinline__ void load_slice(const T* p, int lim, T (&v)[VPL * Vec<T>::W]) {
  constexpr int VW = Vec<T>::W;
  if constexpr (VPL % 2 == 0 && sizeof(T) == 4) {
#pragma unroll
    for (int c = 0; c < VPL; c += 2) {
      if (c < lim) {
        float* o = reinterpret_cast<float*>(&v[c * VW]);
        asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(o[0]), "=f"(o[1]), "=f"(o[2]), "=f"(o[3]), "=f"(o[4]), "=f"(o[5]),
                       "=f"(o[6]), "=f"(o[7])
                     : "l"(p + c * VW));
      }
    }
  } else {
#pragma unroll
    for (int c = 0; c < VPL; ++c) {
      if (c < lim) {
        Vec<T> q;
        load_chunk(p + c * VW, q);
#pragma unroll
        for (int e = 0; e < VW; ++e) v[c * VW + e] = q.v[e];
      }
    }
  }
}

template <typename T>
struct Drawn {
  bool valid;
  T x;
  double w;
  int flag;
  double yg;
};

template <typename T, int DM>
__device__ __forceinline__ const Seg& seg_of(const FusedArgs<T>& a, int64_t tile) {
  if (a.nseg > 2 && tile >= a.seg[2].tiles_begin) return a.seg[2];
  if (a.nseg > 1 && tile >= a.seg[1].tiles_begin) return a.seg[1];
  return a.seg[0];
}

// Phase A: lane-per-sample draw of ordinal t of segment sg.
template <typename T, int DM>
__device__ __forceinline__ void phase_a(const FusedArgs<T>& a, const Seg& sg, int64_t t,
                                        uint32_t (&ik)[DM], Drawn<T>& s) {
  const int d = a.d;
  s.valid = t < sg.t_end;
  s.x = static_cast<T>(0);
  s.w = sg.weight;
  s.flag = sg.flag;
  s.yg = 0.0;
#pragma unroll
  for (int k = 0; k < DM; ++k) ik[k] = 0;
  if (!s.valid) return;
  const int kind = sg.kind;
  if (kind == SEG_UNIFORM || kind == SEG_DRAW_ZERO || kind == SEG_ZERO_LIST) {
    const uint64_t tt = (kind == SEG_ZERO_LIST) ? a.zero_list[t] : static_cast<uint64_t>(t);
#pragma unroll
    for (int g4 = 0; g4 < (DM + 3) / 4; ++g4) {
      if (g4 * 4 < d) {
        const U4 b = philox_block(a.seed, sg.tag, static_cast<uint32_t>(g4), 0u, a.iter, tt);
#pragma unroll
        for (int sl = 0; sl < 4; ++sl) {
          const int k = g4 * 4 + sl;
          if (k < DM && k < d) {
            const uint64_t prod = static_cast<uint64_t>(word_of(b, sl)) * a.dims[k];
            ik[k] = (static_cast<uint32_t>(prod) >= a.thr[k])
                        ? static_cast<uint32_t>(prod >> 32)
                        : bounded32_from(a.seed, sg.tag, a.iter, tt, k, a.dims[k], a.thr[k], 1u);
          }
        }
      }
    }
    if (kind == SEG_UNIFORM) {
      uint64_t lin = 0;
#pragma unroll
      for (int k = 0; k < DM; ++k)
        if (k < d) lin += static_cast<uint64_t>(ik[k]) * a.stride[k];
      switch (a.xkind) {
        case X_DENSE_U8:
          s.x = static_cast<T>(ld_stream_u8(static_cast<const uint8_t*>(a.dense) + lin));
          break;
        case X_DENSE_F32:
          s.x = static_cast<T>(ld_stream_f32(static_cast<const float*>(a.dense) + lin));
          break;
        case X_DENSE_F64:
          s.x = static_cast<T>(ld_stream_f64(static_cast<const double*>(a.dense) + lin));
          break;
        case X_SPARSE: {
          const int64_t slot = hash_find(a.hkeys, a.hmask, lin);
          s.x = slot < 0 ? static_cast<T>(0) : a.vals[a.hvals[slot]];
          break;
        }
        default:
          break;
      }
    }
  } else if (kind == SEG_PICK) {
    uint64_t e;
    if (a.eta <= (1ull << 32)) {
      const U4 b = philox_block(a.seed, sg.tag, 0u, 0u, a.iter, static_cast<uint64_t>(t));
      const uint64_t prod = static_cast<uint64_t>(b.x) * a.eta;
      e = (static_cast<uint32_t>(prod) >= a.thr_eta)
              ? (prod >> 32)
              : bounded32_from(a.seed, sg.tag, a.iter, static_cast<uint64_t>(t), 0, a.eta,
                               a.thr_eta, 1u);
    } else {
      e = bounded64(a.seed, sg.tag, a.iter, static_cast<uint64_t>(t), 0, a.eta);
    }
    if (static_cast<int64_t>(e) < a.nz_begin || static_cast<int64_t>(e) >= a.nz_end) {
      s.valid = false;
    } else {
      // One aligned record per nonzero: value + coordinates arrive in one
      // 16/32-byte vector load (a single sector for d <= 7 in fp32).
      const int64_t el = static_cast<int64_t>(e) - a.nz_begin;
      constexpr int VWD = sizeof(T) / 4;            // value words
      constexpr int NQ = (VWD + DM + 3) / 4;        // uint4 loads covering value + DM coords
      const uint4* rp = reinterpret_cast<const uint4*>(a.nzrec + el * a.rec_words);
      uint32_t wds[NQ * 4];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (q * 4 < a.rec_words) v = __ldg(rp + q);
        wds[q * 4 + 0] = v.x;
        wds[q * 4 + 1] = v.y;
        wds[q * 4 + 2] = v.z;
        wds[q * 4 + 3] = v.w;
      }
#pragma unroll
      for (int k = 0; k < DM; ++k)
        if (k < d) ik[k] = wds[VWD + k];
      if constexpr (VWD == 1) {
        s.x = __uint_as_float(wds[0]);
      } else {
        s.x = static_cast<T>(__hiloint2double(static_cast<int>(wds[1]), static_cast<int>(wds[0])));
      }
    }
  } else {  // SEG_GIVEN
#pragma unroll
    for (int k = 0; k < DM; ++k)
      if (k < d) ik[k] = static_cast<uint32_t>(a.g_idx[t * d + k]);
    if (a.g_y) {
      s.yg = a.g_y[t];
    } else {
      s.x = static_cast<T>(a.g_x[t]);
      s.w = a.g_w[t];
      s.flag = a.g_flag ? a.g_flag[t] : 0;
    }
  }
}

template <typename T, int DM, int G, int VPL, bool REC>
__device__ __forceinline__ void phase_b(const FusedArgs<T>& a, const Seg& sg, int64_t tile,
                                        const uint32_t (&ik)[DM], const Drawn<T>& s) {
  constexpr int VW = Vec<T>::W;
  constexpr int NGRP = 32 / G;
  constexpr int SL = VPL * VW;  // elements of one lane's row slice
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int grp = lane / G;
  const int gl = lane % G;
  const int d = a.d;
  const bool given = sg.kind == SEG_GIVEN;
  const bool ygiven = given && a.g_y != nullptr;
  const T wseg = static_cast<T>(sg.weight);
  const int chunk0 = gl * VPL;                   // first owned chunk
  const bool owns = chunk0 < a.nchunks;          // lane holds real columns
#pragma unroll 1
  for (int pass = 0; pass < G; ++pass) {
    const int src = pass * NGRP + grp;
    const bool v = __shfl_sync(FULL, s.valid, src);
    uint32_t ii[DM];
#pragma unroll
    for (int k = 0; k < DM; ++k) ii[k] = __shfl_sync(FULL, ik[k], src);
    const T xv = __shfl_sync(FULL, s.x, src);
    T wv = wseg;
    double wd = sg.weight;
    int fv = sg.flag;
    double yg = 0.0;
    if (given) {  // warp-uniform
      wd = __shfl_sync(FULL, s.w, src);
      wv = static_cast<T>(wd);
      fv = __shfl_sync(FULL, s.flag, src);
      yg = __shfl_sync(FULL, s.yg, src);
    }
    const bool act = v && owns;
    T row[DM][SL];
    T pre[DM][SL];
#pragma unroll
    for (int k = 0; k < DM; ++k) {
#pragma unroll
      for (int e = 0; e < SL; ++e) row[k][e] = static_cast<T>(0);
      if (k < d && act)
        load_slice<T, VPL>(a.A + a.off[k] + static_cast<int64_t>(ii[k]) * a.rp + chunk0 * VW,
                           a.nchunks - chunk0, row[k]);
    }
    T mp = static_cast<T>(0);
#pragma unroll
    for (int e = 0; e < SL; ++e) {
      T p = static_cast<T>(1);
#pragma unroll
      for (int k = 0; k < DM; ++k) {
        if (k < d) {
          pre[k][e] = p;
          p = p * row[k][e];
        }
      }
      mp += p;
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) mp += __shfl_xor_sync(FULL, mp, o);
    const T m = mp;
    T y;
    if (ygiven) {
      y = static_cast<T>(yg);
    } else {
      T g = loss_deriv_fast(a.loss, a.delta, xv, m);
      if (fv) g = g - loss_deriv_fast(a.loss, a.delta, static_cast<T>(0), m);
      y = wv * g;
    }
    if (REC) {
      if (v && gl == 0) {
        const int64_t ts = sg.t_begin + (tile - sg.tiles_begin) * 32 + src;
        const int64_t pos = sg.out_offset + (ts - sg.t_begin);
        if (a.r_idx)
          for (int k = 0; k < d; ++k) a.r_idx[pos * d + k] = ii[k];
        if (a.r_x) a.r_x[pos] = static_cast<double>(xv);
        if (a.r_w) a.r_w[pos] = wd;
        if (a.r_flag) a.r_flag[pos] = fv;
        if (a.r_m) a.r_m[pos] = static_cast<double>(m);
        if (a.r_y) a.r_y[pos] = static_cast<double>(y);
      }
    }
    if (a.scatter && act) {
      // Suffix walk: excl_k = prefix_k * suffix_k (kernels.cpp:21-37).
      T suf[SL];
#pragma unroll
      for (int e = 0; e < SL; ++e) suf[e] = static_cast<T>(1);
#pragma unroll
      for (int k = DM - 1; k >= 0; --k) {
        if (k < d) {
          T* gp = a.G + static_cast<int64_t>(blockIdx.x % a.nrep) * a.rep_stride + a.off[k] +
                  static_cast<int64_t>(ii[k]) * a.rp + chunk0 * VW;
#pragma unroll
          for (int c = 0; c < VPL; ++c) {
            T out[VW];
#pragma unroll
            for (int e = 0; e < VW; ++e) out[e] = y * (pre[k][c * VW + e] * suf[c * VW + e]);
            if (chunk0 + c < a.nchunks) red_chunk(gp + c * VW, out);
          }
#pragma unroll
          for (int e = 0; e < SL; ++e) suf[e] = suf[e] * row[k][e];
        }
      }
    }
  }
}

template <typename T, int DM, int G, int VPL, bool REC, int MINB>
__global__ void __launch_bounds__(256, MINB) fused_grad_kernel(const FusedArgs<T> a,
                                                               int64_t total_tiles) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  int64_t tile = warp0;
  if (tile >= total_tiles) return;
  uint32_t ik[DM];
  Drawn<T> s;
  {
    const Seg& sg = seg_of<T, DM>(a, tile);
    phase_a<T, DM>(a, sg, sg.t_begin + (tile - sg.tiles_begin) * 32 + lane, ik, s);
  }
  for (; tile < total_tiles; tile += nwarps) {
    const int64_t next = tile + nwarps;
    uint32_t ik2[DM];
    Drawn<T> s2;
    if (next < total_tiles) {  // prefetch: next tile's draws + tensor gathers in flight
      const Seg& sg2 = seg_of<T, DM>(a, next);
      phase_a<T, DM>(a, sg2, sg2.t_begin + (next - sg2.tiles_begin) * 32 + lane, ik2, s2);
    } else {
      s2.valid = false;
#pragma unroll
      for (int k = 0; k < DM; ++k) ik2[k] = 0;
    }
    const Seg& sg = seg_of<T, DM>(a, tile);
    phase_b<T, DM, G, VPL, REC>(a, sg, tile, ik, s);
#pragma unroll
    for (int k = 0; k < DM; ++k) ik[k] = ik2[k];
    s = s2;
  }
}

// Lane geometry: nchunks 16-byte chunks per row; G lanes per sample, VPL
// contiguous chunks per lane.  Default: VPL = 2 (256-bit loads) when the row
// has >= 4 chunks, else VPL = 1; GCPB_VPL overrides (1 or 2) for tuning.
inline int pow2ceil(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

template <typename T, int DM, bool REC>
cudaError_t launch_fused_dm(const FusedArgs<T>& a, int64_t total_tiles, cudaStream_t stream,
                            int num_sms, int vpl_pref) {
  const int nchunks = a.nchunks;
  int vpl = 1;
  if (!REC && DM <= 4) vpl = vpl_pref;
  int G = pow2ceil((nchunks + vpl - 1) / vpl);
  if (G > 32) {
    G = 32;
    vpl = pow2ceil((nchunks + 31) / 32);
  }
  auto go = [&](auto kern) -> cudaError_t {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
    if (per_sm < 1) per_sm = 1;
    int64_t blocks = (total_tiles + 7) / 8;
    const int64_t cap = static_cast<int64_t>(num_sms) * per_sm;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    kern<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(a, total_tiles);
    return cudaGetLastError();
  };
  if (vpl == 1) {
    switch (G) {
      case 1: return go(fused_grad_kernel<T, DM, 1, 1, REC, GCPB_MINB>);
      case 2: return go(fused_grad_kernel<T, DM, 2, 1, REC, GCPB_MINB>);
      case 4: return go(fused_grad_kernel<T, DM, 4, 1, REC, GCPB_MINB>);
      case 8: return go(fused_grad_kernel<T, DM, 8, 1, REC, GCPB_MINB>);
      case 16: return go(fused_grad_kernel<T, DM, 16, 1, REC, GCPB_MINB>);
      default: return go(fused_grad_kernel<T, DM, 32, 1, REC, GCPB_MINB>);
    }
  }
  if constexpr (!REC && DM <= 4) {
    if (vpl == 2) {
      switch (G) {
        case 1: return go(fused_grad_kernel<T, DM, 1, 2, REC, GCPB_MINB>);
        case 2: return go(fused_grad_kernel<T, DM, 2, 2, REC, GCPB_MINB>);
        case 4: return go(fused_grad_kernel<T, DM, 4, 2, REC, GCPB_MINB>);
        case 8: return go(fused_grad_kernel<T, DM, 8, 2, REC, GCPB_MINB>);
        case 16: return go(fused_grad_kernel<T, DM, 16, 2, REC, GCPB_MINB>);
        default: return go(fused_grad_kernel<T, DM, 32, 2, REC, GCPB_MINB>);
      }
    }
  }
  if (vpl <= 2) return go(fused_grad_kernel<T, DM, 32, 2, REC, 1>);
  if (vpl <= 4) return go(fused_grad_kernel<T, DM, 32, 4, REC, 1>);
  return go(fused_grad_kernel<T, DM, 32, 8, REC, 1>);
}

template <typename T, bool REC>
cudaError_t launch_fused_rec(const FusedArgs<T>& a, int64_t total_tiles, cudaStream_t stream,
                             int num_sms, int vpl_pref) {
  if (a.d <= 3) return launch_fused_dm<T, 3, REC>(a, total_tiles, stream, num_sms, vpl_pref);
  if (a.d == 4) return launch_fused_dm<T, 4, REC>(a, total_tiles, stream, num_sms, vpl_pref);
  if (a.d <= 8) return launch_fused_dm<T, 8, REC>(a, total_tiles, stream, num_sms, vpl_pref);
  return launch_fused_dm<T, 16, REC>(a, total_tiles, stream, num_sms, vpl_pref);
}

template <typename T>
cudaError_t launch_fused(const FusedArgs<T>& a, int64_t total_tiles, bool record,
                         cudaStream_t stream, int num_sms) {
  if (total_tiles <= 0) return cudaSuccess;
  static int vpl_pref = [] {
    const char* e = getenv("GCPB_VPL");
    return e ? (atoi(e) == 2 ? 2 : 1) : 0;
  }();
  int vpl = vpl_pref;
  if (vpl == 0) vpl = 1;  // measured: 256-bit lane slices (vpl 2) cost occupancy
  if (record) return launch_fused_rec<T, true>(a, total_tiles, stream, num_sms, 1);
  return launch_fused_rec<T, false>(a, total_tiles, stream, num_sms, vpl);
}

}  // namespace gcpb
