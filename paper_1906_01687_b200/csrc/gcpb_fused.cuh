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
// Work decomposition: a warp owns a tile of 32 consecutive
// sample ordinals.  Phase A: lane L draws sample L of the tile (Philox block,
// Lemire bounded draws, tensor value gather) — 32 independent gathers in
// flight per warp.  Phase B: the warp splits into 32/G groups of G lanes; in G
// passes each group takes one sample (broadcast by shuffle), lane j of the
// group owns 16-byte chunks j, j+G, ... of every factor row, loads the d rows
// once (reference gathers them twice: entry + LOO), forms prefix products,
// reduces m over the group with xor-shuffles, evaluates y, then walks the
// suffix products and issues one 16-byte vector reduction per (mode, chunk).
#pragma once
#include "gcpb_kernels.cuh"

namespace gcpb {

template <typename T, int DM, int G, int VPL, bool REC>
__global__ void __launch_bounds__(256) fused_grad_kernel(const FusedArgs<T> a,
                                                         int64_t total_tiles) {
  constexpr int VW = Vec<T>::W;
  constexpr int NGRP = 32 / G;
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int grp = lane / G;
  const int gl = lane % G;
  const unsigned gmask = (G == 32) ? FULL : (((1u << G) - 1u) << (grp * G));
  const int d = a.d;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;

  for (int64_t tile = warp0; tile < total_tiles; tile += nwarps) {
    // ---- segment of this tile (warp-uniform) ----
    int s = 0;
    if (a.nseg > 1 && tile >= a.seg[1].tiles_begin) s = 1;
    if (a.nseg > 2 && tile >= a.seg[2].tiles_begin) s = 2;
    const Seg sg = (s == 0) ? a.seg[0] : ((s == 1) ? a.seg[1] : a.seg[2]);
    const int64_t t = sg.t_begin + (tile - sg.tiles_begin) * 32 + lane;

    // ---- Phase A: lane-per-sample draw ----
    bool valid = t < sg.t_end;
    uint32_t ik[DM];
#pragma unroll
    for (int k = 0; k < DM; ++k) ik[k] = 0;
    T x = static_cast<T>(0);
    double w = sg.weight;
    int flag = sg.flag;
    double ygiven = 0.0;
    const bool draws_index =
        sg.kind == SEG_UNIFORM || sg.kind == SEG_DRAW_ZERO || sg.kind == SEG_ZERO_LIST;
    if (valid && draws_index) {
      uint64_t tt = static_cast<uint64_t>(t);
      if (sg.kind == SEG_ZERO_LIST) tt = a.zero_list[t];
#pragma unroll
      for (int g4 = 0; g4 < (DM + 3) / 4; ++g4) {
        if (g4 * 4 < d) {
          const U4 b = philox_block(a.seed, sg.tag, static_cast<uint32_t>(g4), 0u, a.iter, tt);
#pragma unroll
          for (int sl = 0; sl < 4; ++sl) {
            const int k = g4 * 4 + sl;
            if (k < DM && k < d) {
              const uint64_t prod = static_cast<uint64_t>(word_of(b, sl)) * a.dims[k];
              if (static_cast<uint32_t>(prod) >= a.thr[k]) {
                ik[k] = static_cast<uint32_t>(prod >> 32);
              } else {
                ik[k] = bounded32_from(a.seed, sg.tag, a.iter, tt, k, a.dims[k], a.thr[k], 1u);
              }
            }
          }
        }
      }
      if (sg.kind == SEG_UNIFORM) {
        uint64_t lin = 0;
#pragma unroll
        for (int k = 0; k < DM; ++k)
          if (k < d) lin += static_cast<uint64_t>(ik[k]) * a.stride[k];
        switch (a.xkind) {
          case X_DENSE_U8:
            x = static_cast<T>(ld_stream_u8(static_cast<const uint8_t*>(a.dense) + lin));
            break;
          case X_DENSE_F32:
            x = static_cast<T>(ld_stream_f32(static_cast<const float*>(a.dense) + lin));
            break;
          case X_DENSE_F64:
            x = static_cast<T>(ld_stream_f64(static_cast<const double*>(a.dense) + lin));
            break;
          case X_SPARSE: {
            const int64_t slot = hash_find(a.hkeys, a.hmask, lin);
            x = slot < 0 ? static_cast<T>(0) : a.vals[a.hvals[slot]];
            break;
          }
          default:
            break;
        }
      }
    } else if (valid && sg.kind == SEG_PICK) {
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
      const int64_t el = static_cast<int64_t>(e) - a.nz_begin;
      if (static_cast<int64_t>(e) < a.nz_begin || static_cast<int64_t>(e) >= a.nz_end) {
        valid = false;
      } else {
#pragma unroll
        for (int k = 0; k < DM; ++k)
          if (k < d) ik[k] = static_cast<uint32_t>(a.coo[k * a.coo_stride + el]);
        x = a.vals[el];
      }
    } else if (valid && sg.kind == SEG_GIVEN) {
#pragma unroll
      for (int k = 0; k < DM; ++k)
        if (k < d) ik[k] = static_cast<uint32_t>(a.g_idx[t * d + k]);
      if (a.g_y) {
        ygiven = a.g_y[t];
      } else {
        x = static_cast<T>(a.g_x[t]);
        w = a.g_w[t];
        flag = a.g_flag ? a.g_flag[t] : 0;
      }
    }

    // ---- Phase B: G lanes per sample ----
#pragma unroll 1
    for (int pass = 0; pass < G; ++pass) {
      const int src = pass * NGRP + grp;
      const bool v = __shfl_sync(FULL, valid, src);
      uint32_t ii[DM];
#pragma unroll
      for (int k = 0; k < DM; ++k) ii[k] = __shfl_sync(FULL, ik[k], src);
      const T xv = __shfl_sync(FULL, x, src);
      const double wv = __shfl_sync(FULL, w, src);
      const int fv = __shfl_sync(FULL, flag, src);
      const double yg = __shfl_sync(FULL, ygiven, src);
      const int64_t ts = __shfl_sync(FULL, t, src);
      if (v) {
        // Gather the d factor rows (each lane: its chunks), prefix products.
        T row[DM][VPL][VW];
        T pre[DM][VPL][VW];
#pragma unroll
        for (int k = 0; k < DM; ++k) {
#pragma unroll
          for (int c = 0; c < VPL; ++c) {
            const int ch = gl + c * G;
            Vec<T> q;
#pragma unroll
            for (int e = 0; e < VW; ++e) q.v[e] = static_cast<T>(0);
            if (k < d && ch < a.nchunks)
              load_chunk(a.A + a.off[k] + static_cast<int64_t>(ii[k]) * a.rp + ch * VW, q);
#pragma unroll
            for (int e = 0; e < VW; ++e) row[k][c][e] = q.v[e];
          }
        }
        T mp = static_cast<T>(0);
#pragma unroll
        for (int c = 0; c < VPL; ++c) {
#pragma unroll
          for (int e = 0; e < VW; ++e) {
            T p = static_cast<T>(1);
#pragma unroll
            for (int k = 0; k < DM; ++k) {
              if (k < d) {
                pre[k][c][e] = p;
                p = p * row[k][c][e];
              }
            }
            mp += p;
          }
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) mp += __shfl_xor_sync(gmask, mp, o);
        const T m = mp;
        T y;
        if (sg.kind == SEG_GIVEN && a.g_y) {
          y = static_cast<T>(yg);
        } else {
          T g = loss_deriv<T>(a.loss, a.delta, xv, m);
          if (fv) g = g - loss_deriv<T>(a.loss, a.delta, static_cast<T>(0), m);
          y = static_cast<T>(wv) * g;
        }
        if (REC) {
          if (gl == 0) {
            const int64_t pos = sg.out_offset + (ts - sg.t_begin);
            if (a.r_idx) {
              for (int k = 0; k < d; ++k) a.r_idx[pos * d + k] = ii[k];
            }
            if (a.r_x) a.r_x[pos] = static_cast<double>(xv);
            if (a.r_w) a.r_w[pos] = wv;
            if (a.r_flag) a.r_flag[pos] = fv;
            if (a.r_m) a.r_m[pos] = static_cast<double>(m);
            if (a.r_y) a.r_y[pos] = static_cast<double>(y);
          }
        }
        if (a.scatter) {
          // Suffix walk: excl_k = prefix_k * suffix_k (kernels.cpp:21-37).
#pragma unroll
          for (int c = 0; c < VPL; ++c) {
            const int ch = gl + c * G;
            if (ch < a.nchunks) {
              T suf[VW];
#pragma unroll
              for (int e = 0; e < VW; ++e) suf[e] = static_cast<T>(1);
#pragma unroll
              for (int k = DM - 1; k >= 0; --k) {
                if (k < d) {
                  T out[VW];
#pragma unroll
                  for (int e = 0; e < VW; ++e) {
                    out[e] = y * (pre[k][c][e] * suf[e]);
                    suf[e] = suf[e] * row[k][c][e];
                  }
                  red_chunk(a.G + a.off[k] + static_cast<int64_t>(ii[k]) * a.rp + ch * VW, out);
                }
              }
            }
          }
        }
      }
    }
  }
}

// Chunk-geometry dispatch: G lanes per sample, VPL chunks per lane.
template <typename T, int DM, bool REC>
cudaError_t launch_fused_dm(const FusedArgs<T>& a, int64_t total_tiles, cudaStream_t stream,
                            int num_sms) {
  const int nchunks = a.nchunks;
  int G = 1;
  while (G < nchunks && G < 32) G <<= 1;
  const int vpl = (nchunks + G - 1) / G;
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
  if (vpl <= 1) {
    switch (G) {
      case 1: return go(fused_grad_kernel<T, DM, 1, 1, REC>);
      case 2: return go(fused_grad_kernel<T, DM, 2, 1, REC>);
      case 4: return go(fused_grad_kernel<T, DM, 4, 1, REC>);
      case 8: return go(fused_grad_kernel<T, DM, 8, 1, REC>);
      case 16: return go(fused_grad_kernel<T, DM, 16, 1, REC>);
      default: return go(fused_grad_kernel<T, DM, 32, 1, REC>);
    }
  }
  if (vpl <= 2) return go(fused_grad_kernel<T, DM, 32, 2, REC>);
  if (vpl <= 4) return go(fused_grad_kernel<T, DM, 32, 4, REC>);
  return go(fused_grad_kernel<T, DM, 32, 8, REC>);
}

template <typename T, bool REC>
cudaError_t launch_fused_rec(const FusedArgs<T>& a, int64_t total_tiles, cudaStream_t stream,
                             int num_sms) {
  if (a.d <= 3) return launch_fused_dm<T, 3, REC>(a, total_tiles, stream, num_sms);
  if (a.d == 4) return launch_fused_dm<T, 4, REC>(a, total_tiles, stream, num_sms);
  if (a.d <= 8) return launch_fused_dm<T, 8, REC>(a, total_tiles, stream, num_sms);
  return launch_fused_dm<T, 16, REC>(a, total_tiles, stream, num_sms);
}

template <typename T>
cudaError_t launch_fused(const FusedArgs<T>& a, int64_t total_tiles, bool record,
                         cudaStream_t stream, int num_sms) {
  if (total_tiles <= 0) return cudaSuccess;
  if (record) return launch_fused_rec<T, true>(a, total_tiles, stream, num_sms);
  return launch_fused_rec<T, false>(a, total_tiles, stream, num_sms);
}

}  // namespace gcpb
