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
// (kernels.cpp:137-168), which becomes red.global vector reductions into
// L2-resident privatized gradient replicas.
//
// Work decomposition: a warp owns tiles of 32 consecutive
// sample ordinals.  Phase A: lane L draws sample L of a tile (Philox block,
// Lemire bounded draws, tensor value / AoS nonzero-record gather) — 32
// independent gathers in flight per warp; Phase A of tile i+1 is issued before
// Phase B of tile i so its HBM latency overlaps compute.  Phase B: the warp
// splits into 32/G groups of G lanes; in G passes each group takes one sample
// (broadcast by shuffle); lane j owns VPL contiguous 16-byte chunks of every
// factor row, loads the d rows once (the reference gathers them twice: entry
// + LOO), forms prefix products, reduces m over the group with xor-shuffles,
// evaluates y, then walks the suffix products and issues one 16-byte vector
// reduction per (mode, chunk).
//
// Phase B has no data-dependent branches: invalid samples (tile tails, picks
// owned by another shard) carry row index 0, lanes beyond the row's last chunk
// load a clamped chunk and are masked out, and only the reductions are
// predicated.  With EXACT the mode count is a compile-time constant (d = 3, 4:
// every BASELINE config), so every per-mode parameter is a constant-bank
// operand.
#pragma once
#include <type_traits>

#include "gcpb_kernels.cuh"

// Minimum resident blocks per SM requested for the common (VPL = 1) kernels;
// caps registers at 65536 / (256 * GCPB_MINB).  Measured: 3 beats 2 and 4.
#ifndef GCPB_MINB
#define GCPB_MINB 3
#endif
// Same for the slim hot-path kernels (no host-given samples, no recording).
#ifndef GCPB_MINB_SLIM
#define GCPB_MINB_SLIM 4
#endif
// Same for the slim hot-row variants (one more live register per sample).
#ifndef GCPB_MINB_HOT
#define GCPB_MINB_HOT 3
#endif
// Same for the three-mode slim hot-row variants (C5: random HBM access, so
// resident warps = loads in flight).
#ifndef GCPB_MINB_HOT3
#define GCPB_MINB_HOT3 3
#endif
// Four-mode hot-row variant with 8-lane groups (C3, r = 32 fp32; L2-reduction
// bound): 4 blocks/SM at 64 registers, measured 202 -> 199 us on C3 (the
// 5/6-lane C4 variant is faster at 3).
#ifndef GCPB_MINB_HOT8
#define GCPB_MINB_HOT8 4
#endif

namespace gcpb {

// Element offset of a factor / gradient row inside its table: 32 bits (one
// register per mode) unless the tables exceed 2^31 padded elements
// (FusedArgs::off64, the OFF64 instantiations).
template <bool OFF64>
using RowOffT = typename std::conditional<OFF64, uint64_t, uint32_t>::type;

template <typename T>
struct Drawn {
  bool valid;
  T x;
  double w;
  int flag;
  double yg;
  uint32_t hs;  // hot slot per mode (8 bits each, 0xFF = not hot); HOT kernels only
};

// Segment fields of one tile, resolved once (not per pass).
struct SegRegs {
  int kind;
  int flag;
  uint32_t tag;
  double weight;
  int64_t t_begin, t_end, tiles_begin, out_offset;
  int64_t ref_off;
};

template <typename T>
__device__ __forceinline__ SegRegs seg_of(const FusedArgs<T>& a, int64_t tile) {
  const int s = (a.nseg > 2 && tile >= a.seg[2].tiles_begin)
                    ? 2
                    : ((a.nseg > 1 && tile >= a.seg[1].tiles_begin) ? 1 : 0);
  const Seg& g = s == 0 ? a.seg[0] : (s == 1 ? a.seg[1] : a.seg[2]);
  SegRegs r;
  r.kind = g.kind;
  r.flag = g.flag;
  r.tag = g.tag;
  r.weight = g.weight;
  r.t_begin = g.t_begin;
  r.t_end = g.t_end;
  r.tiles_begin = g.tiles_begin;
  r.out_offset = g.out_offset;
  r.ref_off = g.ref_off;
  if (g.len_dev) {
    const int64_t n = *g.len_dev;
    if (n < r.t_end - r.t_begin) r.t_end = r.t_begin + (n > 0 ? n : 0);
  }
  return r;
}

// Phase A: lane-per-sample draw of ordinal t of segment sg.
template <typename T, int DM, bool EXACT, bool GV = true, bool HOT = false>
__device__ __forceinline__ void phase_a(const FusedArgs<T>& a, const SegRegs& sg, int64_t t,
                                        uint64_t iter, uint32_t (&ik)[DM], Drawn<T>& s) {
  const int d = EXACT ? DM : a.d;
  s.valid = t < sg.t_end;
  if (HOT) s.hs = 0xFFFFFFFFu;
  s.x = static_cast<T>(0);
  if (GV) {
    s.w = sg.weight;
    s.flag = sg.flag;
    s.yg = 0.0;
  }
#pragma unroll
  for (int k = 0; k < DM; ++k) ik[k] = 0;
  if (!s.valid) return;
  const int kind = sg.kind;
  if (kind == SEG_UNIFORM || kind == SEG_DRAW_ZERO || kind == SEG_ZERO_LIST) {
    if (kind == SEG_ZERO_LIST) GCPB_CHECK(a.chk, t >= 0 && t < a.chk_zl, 1, t);
    const uint64_t tt = (kind == SEG_ZERO_LIST)
                            ? (a.zero_list32 ? a.zl_base + __ldcs(a.zero_list32 + t) : a.zero_list[t])
                            : static_cast<uint64_t>(t);
    if (a.refstream) {  // parity mode: the reference's RngStream sequence
      const uint64_t rbase = *a.ref_ctr;
#pragma unroll
      for (int k = 0; k < DM; ++k)
        if (EXACT || k < d)
          ik[k] = static_cast<uint32_t>(refstream_below(
              a.ref_key, rbase + static_cast<uint64_t>(sg.ref_off) + tt * d + k + 1, a.dims[k],
              a.thr64[k], a.ref_flag));
    }
#pragma unroll
    for (int g4 = 0; g4 < (DM + 3) / 4; ++g4) {
      if (!a.refstream && (EXACT || g4 * 4 < d)) {
        const U4 b = philox_block(a.seed, sg.tag, static_cast<uint32_t>(g4), 0u, iter, tt);
#pragma unroll
        for (int sl = 0; sl < 4; ++sl) {
          const int k = g4 * 4 + sl;
          if (k < DM && (EXACT || k < d)) {
            const uint64_t prod = static_cast<uint64_t>(word_of(b, sl)) * a.dims[k];
            ik[k] = (static_cast<uint32_t>(prod) >= a.thr[k])
                        ? static_cast<uint32_t>(prod >> 32)
                        : bounded32_from(a.seed, sg.tag, iter, tt, k, a.dims[k], a.thr[k], 1u);
          }
        }
      }
    }
    if (kind == SEG_UNIFORM) {
      uint64_t lin = 0;
#pragma unroll
      for (int k = 0; k < DM; ++k)
        if (EXACT || k < d) lin += static_cast<uint64_t>(ik[k]) * a.stride[k];
      switch (a.xkind) {
        case X_DENSE_BIT: {
          const uint32_t w = ld_stream_u32(static_cast<const uint32_t*>(a.dense) + (lin >> 5));
          s.x = static_cast<T>((w >> (lin & 31u)) & 1u);
          break;
        }
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
          int64_t slot;
          if (a.wide) {  // N >= 2^64: 128-bit keys
            const unsigned __int128 l = wide_lin(ik, a.stride, a.stride_hi, d);
            slot = hash_find_wide(a.hkeys, a.hkeys_hi, a.hmask, static_cast<uint64_t>(l),
                                  static_cast<uint64_t>(l >> 64));
          } else {
            slot = hash_find(a.hkeys, a.hmask, lin);
          }
          s.x = slot < 0 ? static_cast<T>(0) : a.vals[a.hvals[slot]];
          break;
        }
        default:
          break;
      }
    }
  } else if (kind == SEG_PICK) {
    uint64_t e;
    if (a.pick_list) {  // drawn beforehand (pick_compact_kernel)
      e = a.pick_list[t];
    } else if (a.refstream) {
      e = refstream_below(a.ref_key, *a.ref_ctr + static_cast<uint64_t>(sg.ref_off + t) + 1, a.eta,
                          a.thr64_eta, a.ref_flag);
    } else if (a.eta <= (1ull << 32)) {
      const U4 b = philox_block(a.seed, sg.tag, 0u, 0u, iter, static_cast<uint64_t>(t));
      const uint64_t prod = static_cast<uint64_t>(b.x) * a.eta;
      e = (static_cast<uint32_t>(prod) >= a.thr_eta)
              ? (prod >> 32)
              : bounded32_from(a.seed, sg.tag, iter, static_cast<uint64_t>(t), 0, a.eta,
                               a.thr_eta, 1u);
    } else {
      e = bounded64(a.seed, sg.tag, iter, static_cast<uint64_t>(t), 0, a.eta);
    }
    if (static_cast<int64_t>(e) < a.nz_begin || static_cast<int64_t>(e) >= a.nz_end) {
      s.valid = false;
    } else {
      // One aligned record per nonzero: value + coordinates arrive in one
      // 16/32-byte vector load (a single sector for d <= 7 in fp32).
      const int64_t el = static_cast<int64_t>(e) - a.nz_begin;
      GCPB_CHECK(a.chk, e < a.eta, 2, e);
      constexpr int VWD = sizeof(T) / 4;      // value words
      constexpr int NQ = (VWD + DM + 3) / 4;  // uint4 loads covering value + DM coords
      const uint4* rp = reinterpret_cast<const uint4*>(a.nzrec + el * a.rec_words);
      uint32_t wds[NQ * 4];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (q * 4 < a.rec_words) v = ld_record_u4(rp + q);
        wds[q * 4 + 0] = v.x;
        wds[q * 4 + 1] = v.y;
        wds[q * 4 + 2] = v.z;
        wds[q * 4 + 3] = v.w;
      }
#pragma unroll
      for (int k = 0; k < DM; ++k)
        if (EXACT || k < d) ik[k] = wds[VWD + k];
      if constexpr (VWD == 1) {
        s.x = __uint_as_float(wds[0]);
      } else {
        s.x = static_cast<T>(__hiloint2double(static_cast<int>(wds[1]), static_cast<int>(wds[0])));
      }
    }
  } else if (GV && (kind == SEG_FULL || kind == SEG_NZ_ALL)) {
    // Exact-gradient walks: every entry (t = first-mode-fastest linear index)
    // or every stored nonzero (t = ordinal); weight 1.
    if (kind == SEG_FULL) {
      uint64_t rem = static_cast<uint64_t>(t);
#pragma unroll
      for (int k = 0; k < DM; ++k)
        if (EXACT || k < d) {
          ik[k] = static_cast<uint32_t>(rem % a.dims[k]);
          rem /= a.dims[k];
        }
      const uint64_t lin = static_cast<uint64_t>(t);
      switch (a.xkind) {
        case X_DENSE_BIT:
          s.x = static_cast<T>((static_cast<const uint32_t*>(a.dense)[lin >> 5] >> (lin & 31u)) & 1u);
          break;
        case X_DENSE_U8:
          s.x = static_cast<T>(static_cast<const uint8_t*>(a.dense)[lin]);
          break;
        case X_DENSE_F32:
          s.x = static_cast<T>(static_cast<const float*>(a.dense)[lin]);
          break;
        case X_DENSE_F64:
          s.x = static_cast<T>(static_cast<const double*>(a.dense)[lin]);
          break;
        case X_SPARSE: {
          const int64_t slot = hash_find(a.hkeys, a.hmask, lin);
          s.x = slot < 0 ? static_cast<T>(0) : a.vals[a.hvals[slot]];
          break;
        }
        default:
          break;
      }
    } else {
      constexpr int VWD = sizeof(T) / 4;
      const uint32_t* rp = a.nzrec + t * a.rec_words;
#pragma unroll
      for (int k = 0; k < DM; ++k)
        if (EXACT || k < d) ik[k] = rp[VWD + k];
      s.x = a.vals[t];
    }
  } else if (GV) {  // SEG_GIVEN
#pragma unroll
    for (int k = 0; k < DM; ++k)
      if (EXACT || k < d) ik[k] = static_cast<uint32_t>(a.g_idx[t * d + k]);
    if (a.g_y) {
      s.yg = a.g_y[t];
    } else {
      s.x = static_cast<T>(a.g_x[t]);
      s.w = a.g_w[t];
      s.flag = a.g_flag ? a.g_flag[t] : 0;
    }
  }
#ifdef GCPB_CHECKED
  if (s.valid) {
#pragma unroll
    for (int k = 0; k < DM; ++k)
      if (EXACT || k < d) GCPB_CHECK(a.chk, ik[k] < a.dims[k], 3, ik[k]);
  }
#endif
  if (HOT && s.valid) {
    static_assert(!HOT || DM <= 4, "hot-row slots pack 8 bits per mode");
    uint32_t hs = 0;
#pragma unroll
    for (int k = 0; k < DM; ++k)
      hs |= static_cast<uint32_t>(__ldg(a.hslot + a.rowbase[k] + ik[k])) << (8 * k);
    s.hs = hs | (DM < 4 ? (0xFFFFFFFFu << (8 * DM)) : 0u);
  }
}

// Reduction target of one (mode, row): the hot-row copy rsel of the row's
// slot when it is hot, else the block's gradient replica.
template <typename T, bool HOT, typename RowOff>
__device__ __forceinline__ T* grad_row(const FusedArgs<T>& a, T* Gb, RowOff roff, uint32_t hsv,
                                       int k, uint32_t rsel) {
  if (HOT) {
    const uint32_t sl = (hsv >> (8 * k)) & 0xFFu;
    if (sl != 0xFFu) {
      GCPB_CHECK(a.chk,
                 static_cast<int64_t>((a.hbase[k] + sl) * static_cast<uint32_t>(a.rh) + rsel + 1) *
                         a.rp <= a.chk_ghot && rsel < static_cast<uint32_t>(a.rh),
                 5, sl);
      return a.Ghot + ((a.hbase[k] + sl) * static_cast<uint32_t>(a.rh) + rsel) *
                          static_cast<uint32_t>(a.rp);
    }
  }
  return Gb + roff;
}

template <typename T, int DM, bool EXACT, int G, int VPL, bool REC, bool GV, bool HOT = false,
          bool OFF64 = false>
__device__ __forceinline__ void phase_b(const FusedArgs<T>& a, const SegRegs& sg, int64_t tile,
                                        const uint32_t (&ik)[DM], const Drawn<T>& s,
                                        T* __restrict__ Gb, uint32_t rsel = 0) {
  constexpr int VW = Vec<T>::W;
  // G need not be a power of two (r = 20 fp32: 5 chunks -> 6 samples per pass
  // instead of 4); lanes beyond NGRP * G idle.
  constexpr int NGRP = 32 / G;
  constexpr int NPASS = (32 + NGRP - 1) / NGRP;
  constexpr bool POW2 = (G & (G - 1)) == 0;
  constexpr int SL = VPL * VW;  // elements of one lane's row slice
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int grp = lane / G;
  const int gl = lane % G;
  const int d = EXACT ? DM : a.d;
  const bool given = GV && sg.kind == SEG_GIVEN;
  const bool ygiven = given && a.g_y != nullptr;
  const T wseg = static_cast<T>(sg.weight);
  // Chunk ownership, clamped so every load stays inside its row; masks zero
  // the contribution of clamped (duplicate) chunks.
  int cidx[VPL];
  T cmask[VPL];
#pragma unroll
  for (int c = 0; c < VPL; ++c) {
    const int ch = gl * VPL + c;
    cidx[c] = ch < a.nchunks ? ch : a.nchunks - 1;
    cmask[c] = ch < a.nchunks ? static_cast<T>(1) : static_cast<T>(0);
  }
  const bool owns_any = gl * VPL < a.nchunks;
#pragma unroll 1
  for (int pass = 0; pass < NPASS; ++pass) {
    const int src = (pass * NGRP + grp) & 31;
    const bool v = __shfl_sync(FULL, s.valid, src) && (POW2 || (grp < NGRP && pass * NGRP + grp < 32));
    uint32_t ii[DM];
#pragma unroll
    for (int k = 0; k < DM; ++k) ii[k] = __shfl_sync(FULL, ik[k], src);
    const T xv = __shfl_sync(FULL, s.x, src);
    const uint32_t hsv = HOT ? __shfl_sync(FULL, s.hs, src) : 0xFFFFFFFFu;
    T wv = wseg;
    double wd = sg.weight;
    int fv = sg.flag;
    double yg = 0.0;
    if constexpr (GV) {
      if (given) {  // warp-uniform
        wd = __shfl_sync(FULL, s.w, src);
        wv = static_cast<T>(wd);
        fv = __shfl_sync(FULL, s.flag, src);
        yg = __shfl_sync(FULL, s.yg, src);
      }
    }
    // Row offsets (32-bit element offsets; factor buffers < 2^32 elements).
    using RowOff = RowOffT<OFF64>;
    RowOff roff[DM];
#pragma unroll
    for (int k = 0; k < DM; ++k)
      roff[k] = static_cast<RowOff>(a.off[k]) + static_cast<RowOff>(ii[k]) * static_cast<RowOff>(a.pitch);
#ifdef GCPB_CHECKED
#pragma unroll
    for (int k = 0; k < DM; ++k)
      if (EXACT || k < d)
        GCPB_CHECK(a.chk, static_cast<int64_t>(roff[k]) + a.nchunks * VW <= a.chk_tbl, 4, roff[k]);
#endif
    T row[DM][SL];
    T pre[DM][SL];
#pragma unroll
    for (int k = 0; k < DM; ++k) {
      if (EXACT || k < d) {
#pragma unroll
        for (int c = 0; c < VPL; ++c) {
          Vec<T> q;
          load_chunk(a.A + roff[k] + cidx[c] * VW, q);
#pragma unroll
          for (int e = 0; e < VW; ++e) row[k][c * VW + e] = q.v[e];
        }
      } else {
#pragma unroll
        for (int e = 0; e < SL; ++e) row[k][e] = static_cast<T>(1);
      }
    }
    T mp = static_cast<T>(0);
#pragma unroll
    for (int c = 0; c < VPL; ++c) {
      T mc = static_cast<T>(0);
#pragma unroll
      for (int e = 0; e < VW; ++e) {
        T p = row[0][c * VW + e];
        pre[0][c * VW + e] = static_cast<T>(1);
#pragma unroll
        for (int k = 1; k < DM; ++k) {
          pre[k][c * VW + e] = p;
          p = p * row[k][c * VW + e];
        }
        mc += p;
      }
      mp += cmask[c] * mc;
    }
    if constexpr (POW2) {
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) mp += __shfl_xor_sync(FULL, mp, o);
    } else {  // every lane of the group sums the group in the same order
      T tot = static_cast<T>(0);
#pragma unroll
      for (int j = 0; j < G; ++j) tot += __shfl_sync(FULL, mp, (grp * G + j) & 31);
      mp = tot;
    }
    const T m = mp;
    T y;
    if (ygiven) {
      y = static_cast<T>(yg);
    } else if (GV && fv == 2) {  // poisson implicit sparse part: -x / (m + eps) (kernels.cpp:226)
      y = -wv * (xv / (m + static_cast<T>(1e-10)));
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
    if (a.scatter) {
      // Suffix walk: excl_k = prefix_k * suffix_k (kernels.cpp:21-37); for
      // non-exact d the unused modes hold ones and issue no reductions.
      const bool act = v && owns_any;
      T suf[SL];
#pragma unroll
      for (int e = 0; e < SL; ++e) suf[e] = static_cast<T>(1);
#pragma unroll
      for (int k = DM - 1; k >= 0; --k) {
        const bool mk = EXACT || k < d;
        T* gk = grad_row<T, HOT>(a, Gb, roff[k], hsv, k, rsel);
#pragma unroll
        for (int c = 0; c < VPL; ++c) {
          T out[VW];
#pragma unroll
          for (int e = 0; e < VW; ++e) out[e] = y * (pre[k][c * VW + e] * suf[c * VW + e]);
          if (act && mk && cmask[c] != static_cast<T>(0))
            red_chunk(gk + cidx[c] * VW, out);
        }
#pragma unroll
        for (int e = 0; e < SL; ++e) suf[e] = suf[e] * row[k][e];
      }
    }
  }
}

// Measurement variant (-DGCPB_PB=2 or 4 through GCPB_NVFLAGS; default build: 1 =
// off): phase B of the slim hot-path kernels with PB passes per batch -- the
// row gathers of PB passes are issued before any of their arithmetic and
// reductions, so a warp keeps PB x DM row loads in flight instead of DM.
// Kept to reproduce DESIGN.md §5's measurement that the C5 kernel is not
// short of loads in flight.
#ifndef GCPB_PB
#define GCPB_PB 1
#endif
template <typename T, int DM, int G, int PB, bool HOT>
__device__ __forceinline__ void phase_b_batched(const FusedArgs<T>& a, const SegRegs& sg,
                                                const uint32_t (&ik)[DM], const Drawn<T>& s,
                                                T* __restrict__ Gb, uint32_t rsel) {
  constexpr int VW = Vec<T>::W;
  constexpr int NGRP = 32 / G;
  constexpr int NPASS = (32 + NGRP - 1) / NGRP;
  constexpr bool POW2 = (G & (G - 1)) == 0;
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int grp = lane / G;
  const int gl = lane % G;
  const T wseg = static_cast<T>(sg.weight);
  const int fv = sg.flag;
  const int cidx = gl < a.nchunks ? gl : a.nchunks - 1;
  const T cmask = gl < a.nchunks ? static_cast<T>(1) : static_cast<T>(0);
  const bool owns = gl < a.nchunks;
#pragma unroll 1
  for (int p0 = 0; p0 < NPASS; p0 += PB) {
    bool v[PB];
    T xv[PB];
    uint32_t hsv[PB];
    uint32_t roff[PB][DM];
    T row[PB][DM][VW];
#pragma unroll
    for (int j = 0; j < PB; ++j) {
      const int pass = p0 + j;
      const int src = (pass * NGRP + grp) & 31;
      v[j] = __shfl_sync(FULL, s.valid, src) && pass < NPASS &&
             (POW2 || (grp < NGRP && pass * NGRP + grp < 32));
      xv[j] = __shfl_sync(FULL, s.x, src);
      hsv[j] = HOT ? __shfl_sync(FULL, s.hs, src) : 0xFFFFFFFFu;
#pragma unroll
      for (int k = 0; k < DM; ++k) {
        roff[j][k] = static_cast<uint32_t>(a.off[k]) +
                     __shfl_sync(FULL, ik[k], src) * static_cast<uint32_t>(a.pitch);
        Vec<T> q;
        load_chunk(a.A + roff[j][k] + cidx * VW, q);
#pragma unroll
        for (int e = 0; e < VW; ++e) row[j][k][e] = q.v[e];
      }
    }
#pragma unroll
    for (int j = 0; j < PB; ++j) {
      T pre[DM][VW];
      T mp = static_cast<T>(0);
#pragma unroll
      for (int e = 0; e < VW; ++e) {
        T p = row[j][0][e];
        pre[0][e] = static_cast<T>(1);
#pragma unroll
        for (int k = 1; k < DM; ++k) {
          pre[k][e] = p;
          p = p * row[j][k][e];
        }
        mp += p;
      }
      mp *= cmask;
      if constexpr (POW2) {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) mp += __shfl_xor_sync(FULL, mp, o);
      } else {
        T tot = static_cast<T>(0);
#pragma unroll
        for (int jj = 0; jj < G; ++jj) tot += __shfl_sync(FULL, mp, (grp * G + jj) & 31);
        mp = tot;
      }
      T g = loss_deriv_fast(a.loss, a.delta, xv[j], mp);
      if (fv) g = g - loss_deriv_fast(a.loss, a.delta, static_cast<T>(0), mp);
      const T y = wseg * g;
      const bool act = v[j] && owns;
      T suf[VW];
#pragma unroll
      for (int e = 0; e < VW; ++e) suf[e] = static_cast<T>(1);
#pragma unroll
      for (int k = DM - 1; k >= 0; --k) {
        T out[VW];
#pragma unroll
        for (int e = 0; e < VW; ++e) {
          out[e] = y * (pre[k][e] * suf[e]);
          suf[e] = suf[e] * row[j][k][e];
        }
        if (act) red_chunk(grad_row<T, HOT>(a, Gb, roff[j][k], hsv[j], k, rsel) + cidx * VW, out);
      }
    }
  }
}

template <typename T, int DM, bool EXACT, int G, int VPL, bool REC, int MINB, bool GV = true,
          bool HOT = false, bool OFF64 = false>
__global__ void __launch_bounds__(256, MINB) fused_grad_kernel(const FusedArgs<T> a,
                                                               int64_t total_tiles) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  T* Gb = a.G + static_cast<int64_t>(blockIdx.x % a.nrep) * a.rep_stride;
  // Iteration of the draw stream: kernel argument plus an optional
  // device-resident base (graph-replayed steps advance it without relaunch).
  const uint64_t iter = a.iter + (a.iter_base ? __ldg(a.iter_base) : 0ull);
  int64_t tile = warp0;
  if (tile >= total_tiles) return;
  uint32_t ik[DM];
  Drawn<T> s;
  const uint32_t rsel = HOT ? static_cast<uint32_t>(warp0) & static_cast<uint32_t>(a.rh - 1) : 0u;
  SegRegs sg = seg_of<T>(a, tile);
  phase_a<T, DM, EXACT, GV, HOT>(a, sg, sg.t_begin + (tile - sg.tiles_begin) * 32 + lane, iter,
                                 ik, s);
  for (; tile < total_tiles; tile += nwarps) {
    const int64_t next = tile + nwarps;
    uint32_t ik2[DM];
    Drawn<T> s2;
    SegRegs sg2 = sg;
    if (next < total_tiles) {  // prefetch: next tile's draws + tensor gathers in flight
      sg2 = seg_of<T>(a, next);
      phase_a<T, DM, EXACT, GV, HOT>(a, sg2, sg2.t_begin + (next - sg2.tiles_begin) * 32 + lane,
                                     iter, ik2, s2);
    } else {
      s2.valid = false;
      if (HOT) s2.hs = 0xFFFFFFFFu;
#pragma unroll
      for (int k = 0; k < DM; ++k) ik2[k] = 0;
    }
    if (__any_sync(0xffffffffu, s.valid)) {  // tiles past a device-resident length
      if constexpr (GCPB_PB > 1 && EXACT && VPL == 1 && !REC && !GV && !OFF64 && DM <= 4)
        phase_b_batched<T, DM, G, GCPB_PB, HOT>(a, sg, ik, s, Gb, rsel);
      else
        phase_b<T, DM, EXACT, G, VPL, REC, GV, HOT, OFF64>(a, sg, tile, ik, s, Gb, rsel);
    }
#pragma unroll
    for (int k = 0; k < DM; ++k) ik[k] = ik2[k];
    s = s2;
    sg = sg2;
  }
}

// Lane geometry: nchunks 16-byte chunks per row; G lanes per sample (pow2 >=
// nchunks, <= 32), VPL chunks per lane when a row exceeds 32 chunks.
inline int pow2ceil(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

template <typename T, int DM, bool EXACT, bool REC>
cudaError_t launch_fused_dm(const FusedArgs<T>& a, int64_t total_tiles, cudaStream_t stream,
                            int num_sms, bool* used_hot, int bps_cap) {
  constexpr int MHOT = DM == 3 ? GCPB_MINB_HOT3 : GCPB_MINB_HOT;
  constexpr int MHOT8 = DM == 4 ? GCPB_MINB_HOT8 : MHOT;
  const int nchunks = a.nchunks;
  int G = pow2ceil(nchunks);
  int vpl = 1;
  if (G > 32) {
    G = 32;
    vpl = pow2ceil((nchunks + 31) / 32);
  }
  bool given = false;  // any segment beyond the samplers needs the general kernel
  for (int s = 0; s < a.nseg; ++s) given = given || a.seg[s].kind >= SEG_GIVEN;
  auto go = [&](auto kern) -> cudaError_t {
    // resident blocks per SM: queried once per kernel instantiation (the
    // query costs microseconds, and small steps are launch-bound)
    static const int per_sm = [&] {
      int v = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, 256, 0);
      return v < 1 ? 1 : v;
    }();
    int64_t blocks = (total_tiles + 7) / 8;
    // bps_cap > 0: fewer resident blocks per SM than fit (random HBM access
    // peaks below full occupancy, profiles/r01_randbw.md)
    const int64_t cap = static_cast<int64_t>(num_sms) * (bps_cap > 0 && bps_cap < per_sm ? bps_cap : per_sm);
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    return launch_k(kern, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, stream, a,
                    total_tiles);
  };
  if (a.off64) {  // tables beyond 2^31 padded elements: 64-bit row offsets
    if constexpr (EXACT && (DM == 3 || DM == 4)) {
      if (vpl == 1) return go(fused_grad_kernel<T, DM, EXACT, 32, 1, REC, 1, true, false, true>);
    }
    return cudaErrorNotSupported;  // the host checks the shape before launching
  }
  if (vpl == 1) {
    if constexpr (!REC && EXACT) {
      if (!given) {  // hot path: no host-given samples -> slim live state
        if constexpr (sizeof(T) == 4) {  // 5 or 6 chunks: non-power-of-two lane groups
          if (nchunks == 5 || nchunks == 6) {
            if constexpr (DM <= 4) {
              if (a.rh > 0) {
                *used_hot = true;
                return nchunks == 5
                           ? go(fused_grad_kernel<T, DM, EXACT, 5, 1, REC, MHOT, false, true>)
                           : go(fused_grad_kernel<T, DM, EXACT, 6, 1, REC, MHOT, false, true>);
              }
            }
            return nchunks == 5
                       ? go(fused_grad_kernel<T, DM, EXACT, 5, 1, REC, GCPB_MINB_SLIM, false>)
                       : go(fused_grad_kernel<T, DM, EXACT, 6, 1, REC, GCPB_MINB_SLIM, false>);
          }
        }
        if constexpr (DM <= 4) {
          if (a.rh > 0) {  // hot rows privatized (sparse, skewed modes)
            *used_hot = true;
            switch (G) {
              case 1: return go(fused_grad_kernel<T, DM, EXACT, 1, 1, REC, MHOT, false, true>);
              case 2: return go(fused_grad_kernel<T, DM, EXACT, 2, 1, REC, MHOT, false, true>);
              case 4: return go(fused_grad_kernel<T, DM, EXACT, 4, 1, REC, MHOT, false, true>);
              case 8: return go(fused_grad_kernel<T, DM, EXACT, 8, 1, REC, MHOT8, false, true>);
              case 16: return go(fused_grad_kernel<T, DM, EXACT, 16, 1, REC, MHOT, false, true>);
              default: return go(fused_grad_kernel<T, DM, EXACT, 32, 1, REC, MHOT, false, true>);
            }
          }
        }
        switch (G) {
          case 1: return go(fused_grad_kernel<T, DM, EXACT, 1, 1, REC, GCPB_MINB_SLIM, false>);
          case 2: return go(fused_grad_kernel<T, DM, EXACT, 2, 1, REC, GCPB_MINB_SLIM, false>);
          case 4: return go(fused_grad_kernel<T, DM, EXACT, 4, 1, REC, GCPB_MINB_SLIM, false>);
          case 8: return go(fused_grad_kernel<T, DM, EXACT, 8, 1, REC, GCPB_MINB_SLIM, false>);
          case 16: return go(fused_grad_kernel<T, DM, EXACT, 16, 1, REC, GCPB_MINB_SLIM, false>);
          default: return go(fused_grad_kernel<T, DM, EXACT, 32, 1, REC, GCPB_MINB_SLIM, false>);
        }
      }
    }
    switch (G) {
      case 1: return go(fused_grad_kernel<T, DM, EXACT, 1, 1, REC, GCPB_MINB>);
      case 2: return go(fused_grad_kernel<T, DM, EXACT, 2, 1, REC, GCPB_MINB>);
      case 4: return go(fused_grad_kernel<T, DM, EXACT, 4, 1, REC, GCPB_MINB>);
      case 8: return go(fused_grad_kernel<T, DM, EXACT, 8, 1, REC, GCPB_MINB>);
      case 16: return go(fused_grad_kernel<T, DM, EXACT, 16, 1, REC, GCPB_MINB>);
      default: return go(fused_grad_kernel<T, DM, EXACT, 32, 1, REC, GCPB_MINB>);
    }
  }
  if (vpl <= 2) return go(fused_grad_kernel<T, DM, EXACT, 32, 2, REC, 1>);
  if (vpl <= 4) return go(fused_grad_kernel<T, DM, EXACT, 32, 4, REC, 1>);
  return go(fused_grad_kernel<T, DM, EXACT, 32, 8, REC, 1>);
}

template <typename T, bool REC>
cudaError_t launch_fused_rec(const FusedArgs<T>& a, int64_t total_tiles, cudaStream_t stream,
                             int num_sms, bool* used_hot, int bps_cap) {
  switch (a.d) {
    case 3: return launch_fused_dm<T, 3, true, REC>(a, total_tiles, stream, num_sms, used_hot, bps_cap);
    case 4: return launch_fused_dm<T, 4, true, REC>(a, total_tiles, stream, num_sms, used_hot, bps_cap);
    case 1:
    case 2: return launch_fused_dm<T, 2, false, REC>(a, total_tiles, stream, num_sms, used_hot, bps_cap);
    default:
      if (a.d <= 8)
        return launch_fused_dm<T, 8, false, REC>(a, total_tiles, stream, num_sms, used_hot, bps_cap);
      return launch_fused_dm<T, 16, false, REC>(a, total_tiles, stream, num_sms, used_hot, bps_cap);
  }
}

// *used_hot reports whether the launched variant sent hot rows to a.Ghot
// (only the hot-path variants do; the caller folds Ghot back only then).
template <typename T>
cudaError_t launch_fused(const FusedArgs<T>& a, int64_t total_tiles, bool record,
                         cudaStream_t stream, int num_sms, bool* used_hot, int bps_cap) {
  *used_hot = false;
  if (total_tiles <= 0) return cudaSuccess;
  if (record) return launch_fused_rec<T, true>(a, total_tiles, stream, num_sms, used_hot, bps_cap);
  return launch_fused_rec<T, false>(a, total_tiles, stream, num_sms, used_hot, bps_cap);
}

}  // namespace gcpb
