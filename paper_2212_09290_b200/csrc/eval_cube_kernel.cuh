// SPDX-License-Identifier: Apache-2.0
#pragma once
//
// K2a — batched evaluation of dense (R,S) candidate cubes on sm_100a.
//
// Per candidate this computes exactly what the reference composes per
// candidate on the CPU:
//   complete_assignment   proj/src/model.cpp:471-549  (Z, F hazards, U recurrence)
//   objective_value       proj/src/model.cpp:369-428  (same summation order)
//   check_assignment      proj/src/model.cpp:430-469  (one XE_F_* bit per family)
//   replay peaks          proj/src/schedule.cpp:326-367 (= max U, acceptance crit. 6)
//   decode legality       proj/src/schedule.cpp:40-129
// without materialising the O(n) assignment map: every family that can fail
// on a completion is evaluated in closed form on bit rows.
//
// Layout.  One warp owns one candidate at a time; lanes stride over
// timesteps t with every device's rows of that t in registers.  The
// candidate (8*D*T*W bytes) is staged global->shared by the bulk-copy (TMA)
// engine, double-buffered per warp behind an mbarrier, so HBM streams while
// the previous candidate is evaluated.  Problem tables (masses, parent /
// consumer masks, mass byte-tables, objective terms) live in shared memory.
//
// Fast paths (the common case of placement-like candidates): a row with at
// most one computation needs no free bookkeeping (its peak is base + m_v);
// copy charges are enumerated only when some device needs a parent that
// another device holds (a mask test); decode's copy-source check runs only
// when a copy exists.  The general paths stay exact for every input.
//
// Objective.  Two modes, both bit-identical to the reference's sequential
// double sum:
//   EXACT  every term is k-bit dyadic and the worst-case total < 2^52 units
//          (xe::exact_fix_k) -> int64 fixed-point sums, any order.
//   serial otherwise: the warp writes each candidate's term indices in the
//          reference loop order into a per-slot list; after kSlots
//          candidates lane s replays slot s's list with sequential FP64 adds.

#include <cfloat>
#include <climits>

#include "bits.cuh"
#include "xe_internal.hpp"

namespace xe {
namespace cube {

constexpr int kWarps = 8;
constexpr int kSlots = 32;

struct EvalArgs {
  DevProblem P;
  const uint32_t* cubes;
  int64_t n;
  double* obj;
  int64_t* peak;
  uint32_t* flags;
  int strict, energy;
  uint32_t valid_mask;
  uint64_t* wbest_key;
  int64_t* wbest_idx;
  int64_t* wvalid;
  // shared-memory plan (byte offsets)
  int off_mass, off_pmask, off_cons, off_mtab, off_tab, off_inptr, off_inedge, off_src, off_dst,
      off_ebad, off_q, off_warp;
  int warp_bytes, off_w_stage, off_w_bar, off_w_terms, off_w_terms2, off_w_slot;
  int stages, cap, cap2, use_bulk;
  int warps;  // warps per CTA (shared-memory plan decides, <= kWarps)
  uint32_t cube_words;
};

template <int NW>
__device__ __forceinline__ int64_t mass_bytes(const Row<NW>& r, const int64_t* mtab, int NB) {
  int64_t s = 0;
#pragma unroll
  for (int j = 0; j < NW; ++j) {
    const uint64_t w = r.w[j];
    if (!w) continue;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const int idx = 8 * j + b;
      if (idx < NB) s += mtab[idx * 256 + ((w >> (8 * b)) & 0xff)];
    }
  }
  return s;
}

template <int NW>
__device__ __forceinline__ int64_t mass_bits(Row<NW> r, const int64_t* mass) {
  int64_t s = 0;
#pragma unroll
  for (int j = 0; j < NW; ++j) {
    uint64_t w = r.w[j];
    while (w) {
      const int b = __ffsll(w) - 1;
      w &= w - 1;
      s += mass[64 * j + b];
    }
  }
  return s;
}

// Row (which, d, t) of a staged candidate.  W32 even -> 8-byte aligned u64
// loads (conflict-free across lanes); odd -> u32 pairs.
template <int NW>
__device__ __forceinline__ Row<NW> cube_row(const uint32_t* cw, int W32, int D, int T, int which,
                                            int d, int t) {
  Row<NW> r;
  const uint32_t* p = cw + ((which * D + d) * T + t) * W32;
  if ((W32 & 1) == 0) {
    const uint64_t* q = reinterpret_cast<const uint64_t*>(p);
#pragma unroll
    for (int j = 0; j < NW; ++j) r.w[j] = (2 * j < W32) ? q[j] : 0ull;
  } else {
#pragma unroll
    for (int j = 0; j < NW; ++j) {
      uint64_t lo = (2 * j < W32) ? p[2 * j] : 0u;
      uint64_t hi = (2 * j + 1 < W32) ? p[2 * j + 1] : 0u;
      r.w[j] = lo | (hi << 32);
    }
  }
  return r;
}

template <int NW, int MAXD>
struct TState {
  Row<NW> R[MAXD], S[MAXD], Sn[MAXD], Z[MAXD];
  Row<NW> Rany, Zany;
};

// Device count: exact at compile time for D <= 4, runtime (<= 8) otherwise.
template <int MAXD>
__device__ __forceinline__ int ndev(const DevProblem& P) {
  return MAXD <= 4 ? MAXD : P.D;
}

template <int NW, int MAXD>
__device__ __forceinline__ void load_t(TState<NW, MAXD>& st, const uint32_t* cw, const DevProblem& P,
                                       int t, bool active) {
  const int D = ndev<MAXD>(P);
  st.Rany = Row<NW>::zero();
  st.Zany = Row<NW>::zero();
  const Row<NW> valid = Row<NW>::below(P.T);  // padding bits >= T are not variables
#pragma unroll
  for (int d = 0; d < MAXD; ++d) {
    if (d < D && active) {
      st.R[d] = cube_row<NW>(cw, P.W32, D, P.T, 0, d, t) & valid;
      st.S[d] = cube_row<NW>(cw, P.W32, D, P.T, 1, d, t) & valid;
      st.Sn[d] = (t + 1 < P.T) ? (cube_row<NW>(cw, P.W32, D, P.T, 1, d, t + 1) & valid) : Row<NW>::zero();
    } else {
      st.R[d] = Row<NW>::zero();
      st.S[d] = Row<NW>::zero();
      st.Sn[d] = Row<NW>::zero();
    }
    st.Z[d] = st.R[d] | st.S[d];
    st.Rany = st.Rany | st.R[d];
    st.Zany = st.Zany | st.Z[d];
  }
}

// Enumerate the copy charges of timestep t in objective_value's order
// (model.cpp:399-411): edges ascending, then computing device dc, then source
// device ds != dc with Z(ds,t,src) = 1.  fn(term_index).
template <int NW, int MAXD, bool ORDERED, class F>
__device__ __forceinline__ void for_copy_terms(const TState<NW, MAXD>& st, const DevProblem& P,
                                               const int32_t* s_inptr, const int32_t* s_inedge,
                                               const int32_t* s_src, const int32_t* s_dst, F&& fn) {
  const int D = ndev<MAXD>(P);
  const int base = D * P.T;
  auto one_edge = [&](int e) {
    const int u = s_src[e], v = s_dst[e];
#pragma unroll
    for (int dc = 0; dc < MAXD; ++dc) {
      if (dc >= D || !st.R[dc].test(v)) continue;
#pragma unroll
      for (int ds = 0; ds < MAXD; ++ds) {
        if (ds >= D || ds == dc || !st.Z[ds].test(u)) continue;
        fn(base + (e * D + ds) * D + dc);
      }
    }
  };
  if (!ORDERED || P.edges_by_dst) {
    // in-edge lists ascend in edge id; with dst-monotone edge order the
    // concatenation over ascending v is ascending in edge id too
#pragma unroll
    for (int j = 0; j < NW; ++j) {
      uint64_t w = st.Rany.w[j];
      while (w) {
        const int v = 64 * j + __ffsll(w) - 1;
        w &= w - 1;
        for (int k = s_inptr[v]; k < s_inptr[v + 1]; ++k) one_edge(s_inedge[k]);
      }
    }
  } else {
    int last = -1;
    for (;;) {
      int best = INT_MAX;
#pragma unroll
      for (int j = 0; j < NW; ++j) {
        uint64_t w = st.Rany.w[j];
        while (w) {
          const int v = 64 * j + __ffsll(w) - 1;
          w &= w - 1;
          for (int k = s_inptr[v]; k < s_inptr[v + 1]; ++k) {
            const int e = s_inedge[k];
            if (e > last) {
              if (e < best) best = e;
              break;
            }
          }
        }
      }
      if (best == INT_MAX) break;
      one_edge(best);
      last = best;
    }
  }
}

// Peak of U over the slots of row (d,t) when it holds >= 2 computations:
// descending over computes, F(u->v) fires for u in (parents(v) + v) that is
// resident, not kept (S(d,t+1,u) = 0) and has no later consumer computed
// (on d; on any device with strict_free) — model.cpp:492-505, 521-537.
// Arguments by value so the rare path keeps everything in registers.
template <int NW>
__device__ __noinline__ int64_t row_peak_general(Row<NW> Rd, Row<NW> Zd, Row<NW> Snd, Row<NW> scan,
                                                 int64_t base, const uint64_t* s_pmask,
                                                 const int64_t* s_mass) {
  Row<NW> seen = Row<NW>::zero();
  int64_t acc = 0, mx = LLONG_MIN, sR = 0, sF = 0;
  for (int v = scan.msb(); v >= 0;) {
    const Row<NW> pm = load_row<NW>(s_pmask + v * NW);
    if (Rd.test(v)) {
      Row<NW> f = pm;
      f.set(v);
      f = andnot(andnot(f & Zd, Snd), seen);
      const int64_t fm = mass_bits<NW>(f, s_mass), mv = s_mass[v];
      mx = max(mx, acc + fm);
      acc += fm - mv;
      sR += mv;
      sF += fm;
    }
    seen = seen | pm;
    v = (scan & ~Row<NW>::at_or_above(v)).msb();
  }
  return max(base, base + sR - sF + mx);
}

// EQ16_HI rows of (d,t): with S(d,t+1,u) = 1 and Z(d,t,u) = 0 (an EQ11
// failure) the HI row fails iff R(d,t,v) = 0 and every later consumer term
// is 1 (model.cpp:200-224); Cd = R(d,t,.) (default) or AND_dd R(dd,t,.)
// (strict).  Returns XE_F_EQ16_HI or 0.
template <int NW>
__device__ __noinline__ uint32_t eq16_hi(Row<NW> Rd, Row<NW> Cd, Row<NW> bad, const uint64_t* s_cons) {
  for (int u = bad.lsb(); u >= 0; bad.clear(u), u = bad.lsb()) {
    const Row<NW> cu = load_row<NW>(s_cons + u * NW);
    if (!andnot(cu, Cd).any()) return XE_F_EQ16_HI;  // self edge F(u,u)
    for (Row<NW> cv = cu; cv.any();) {
      const int v = cv.lsb();
      cv.clear(v);
      if (!Rd.test(v) && !andnot(cu & Row<NW>::above(v), Cd).any()) return XE_F_EQ16_HI;
    }
  }
  return 0;
}

// decode(): a copy for a compute (d, v <= t) comes from the lowest device
// holding the tensor u; it is illegal when that source freed u at an earlier
// step of the same timestep (schedule.cpp:52-71).  Rs/keep describe the
// source device; returns XE_F_DECODE|XE_F_DECODE_FREED or 0.
template <int NW>
__device__ __noinline__ uint32_t decode_freed_one(Row<NW> Rs, Row<NW> Rany, Row<NW> Rd, int u, int t,
                                                  int sdev, int d, int strict, const uint64_t* s_cons) {
  const Row<NW> cu = load_row<NW>(s_cons + u * NW);
  int fs = -1;
  const Row<NW> c = cu & (strict ? Rany : Rs);
  if (c.any()) {
    const int m = c.msb();
    fs = Rs.test(m) ? m : -1;
  } else if (Rs.test(u)) {
    fs = u;
  }
  if (fs < 0) return 0;
  const int vmax = (cu & Rd & ~Row<NW>::above(t)).msb();
  return (fs < vmax || (fs == vmax && sdev < d)) ? (XE_F_DECODE | XE_F_DECODE_FREED) : 0u;
}

// Sequential objective by one lane straight from the staged cube — used
// only when a candidate's term list exceeds the per-slot capacity.
template <int NW, int MAXD>
__device__ __noinline__ double objective_lane(const uint32_t* cw, const DevProblem& P,
                                              const double* tab, const int32_t* s_inptr,
                                              const int32_t* s_inedge, const int32_t* s_src,
                                              const int32_t* s_dst, int energy) {
  const int D = ndev<MAXD>(P), T = P.T;
  double total = 0.0;
  for (int d = 0; d < D; ++d)
    for (int t = 0; t < T; ++t) {
      Row<NW> r = cube_row<NW>(cw, P.W32, D, T, 0, d, t) & Row<NW>::below(T);
      for (int i = r.lsb(); i >= 0; r.clear(i), i = r.lsb()) total = __dadd_rn(total, tab[d * T + i]);
    }
  for (int t = 0; t < T; ++t) {
    TState<NW, MAXD> st;
    load_t<NW, MAXD>(st, cw, P, t, true);
    for_copy_terms<NW, MAXD, true>(st, P, s_inptr, s_inedge, s_src, s_dst,
                                   [&](int idx) { total = __dadd_rn(total, tab[idx]); });
  }
  if (energy) {
    const int eb = D * T + P.E * D * D;
    for (int d = 0; d < D; ++d)
      for (int t = 0; t < T; ++t) {
        Row<NW> r = cube_row<NW>(cw, P.W32, D, T, 0, d, t) & Row<NW>::below(T);
        for (int i = r.lsb(); i >= 0; r.clear(i), i = r.lsb()) total = __dadd_rn(total, tab[eb + d * T + i]);
      }
  }
  return total;
}

// 64-bit warp max from two 32-bit REDUX ops (values are non-negative).
__device__ __forceinline__ int64_t warp_max_u63(int64_t v) {
  const uint32_t hi = static_cast<uint32_t>(static_cast<uint64_t>(v) >> 32);
  const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
  const uint32_t lo = hi == mh ? static_cast<uint32_t>(v) : 0u;
  const uint32_t ml = __reduce_max_sync(0xffffffffu, lo);
  return static_cast<int64_t>((static_cast<uint64_t>(mh) << 32) | ml);
}

template <int NW, int MAXD, bool EXACT>
__global__ void __launch_bounds__(kWarps * 32, 2) eval_cube_kernel(const EvalArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const DevProblem& P = a.P;
  const int D = ndev<MAXD>(P), T = P.T, E = P.E;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;

  int64_t* s_mass = reinterpret_cast<int64_t*>(smem + a.off_mass);
  uint64_t* s_pmask = reinterpret_cast<uint64_t*>(smem + a.off_pmask);
  uint64_t* s_cons = reinterpret_cast<uint64_t*>(smem + a.off_cons);
  int64_t* s_mtab = reinterpret_cast<int64_t*>(smem + a.off_mtab);
  double* s_tab = reinterpret_cast<double*>(smem + a.off_tab);
  int64_t* s_tfix = reinterpret_cast<int64_t*>(smem + a.off_tab);
  int32_t* s_inptr = reinterpret_cast<int32_t*>(smem + a.off_inptr);
  int32_t* s_inedge = reinterpret_cast<int32_t*>(smem + a.off_inedge);
  int32_t* s_src = reinterpret_cast<int32_t*>(smem + a.off_src);
  int32_t* s_dst = reinterpret_cast<int32_t*>(smem + a.off_dst);
  uint64_t* s_ebad = reinterpret_cast<uint64_t*>(smem + a.off_ebad);
  double* s_q = reinterpret_cast<double*>(smem + a.off_q);

  // ---- problem tables -> shared (once per CTA) ----
  for (int i = threadIdx.x; i < T; i += blockDim.x) s_mass[i] = P.mass[i];
  for (int i = threadIdx.x; i < T * NW; i += blockDim.x) {
    s_pmask[i] = P.pmask[i];
    s_cons[i] = P.cons[i];
  }
  for (int i = threadIdx.x; i < P.NB * 256; i += blockDim.x) s_mtab[i] = P.mtab[i];
  for (int i = threadIdx.x; i < P.n_table; i += blockDim.x) {
    if (EXACT) s_tfix[i] = P.tfix[i];
    else s_tab[i] = P.table[i];
  }
  for (int i = threadIdx.x; i <= T; i += blockDim.x) s_inptr[i] = P.in_ptr[i];
  for (int i = threadIdx.x; i < E; i += blockDim.x) {
    s_inedge[i] = P.in_edge[i];
    s_src[i] = P.src[i];
    s_dst[i] = P.dst[i];
  }
  if (a.energy) {
    for (int i = threadIdx.x; i < D * NW; i += blockDim.x) s_ebad[i] = P.ebad[i];
    if (P.has_total)
      for (int i = threadIdx.x; i < D * T; i += blockDim.x) s_q[i] = P.q[i];
  }

  // ---- per-warp region ----
  unsigned char* wreg = smem + a.off_warp + wid * a.warp_bytes;
  uint32_t* stage_buf = reinterpret_cast<uint32_t*>(wreg + a.off_w_stage);
  uint64_t* bars = reinterpret_cast<uint64_t*>(wreg + a.off_w_bar);
  uint16_t* terms = reinterpret_cast<uint16_t*>(wreg + a.off_w_terms);
  uint16_t* terms2 = reinterpret_cast<uint16_t*>(wreg + a.off_w_terms2);  // energy terms
  double* slot_obj = reinterpret_cast<double*>(wreg + a.off_w_slot);
  uint32_t* slot_flags = reinterpret_cast<uint32_t*>(slot_obj + kSlots);
  int32_t* slot_cnt = reinterpret_cast<int32_t*>(slot_flags + kSlots);
  int32_t* slot_cnt2 = slot_cnt + kSlots;
  int64_t* slot_peak = reinterpret_cast<int64_t*>(slot_cnt2 + kSlots);  // [kSlots][D]

  if (lane == 0)
    for (int s = 0; s < a.stages; ++s) mbar_init(&bars[s], 1);
  fence_mbar_init();
  __syncthreads();

  const int64_t gwarp = static_cast<int64_t>(blockIdx.x) * a.warps + wid;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * a.warps;
  const int64_t nblocks = (a.n + kSlots - 1) / kSlots;
  const uint32_t cube_bytes = a.cube_words * 4u;
  const int tail_bits = T & 31;
  const uint32_t tail_mask = tail_bits ? ((1u << tail_bits) - 1u) : 0xffffffffu;
  const int row_words = T * P.W32;  // u32 words of one device's R cube

  uint64_t best_key = ~0ull;
  int64_t best_idx = -1, n_valid = 0;

  auto cand_of = [&](int64_t k) -> int64_t {  // k-th candidate of this warp
    const int64_t blk = gwarp + (k / kSlots) * nwarps;
    return blk * kSlots + (k % kSlots);
  };
  auto issue = [&](int64_t c, int stage) {
    if (c >= a.n) return;
    const uint32_t* src = a.cubes + static_cast<size_t>(c) * a.cube_words;
    uint32_t* dst = stage_buf + static_cast<size_t>(stage) * a.cube_words;
    if (a.use_bulk) {
      if (lane == 0) {
        fence_proxy_async();
        mbar_expect_tx(&bars[stage], cube_bytes);
        bulk_g2s(dst, src, cube_bytes, &bars[stage]);
      }
    } else {
      for (uint32_t i = lane; i < a.cube_words; i += 32) dst[i] = __ldg(src + i);
      __syncwarp();
    }
  };

  uint32_t phase_bits = 0;
  int64_t k = 0;
  if (gwarp < nblocks) issue(cand_of(0), 0);

  for (int64_t blk = gwarp; blk < nblocks; blk += nwarps) {
    const int64_t first = blk * kSlots;
    const int nslot = static_cast<int>(a.n - first < kSlots ? a.n - first : kSlots);
    for (int s = 0; s < nslot; ++s, ++k) {
      const int stage = static_cast<int>(k % a.stages);
      {  // prefetch the warp's next candidate into the other stage
        const int64_t nk = k + 1;
        int64_t nc = (nk % kSlots == 0) ? cand_of(nk) : (s + 1 < nslot ? first + s + 1 : a.n);
        issue(nc, static_cast<int>(nk % a.stages));
      }
      if (a.use_bulk) {
        mbar_wait(&bars[stage], (phase_bits >> stage) & 1u);
        phase_bits ^= 1u << stage;
      }
      const uint32_t* cw = stage_buf + static_cast<size_t>(stage) * a.cube_words;

      // ---- serial mode: per-device R popcounts give each device's term base
      int baseR[MAXD], sumR = 0;
      if (!EXACT) {
#pragma unroll
        for (int d = 0; d < MAXD; ++d) {
          int c = 0;
          if (d < D)
            for (int w = lane; w < row_words; w += 32) {
              uint32_t x = cw[d * row_words + w];
              if ((w % P.W32) == P.W32 - 1) x &= tail_mask;
              c += __popc(x);
            }
          c = __reduce_add_sync(0xffffffffu, c);
          baseR[d] = sumR;
          sumR += c;
        }
      }
      // copy terms are checked against the capacity as they are counted
      const bool list_ok = EXACT || (sumR <= a.cap && (!a.energy || sumR <= a.cap2));
      bool overflow = !list_ok;
      uint16_t* list = terms + s * a.cap;
      uint16_t* list2 = terms2 + s * a.cap2;

      uint32_t fl = 0;
      int eq9 = 0, runC = 0;
      int runR[MAXD];
      int64_t pk[MAXD];
#pragma unroll
      for (int d = 0; d < MAXD; ++d) {
        pk[d] = 0;
        runR[d] = 0;
      }
      int64_t fix = 0;

      for (int t0 = 0; t0 < T; t0 += 32) {
        const int t = t0 + lane;
        const bool act = t < T;
        TState<NW, MAXD> st;
        load_t<NW, MAXD>(st, cw, P, t, act);
        Row<NW> need_all = Row<NW>::zero(), need_le = Row<NW>::zero();
        Row<NW> needD[MAXD], needAllD[MAXD];
        if (act) {
          const Row<NW> above_t = Row<NW>::above(t), ge_t = Row<NW>::at_or_above(t);
          int nd = 0;
#pragma unroll
          for (int d = 0; d < MAXD; ++d) {
            if (d >= D) continue;
            if ((st.R[d] & above_t).any() || (st.S[d] & ge_t).any()) fl |= XE_F_FIXED_ZERO;
            nd += st.R[d].test(t);
            const Row<NW> bad = andnot(st.Sn[d], st.Z[d]);  // EQ11
            if (bad.any()) {
              Row<NW> allR = st.R[0];
#pragma unroll
              for (int x = 1; x < MAXD; ++x)
                if (x < D) allR = allR & st.R[x];
              fl |= XE_F_EQ11 | eq16_hi<NW>(st.R[d], a.strict ? allR : st.R[d], bad, s_cons);
            }
            if (a.energy && (st.R[d] & load_row<NW>(s_ebad + d * NW)).any()) fl |= XE_F_ENERGY_DEV;
          }
          if (nd != 1) fl |= XE_F_EQ8;
          eq9 += nd;

          // ---- memory: base (saved tensors) + computations of row (d,t)
#pragma unroll
          for (int d = 0; d < MAXD; ++d) {
            needD[d] = Row<NW>::zero();
            needAllD[d] = Row<NW>::zero();
            if (d >= D) continue;
            const int64_t base = mass_bytes<NW>(st.S[d], s_mtab, P.NB);
            const int c = st.R[d].popc();
            int64_t rp = base;
            if (c == 1) rp = base + s_mass[st.R[d].lsb()];
            else if (c > 1)
              rp = row_peak_general<NW>(st.R[d], st.Z[d], st.Sn[d], a.strict ? st.Rany : st.R[d], base,
                                        s_pmask, s_mass);
            pk[d] = max(pk[d], rp);
          }
          // ---- dependency masks over the computations of timestep t
          for (Row<NW> rem = st.Rany; rem.any();) {
            const int v = rem.lsb();
            rem.clear(v);
            const Row<NW> pm = load_row<NW>(s_pmask + v * NW);
            need_all = need_all | pm;
            const bool le = v <= t;
            if (le) need_le = need_le | pm;
#pragma unroll
            for (int d = 0; d < MAXD; ++d)
              if (d < D && st.R[d].test(v)) {
                needAllD[d] = needAllD[d] | pm;
                if (le) needD[d] = needD[d] | pm;
              }
          }
          if (andnot(need_all, st.Zany).any()) fl |= XE_F_EQ12;
          if (andnot(need_le, st.Zany).any()) fl |= XE_F_DECODE;
#pragma unroll
          for (int d = 0; d < MAXD; ++d) {
            if (d >= D) continue;
            Row<NW> miss = andnot(needD[d], st.Z[d]) & st.Zany;
            for (int u = miss.lsb(); u >= 0; miss.clear(u), u = miss.lsb()) {
              int sdev = 0;
#pragma unroll
              for (int x = MAXD - 1; x >= 0; --x)
                if (x < D && st.Z[x].test(u)) sdev = x;
              Row<NW> Rs = st.R[0];
              bool keep = false;
#pragma unroll
              for (int x = 0; x < MAXD; ++x)
                if (x == sdev) {
                  Rs = st.R[x];
                  keep = st.Sn[x].test(u);
                }
              if (!keep) fl |= decode_freed_one<NW>(Rs, st.Rany, st.R[d], u, t, sdev, d, a.strict, s_cons);
            }
          }

          // ---- ENERGY_TOTAL row of timestep t: sequential sum in (d, i) order
          if (a.energy && P.has_total) {
            double lhs = 0.0, scale = fmax(1.0, fabs(P.total_rhs));
#pragma unroll
            for (int d = 0; d < MAXD; ++d) {
              if (d >= D) continue;
              Row<NW> r = st.R[d];
              for (int i = r.lsb(); i >= 0; r.clear(i), i = r.lsb()) {
                const double q = s_q[d * T + i];
                if (q != 0.0) {
                  lhs = __dadd_rn(lhs, q);
                  scale = fmax(scale, fabs(q));
                }
              }
            }
            if (__dsub_rn(lhs, P.total_rhs) > 1e-6 * scale) fl |= XE_F_ENERGY_TOTAL;
          }
        } else {
#pragma unroll
          for (int d = 0; d < MAXD; ++d) {
            needD[d] = Row<NW>::zero();
            needAllD[d] = Row<NW>::zero();
          }
        }

        // copy charges exist iff some device needs a parent another device holds
        bool has_copy = false;
#pragma unroll
        for (int dc = 0; dc < MAXD; ++dc)
#pragma unroll
          for (int ds = 0; ds < MAXD; ++ds)
            if (dc < D && ds < D && ds != dc && (needAllD[dc] & st.Z[ds]).any()) has_copy = true;

        // ---- objective terms
        if (EXACT) {
          if (act) {
            const int eb = D * T + E * D * D;
#pragma unroll
            for (int d = 0; d < MAXD; ++d) {
              if (d >= D) continue;
              Row<NW> r = st.R[d];
              for (int i = r.lsb(); i >= 0; r.clear(i), i = r.lsb()) {
                fix += s_tfix[d * T + i];
                if (a.energy) fix += s_tfix[eb + d * T + i];
              }
            }
            if (has_copy)
              for_copy_terms<NW, MAXD, false>(st, P, s_inptr, s_inedge, s_src, s_dst,
                                              [&](int idx) { fix += s_tfix[idx]; });
          }
        } else if (!overflow) {
          const int eb = D * T + E * D * D;
#pragma unroll
          for (int d = 0; d < MAXD; ++d) {
            if (d >= D) continue;
            int chunk_tot;
            int pos = baseR[d] + runR[d] + warp_excl_scan(st.R[d].popc(), lane, &chunk_tot);
            runR[d] += chunk_tot;
            Row<NW> r = st.R[d];
            for (int i = r.lsb(); i >= 0; r.clear(i), i = r.lsb(), ++pos) {
              list[pos] = static_cast<uint16_t>(d * T + i);
              if (a.energy) list2[pos] = static_cast<uint16_t>(eb + d * T + i);
            }
          }
          if (__any_sync(0xffffffffu, has_copy)) {
            int c = 0;
            if (has_copy)
              for_copy_terms<NW, MAXD, true>(st, P, s_inptr, s_inedge, s_src, s_dst, [&](int) { ++c; });
            int chunk_tot;
            int pos = sumR + runC + warp_excl_scan(c, lane, &chunk_tot);
            runC += chunk_tot;
            if (sumR + runC > a.cap) {
              overflow = true;
            } else if (has_copy) {
              for_copy_terms<NW, MAXD, true>(st, P, s_inptr, s_inedge, s_src, s_dst,
                                             [&](int idx) { list[pos++] = static_cast<uint16_t>(idx); });
            }
          }
        }
      }

      // ---- warp reductions for this candidate ----
      fl = __reduce_or_sync(0xffffffffu, fl);
      eq9 = __reduce_add_sync(0xffffffffu, eq9);
      if (eq9 != T) fl |= XE_F_EQ9;
#pragma unroll
      for (int d = 0; d < MAXD; ++d) {
        if (d >= D) continue;
        const int64_t pv = warp_max_u63(pk[d]);
        if (pv > P.budget[d]) fl |= XE_F_BUDGET;
        if (static_cast<double>(pv) > P.ubound[d]) fl |= XE_F_U_BOUND;
        if (lane == 0) slot_peak[s * D + d] = pv;
      }
      if (lane == 0) slot_flags[s] = fl;

      if (EXACT) {
        const int64_t tot = warp_sum_i64(fix);
        if (lane == 0) {
          slot_obj[s] = ldexp(static_cast<double>(tot), -P.fix_k);
          slot_cnt[s] = -1;
        }
      } else if (overflow) {
        if (lane == 0) {
          slot_obj[s] = objective_lane<NW, MAXD>(cw, P, s_tab, s_inptr, s_inedge, s_src, s_dst, a.energy);
          slot_cnt[s] = -1;
        }
      } else if (lane == 0) {
        slot_cnt[s] = sumR + runC;
        slot_cnt2[s] = a.energy ? sumR : 0;
      }
      __syncwarp();
    }

    // ---- chain phase: lane s replays slot s's term list (serial mode) ----
    if (!EXACT && lane < nslot && slot_cnt[lane] >= 0) {
      const uint16_t* l1 = terms + lane * a.cap;
      const uint16_t* l2 = terms2 + lane * a.cap2;
      double total = 0.0;
      const int c1 = slot_cnt[lane], c2 = slot_cnt2[lane];
      for (int j = 0; j < c1; ++j) total = __dadd_rn(total, s_tab[l1[j]]);
      for (int j = 0; j < c2; ++j) total = __dadd_rn(total, s_tab[l2[j]]);
      slot_obj[lane] = total;
    }
    __syncwarp();
    // ---- block outputs (coalesced) ----
    if (lane < nslot) {
      const int64_t c = first + lane;
      const double o = slot_obj[lane];
      const uint32_t f = slot_flags[lane];
      if (a.obj) a.obj[c] = o;
      if (a.flags) a.flags[c] = f;
      if ((f & a.valid_mask) == 0) {
        ++n_valid;
        const uint64_t key = __double_as_longlong(o);
        if (key < best_key || (key == best_key && c < best_idx)) {
          best_key = key;
          best_idx = c;
        }
      }
    }
    if (a.peak)
      for (int i = lane; i < nslot * D; i += 32) a.peak[first * D + i] = slot_peak[i];
    __syncwarp();
  }

  // ---- per-warp best (lexicographic on (objective bits, index)) ----
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t ok = __shfl_xor_sync(0xffffffffu, best_key, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, best_idx, o);
    if (ok < best_key || (ok == best_key && oi >= 0 && (best_idx < 0 || oi < best_idx))) {
      best_key = ok;
      best_idx = oi;
    }
  }
  n_valid = warp_sum_i64(n_valid);
  if (lane == 0) {
    a.wbest_key[gwarp] = best_key;
    a.wbest_idx[gwarp] = best_idx;
    a.wvalid[gwarp] = n_valid;
  }
}

template <int NW, int MAXD, bool EXACT>
int launch_t(const EvalArgs& a, int grid_cap, int smem, cudaStream_t s, int nsm) {
  auto k = eval_cube_kernel<NW, MAXD, EXACT>;
  XE_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 0;
  XE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, a.warps * 32, smem));
  if (per_sm < 1) fail(XE_ERR_TOO_LARGE, "evaluator does not fit on an SM");
  const int grid = std::max(1, std::min(grid_cap, nsm * per_sm));  // persistent: one wave
  k<<<grid, a.warps * 32, smem, s>>>(a);
  XE_CUDA(cudaGetLastError());
  return grid;
}

template <int NW, int MAXD>
int launch_m(const EvalArgs& a, int grid, int smem, cudaStream_t s, int nsm) {
  if (a.P.fix_k >= 0) return launch_t<NW, MAXD, true>(a, grid, smem, s, nsm);
  return launch_t<NW, MAXD, false>(a, grid, smem, s, nsm);
}

template <int NW>
int launch_d(const EvalArgs& a, int grid, int smem, cudaStream_t s, int nsm) {
  switch (a.P.D) {
    case 1: return launch_m<NW, 1>(a, grid, smem, s, nsm);
    case 2: return launch_m<NW, 2>(a, grid, smem, s, nsm);
    case 3: return launch_m<NW, 3>(a, grid, smem, s, nsm);
    case 4: return launch_m<NW, 4>(a, grid, smem, s, nsm);
    default: return launch_m<NW, 8>(a, grid, smem, s, nsm);
  }
}

}  // namespace cube
}  // namespace xe
