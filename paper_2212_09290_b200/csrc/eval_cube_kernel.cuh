// SPDX-License-Identifier: Apache-2.0
#pragma once
//
// K2a — shared definitions of the dense (R,S) cube evaluators: the launch
// arguments and the bit-row helpers used by eval_cube_v3.cuh (one warp per
// candidate, T <= 256) and eval_il.cu (one lane per candidate, T <= 64).
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
// Layout of eval_cube_v3.cuh.  One warp owns one candidate at a time; lanes stride over
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

}  // namespace cube
}  // namespace xe
