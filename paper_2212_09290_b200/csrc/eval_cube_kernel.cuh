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
// timesteps t, every device's rows of that t in registers.  The candidate
// (8*D*T*W bytes) is staged global->shared by the bulk-copy (TMA) engine,
// double-buffered per warp behind an mbarrier, so HBM streams while the
// previous candidate is evaluated.  Problem tables (masses, parent/consumer
// masks, mass byte-tables, objective terms) live in shared memory per CTA.
//
// Objective.  Two modes, both bit-identical to the reference's sequential
// double sum:
//   EXACT  every term is k-bit dyadic and the worst-case total < 2^52 units
//          (xe::exact_fix_k) -> int64 fixed-point sums, any order, warp reduce.
//   serial otherwise: the warp writes each candidate's term indices in the
//          reference loop order into a per-slot list; after SLOTS candidates
//          lane s replays slot s's list with sequential FP64 adds (no FMA).

#include <cfloat>
#include <climits>

#include "bits.cuh"
#include "xe_internal.hpp"

namespace xe {
namespace cube {

constexpr int kWarps = 8;
constexpr int kSlots = 16;

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
  int warp_bytes, off_w_stage, off_w_bar, off_w_terms, off_w_slot;
  int stages, cap, use_bulk;
  int warps;  // warps per CTA (shared-memory plan decides, <= kWarps)
  uint32_t cube_words;
};

template <int NW>
__device__ __forceinline__ int64_t mass_bytes(const Row<NW>& r, const int64_t* mtab, int NB) {
  int64_t s = 0;
#pragma unroll
  for (int j = 0; j < NW; ++j) {
    uint64_t w = r.w[j];
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      int idx = 8 * j + b;
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
      int b = __ffsll(w) - 1;
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
  const uint32_t* p = cw + ((static_cast<size_t>(which) * D + d) * T + t) * W32;
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

template <int NW, int MAXD>
__device__ __forceinline__ void load_t(TState<NW, MAXD>& st, const uint32_t* cw, const DevProblem& P,
                                       int t, bool active) {
  st.Rany = Row<NW>::zero();
  st.Zany = Row<NW>::zero();
  const Row<NW> valid = Row<NW>::below(P.T);  // padding bits >= T are not variables
#pragma unroll
  for (int d = 0; d < MAXD; ++d) {
    if (d < P.D && active) {
      st.R[d] = cube_row<NW>(cw, P.W32, P.D, P.T, 0, d, t) & valid;
      st.S[d] = cube_row<NW>(cw, P.W32, P.D, P.T, 1, d, t) & valid;
      st.Sn[d] = (t + 1 < P.T) ? (cube_row<NW>(cw, P.W32, P.D, P.T, 1, d, t + 1) & valid) : Row<NW>::zero();
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
  if (P.D < 2 || !st.Rany.any()) return;
  const int base = P.D * P.T;
  auto one_edge = [&](int e) {
    const int u = s_src[e], v = s_dst[e];
#pragma unroll
    for (int dc = 0; dc < MAXD; ++dc) {
      if (dc >= P.D || !st.R[dc].test(v)) continue;
#pragma unroll
      for (int ds = 0; ds < MAXD; ++ds) {
        if (ds >= P.D || ds == dc || !st.Z[ds].test(u)) continue;
        fn(base + (e * P.D + ds) * P.D + dc);
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
        int v = 64 * j + __ffsll(w) - 1;
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
          int v = 64 * j + __ffsll(w) - 1;
          w &= w - 1;
          for (int k = s_inptr[v]; k < s_inptr[v + 1]; ++k) {
            int e = s_inedge[k];
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

// Sequential objective by one lane straight from the staged cube — used
// only when a candidate's term list exceeds the per-slot capacity.
template <int NW, int MAXD>
__device__ double objective_lane(const uint32_t* cw, const DevProblem& P, const double* tab,
                                 const int32_t* s_inptr, const int32_t* s_inedge,
                                 const int32_t* s_src, const int32_t* s_dst, int energy) {
  double total = 0.0;
  for (int d = 0; d < P.D; ++d)
    for (int t = 0; t < P.T; ++t) {
      Row<NW> r = cube_row<NW>(cw, P.W32, P.D, P.T, 0, d, t) & Row<NW>::below(P.T);
      for (int i = r.lsb(); i >= 0; r.clear(i), i = r.lsb()) total = __dadd_rn(total, tab[d * P.T + i]);
    }
  for (int t = 0; t < P.T; ++t) {
    TState<NW, MAXD> st;
    load_t<NW, MAXD>(st, cw, P, t, true);
    for_copy_terms<NW, MAXD, true>(st, P, s_inptr, s_inedge, s_src, s_dst,
                                   [&](int idx) { total = __dadd_rn(total, tab[idx]); });
  }
  if (energy) {
    const int eb = P.D * P.T + P.E * P.D * P.D;
    for (int d = 0; d < P.D; ++d)
      for (int t = 0; t < P.T; ++t) {
        Row<NW> r = cube_row<NW>(cw, P.W32, P.D, P.T, 0, d, t) & Row<NW>::below(P.T);
        for (int i = r.lsb(); i >= 0; r.clear(i), i = r.lsb()) total = __dadd_rn(total, tab[eb + d * P.T + i]);
      }
  }
  return total;
}

template <int NW, int MAXD, bool EXACT>
__global__ void __launch_bounds__(kWarps * 32) eval_cube_kernel(const EvalArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const DevProblem& P = a.P;
  const int D = P.D, T = P.T, E = P.E;
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
  double* slot_obj = reinterpret_cast<double*>(wreg + a.off_w_slot);
  uint32_t* slot_flags = reinterpret_cast<uint32_t*>(slot_obj + kSlots);
  int32_t* slot_cnt = reinterpret_cast<int32_t*>(slot_flags + kSlots);
  int64_t* slot_peak = reinterpret_cast<int64_t*>(slot_cnt + kSlots);  // [kSlots][D]

  if (lane == 0)
    for (int s = 0; s < a.stages; ++s) mbar_init(&bars[s], 1);
  fence_mbar_init();
  __syncthreads();

  const int64_t gwarp = static_cast<int64_t>(blockIdx.x) * a.warps + wid;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * a.warps;
  const int64_t nblocks = (a.n + kSlots - 1) / kSlots;
  const uint32_t cube_bytes = a.cube_words * 4u;

  uint64_t best_key = ~0ull;
  int64_t best_idx = -1, n_valid = 0;

  // candidate sequence of this warp: blocks gwarp, gwarp+nwarps, ...; slots 0..15
  auto cand_of = [&](int64_t k) -> int64_t {  // k-th candidate of this warp
    int64_t blk = gwarp + (k / kSlots) * nwarps;
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

  uint32_t phase_bits = 0;  // per-stage parity
  int64_t k = 0;
  if (gwarp < nblocks) issue(cand_of(0), 0);

  for (int64_t blk = gwarp; blk < nblocks; blk += nwarps) {
    const int64_t first = blk * kSlots;
    const int nslot = static_cast<int>(a.n - first < kSlots ? a.n - first : kSlots);
    for (int s = 0; s < nslot; ++s, ++k) {
      const int stage = static_cast<int>(k % a.stages);
      // prefetch the next candidate of this warp into the next stage
      {
        int64_t nk = k + 1;
        int64_t nc = (nk % kSlots == 0) ? cand_of(nk) : (first + s + 1 < first + nslot ? first + s + 1 : a.n);
        if (nk % kSlots == 0 && nc >= a.n) nc = a.n;
        issue(nc, static_cast<int>(nk % a.stages));
      }
      if (a.use_bulk) {
        mbar_wait(&bars[stage], (phase_bits >> stage) & 1u);
        phase_bits ^= 1u << stage;
      }
      const uint32_t* cw = stage_buf + static_cast<size_t>(stage) * a.cube_words;

      // ================= pass 1: validity, memory, term counts =================
      uint32_t fl = 0;
      int eq9 = 0;
      int64_t pk[MAXD];
      int cntR[MAXD];
#pragma unroll
      for (int d = 0; d < MAXD; ++d) {
        pk[d] = 0;
        cntR[d] = 0;
      }
      int cntC = 0;
      int64_t fix = 0;

      for (int t0 = 0; t0 < T; t0 += 32) {
        const int t = t0 + lane;
        const bool act = t < T;
        TState<NW, MAXD> st;
        load_t<NW, MAXD>(st, cw, P, t, act);
        if (act) {
          const Row<NW> above_t = Row<NW>::above(t), ge_t = Row<NW>::at_or_above(t);
          int nd = 0;
#pragma unroll
          for (int d = 0; d < MAXD; ++d) {
            if (d >= D) continue;
            if ((st.R[d] & above_t).any() || (st.S[d] & ge_t).any()) fl |= XE_F_FIXED_ZERO;
            nd += st.R[d].test(t);
          }
          if (nd != 1) fl |= XE_F_EQ8;
          eq9 += nd;

          // EQ11 (+ the EQ16_HI rows that can only fail with it)
          Row<NW> allR = st.R[0];
#pragma unroll
          for (int d = 1; d < MAXD; ++d)
            if (d < D) allR = allR & st.R[d];
#pragma unroll
          for (int d = 0; d < MAXD; ++d) {
            if (d >= D) continue;
            Row<NW> bad = andnot(st.Sn[d], st.Z[d]);
            if (!bad.any()) continue;
            fl |= XE_F_EQ11;
            const Row<NW> Cd = a.strict ? allR : st.R[d];
            for (int u = bad.lsb(); u >= 0; bad.clear(u), u = bad.lsb()) {
              Row<NW> cu = load_row<NW>(s_cons + u * NW);
              bool hi = !andnot(cu, Cd).any();  // self edge F(u,u)
              for (Row<NW> cv = cu; !hi && cv.any();) {
                int v = cv.lsb();
                cv.clear(v);
                if (!st.R[d].test(v) && !andnot(cu & Row<NW>::above(v), Cd).any()) hi = true;
              }
              if (hi) fl |= XE_F_EQ16_HI;
            }
          }
          if (a.energy) {
#pragma unroll
            for (int d = 0; d < MAXD; ++d)
              if (d < D && (st.R[d] & load_row<NW>(s_ebad + d * NW)).any()) fl |= XE_F_ENERGY_DEV;
          }

          // ---- memory: U recurrence per device, frees per Eq.16 hazards ----
          int64_t base[MAXD], acc[MAXD], mx[MAXD], sR[MAXD], sF[MAXD];
          Row<NW> seen[MAXD], needD[MAXD];
#pragma unroll
          for (int d = 0; d < MAXD; ++d) {
            base[d] = (d < D) ? mass_bytes<NW>(st.S[d], s_mtab, P.NB) : 0;
            acc[d] = 0;
            mx[d] = LLONG_MIN;
            sR[d] = 0;
            sF[d] = 0;
            seen[d] = Row<NW>::zero();
            needD[d] = Row<NW>::zero();
          }
          Row<NW> seen_all = Row<NW>::zero(), need_all = Row<NW>::zero(), need_le = Row<NW>::zero();
          for (int v = st.Rany.msb(); v >= 0;) {
            const Row<NW> pm = load_row<NW>(s_pmask + v * NW);
            const int64_t mv = s_mass[v];
            need_all = need_all | pm;
            if (v <= t) need_le = need_le | pm;
#pragma unroll
            for (int d = 0; d < MAXD; ++d) {
              if (d >= D || !st.R[d].test(v)) continue;
              Row<NW> f = pm;
              f.set(v);
              f = andnot(andnot(f & st.Z[d], st.Sn[d]), a.strict ? seen_all : seen[d]);
              const int64_t fm = mass_bits<NW>(f, s_mass);
              mx[d] = max(mx[d], acc[d] + fm);
              acc[d] += fm - mv;
              sR[d] += mv;
              sF[d] += fm;
              seen[d] = seen[d] | pm;
              if (v <= t) needD[d] = needD[d] | pm;
            }
            seen_all = seen_all | pm;
            // next lower set bit of Rany
            Row<NW> rest = st.Rany & ~Row<NW>::at_or_above(v);
            v = rest.msb();
          }
#pragma unroll
          for (int d = 0; d < MAXD; ++d) {
            if (d >= D) continue;
            int64_t rp = base[d];
            if (sR[d] > 0) rp = max(rp, base[d] + sR[d] - sF[d] + mx[d]);
            pk[d] = max(pk[d], rp);
          }
          if (andnot(need_all, st.Zany).any()) fl |= XE_F_EQ12;
          if (andnot(need_le, st.Zany).any()) fl |= XE_F_DECODE;

          // decode: copy source freed earlier in this timestep (schedule.cpp:68-71)
#pragma unroll
          for (int d = 0; d < MAXD; ++d) {
            if (d >= D) continue;
            Row<NW> miss = andnot(needD[d], st.Z[d]) & st.Zany;
            for (int u = miss.lsb(); u >= 0; miss.clear(u), u = miss.lsb()) {
              int sdev = 0;
#pragma unroll
              for (int x = MAXD - 1; x >= 0; --x)
                if (x < D && st.Z[x].test(u)) sdev = x;
              int fs = -1;
              Row<NW> Rs;
#pragma unroll
              for (int x = 0; x < MAXD; ++x)
                if (x == sdev) Rs = st.R[x];
              bool keep = false;
#pragma unroll
              for (int x = 0; x < MAXD; ++x)
                if (x == sdev) keep = st.Sn[x].test(u);
              if (!keep) {
                const Row<NW> cu = load_row<NW>(s_cons + u * NW);
                if (a.strict) {
                  Row<NW> c = cu & st.Rany;
                  if (c.any()) {
                    int m = c.msb();
                    fs = Rs.test(m) ? m : -1;
                  } else if (Rs.test(u)) {
                    fs = u;
                  }
                } else {
                  Row<NW> c = cu & Rs;
                  if (c.any()) fs = c.msb();
                  else if (Rs.test(u)) fs = u;
                }
              }
              if (fs >= 0) {
                Row<NW> cv = load_row<NW>(s_cons + u * NW) & st.R[d] & ~Row<NW>::above(t);
                int vmax = cv.msb();
                if (fs < vmax || (fs == vmax && sdev < d)) fl |= XE_F_DECODE | XE_F_DECODE_FREED;
              }
            }
          }

          // ENERGY_TOTAL row of timestep t: sequential sum in (d, i) order
          if (a.energy && P.has_total) {
            double lhs = 0.0, scale = fmax(1.0, fabs(P.total_rhs));
            for (int d = 0; d < D; ++d) {
              Row<NW> r;
#pragma unroll
              for (int x = 0; x < MAXD; ++x)
                if (x == d) r = st.R[x];
              for (int i = r.lsb(); i >= 0; r.clear(i), i = r.lsb()) {
                double q = s_q[d * T + i];
                if (q != 0.0) {
                  lhs = __dadd_rn(lhs, q);
                  scale = fmax(scale, fabs(q));
                }
              }
            }
            if (__dsub_rn(lhs, P.total_rhs) > 1e-6 * scale) fl |= XE_F_ENERGY_TOTAL;
          }
        }

        // ---- objective terms ----
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
            for_copy_terms<NW, MAXD, false>(st, P, s_inptr, s_inedge, s_src, s_dst,
                                            [&](int idx) { fix += s_tfix[idx]; });
          }
        } else {
#pragma unroll
          for (int d = 0; d < MAXD; ++d)
            if (d < D) cntR[d] += st.R[d].popc();
          for_copy_terms<NW, MAXD, false>(st, P, s_inptr, s_inedge, s_src, s_dst,
                                          [&](int) { ++cntC; });
        }
      }

      // ---- warp reductions for this candidate ----
      fl = __reduce_or_sync(0xffffffffu, fl);
      eq9 = __reduce_add_sync(0xffffffffu, eq9);
      if (eq9 != T) fl |= XE_F_EQ9;
      int64_t peakv[MAXD];
#pragma unroll
      for (int d = 0; d < MAXD; ++d) {
        peakv[d] = (d < D) ? warp_max_i64(pk[d]) : 0;
        if (d < D) {
          if (peakv[d] > P.budget[d]) fl |= XE_F_BUDGET;
          if (static_cast<double>(peakv[d]) > P.ubound[d]) fl |= XE_F_U_BOUND;
        }
      }
      const int64_t cidx = first + s;
      if (lane == 0) {
        slot_flags[s] = fl;
#pragma unroll
        for (int d = 0; d < MAXD; ++d)
          if (d < D) slot_peak[s * D + d] = peakv[d];
      }

      if (EXACT) {
        int64_t tot = warp_sum_i64(fix);
        if (lane == 0) {
          slot_obj[s] = ldexp(static_cast<double>(tot), -P.fix_k);
          slot_cnt[s] = -1;
        }
      } else {
        // ================= pass 2: term lists in reference order =================
        int totR[MAXD], baseR[MAXD];
        int sumR = 0;
#pragma unroll
        for (int d = 0; d < MAXD; ++d) {
          totR[d] = (d < D) ? __reduce_add_sync(0xffffffffu, cntR[d]) : 0;
          baseR[d] = sumR;
          sumR += totR[d];
        }
        const int totC = __reduce_add_sync(0xffffffffu, cntC);
        const int total = sumR + totC + (a.energy ? sumR : 0);
        if (total > a.cap) {
          double v = 0.0;
          if (lane == 0)
            v = objective_lane<NW, MAXD>(cw, P, s_tab, s_inptr, s_inedge, s_src, s_dst, a.energy);
          if (lane == 0) {
            slot_obj[s] = v;
            slot_cnt[s] = -1;
          }
        } else {
          uint16_t* list = terms + s * a.cap;
          int runR[MAXD];
#pragma unroll
          for (int d = 0; d < MAXD; ++d) runR[d] = 0;
          int runC = 0;
          const int eb = D * T + E * D * D;
          for (int t0 = 0; t0 < T; t0 += 32) {
            const int t = t0 + lane;
            const bool act = t < T;
            TState<NW, MAXD> st;
            load_t<NW, MAXD>(st, cw, P, t, act);
#pragma unroll
            for (int d = 0; d < MAXD; ++d) {
              if (d >= D) continue;
              int chunk_tot;
              int pos = baseR[d] + runR[d] + warp_excl_scan(st.R[d].popc(), lane, &chunk_tot);
              runR[d] += chunk_tot;
              Row<NW> r = st.R[d];
              for (int i = r.lsb(); i >= 0; r.clear(i), i = r.lsb(), ++pos) {
                list[pos] = static_cast<uint16_t>(d * T + i);
                if (a.energy) list[pos + sumR + totC] = static_cast<uint16_t>(eb + d * T + i);
              }
            }
            int c = 0;
            for_copy_terms<NW, MAXD, true>(st, P, s_inptr, s_inedge, s_src, s_dst, [&](int) { ++c; });
            int chunk_tot;
            int pos = sumR + runC + warp_excl_scan(c, lane, &chunk_tot);
            runC += chunk_tot;
            for_copy_terms<NW, MAXD, true>(st, P, s_inptr, s_inedge, s_src, s_dst,
                                           [&](int idx) { list[pos++] = static_cast<uint16_t>(idx); });
          }
          if (lane == 0) slot_cnt[s] = total;
        }
      }
      __syncwarp();
      (void)cidx;
    }

    // ---- chain phase: lane s replays slot s's term list (serial mode) ----
    if (!EXACT && lane < nslot && slot_cnt[lane] >= 0) {
      const uint16_t* list = terms + lane * a.cap;
      double total = 0.0;
      const int cnt = slot_cnt[lane];
      for (int j = 0; j < cnt; ++j) total = __dadd_rn(total, s_tab[list[j]]);
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
    uint64_t ok = __shfl_xor_sync(0xffffffffu, best_key, o);
    int64_t oi = __shfl_xor_sync(0xffffffffu, best_idx, o);
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
  int grid = std::max(1, std::min(grid_cap, nsm * per_sm));  // persistent: one wave
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
  if (a.P.D <= 2) return launch_m<NW, 2>(a, grid, smem, s, nsm);
  if (a.P.D <= 4) return launch_m<NW, 4>(a, grid, smem, s, nsm);
  return launch_m<NW, 8>(a, grid, smem, s, nsm);
}

}  // namespace cube
}  // namespace xe
