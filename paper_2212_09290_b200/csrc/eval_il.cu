// SPDX-License-Identifier: Apache-2.0
//
// K2a v4 — lane-per-candidate evaluation of dense (R,S) cubes stored in the
// candidate-interleaved layout "xe_cube_il" (include/xengine_b200.h):
//
//   u64 word (which, d, t) of candidate c lives at
//       il[((c / 32) * K + ((which * D + d) * T + t)) * 32 + c % 32],
//   K = 2*D*T rows (T <= 64: one u64 per bit row; bit i = operator i).
//
// A warp owns 32 candidates; lane l evaluates candidate 32g+l alone, so
// every global load of the warp is one coalesced 256-byte line and nothing
// is staged in shared memory but the problem tables.  Per candidate it
// computes what the reference composes on the CPU:
//   objective_value      proj/src/model.cpp:369-428  (sequential fp64, same order)
//   complete_assignment  proj/src/model.cpp:471-549  (F hazards, U recurrence)
//   check_assignment     proj/src/model.cpp:430-469  (one XE_F_* bit per family)
//   replay peaks         proj/src/schedule.cpp:326-367
//   decode legality      proj/src/schedule.cpp:40-129
//
// Passes per lane:
//   B  (d-major over R rows)  the compute terms of the objective in the
//      reference's (d,t,i) order, R fixed-zero, EQ8/EQ9 diagonal census,
//      ENERGY_DEV;
//   A  (t-major, all devices' rows of t in registers, t+1 prefetched)  the
//      copy terms continuing the same running sum in (t,e,dc,ds) order,
//      S fixed-zero, EQ11/EQ16_HI, the U recurrence and per-device peaks,
//      EQ12, decode legality, ENERGY_TOTAL;
//   E  (d-major, energy only)  the alpha*q terms.
// Pass A re-reads the R rows pass B just streamed; they come from L2, so
// HBM sees each candidate once.  Built with -fmad=false.
//
// This kernel keeps the reference's summation order term by term; it serves
// the energy model and the exact re-score of the streaming evaluator's
// best-of-batch (eval_stream.cu).

#include "eval_cube_kernel.cuh"

namespace xe {
namespace il {

using cube::eq16_hi;
using cube::for_copy_terms;
using cube::row_peak_general;
using cube::TState;

constexpr int kWarps = 8;
// fixed shared-memory prefix (T <= 64): byte tables [8][256], masses [64],
// parent / consumer masks [64]
constexpr int kOffMtab = 0, kOffMass = 8 * 256 * 8, kOffPmask = kOffMass + 64 * 8, kOffCons = kOffPmask + 64 * 8,
              kFixed = kOffCons + 64 * 8;

struct IlArgs {
  DevProblem P;
  const uint64_t* il;
  int64_t n;
  double* obj;
  int64_t* peak;
  uint32_t* flags;
  int strict, energy;
  uint32_t valid_mask;
  uint64_t* wbest_key;
  int64_t* wbest_idx;
  int64_t* wvalid;
  int copy_in_smem;  // 1: the copy-term table fits in shared memory
  int off_mass, off_pmask, off_cons, off_mtab, off_tab, off_inptr, off_inedge, off_src, off_dst,
      off_ebad, off_q, off_warp, warp_bytes, smem_bytes, q_cap;
};

// Rows holding >= 2 computations (recompute edits) need the free walk of
// row_peak_nw1; a lane meeting one defers it to a per-warp queue, and the
// warp drains the queue one row per lane, so the walk runs at full width
// instead of at the pace of the slowest lane every timestep.
struct PeakRow {
  uint64_t r, z, sn, scan;
  int64_t base;
  int32_t owner;  // lane * MAXD + d
  int32_t pad;
};
// queue capacity: one timestep can add up to 32 * D rows
inline int queue_cap(int D) { return 32 * (D <= 4 ? D : 8) + 32; }

__device__ __forceinline__ int64_t mass_of_bits(uint64_t w, const int64_t* mass) {
  int64_t s = 0;
  while (w) {
    const int b = __ffsll(w) - 1;
    w &= w - 1;
    s += mass[b];
  }
  return s;
}

// Peak of U over the slots of row (d,t) holding >= 2 computations, ascending
// over the computed slots b: U(b) = U(b-1) - freed(b-1) + m_b, sampled after
// the allocation; F(u->b) fires for u in parents(b) + {b} that is resident,
// not kept (S(d,t+1,u) = 0) and has no consumer after b computed on d
// (strict_free: on any device) — model.cpp:492-505, 521-537.
template <class M>
__device__ __noinline__ M row_peak_nw1(uint64_t r, uint64_t z, uint64_t sn, uint64_t scan, M base, int T,
                                       const uint64_t* s_pmask, const uint64_t* s_cons, const M* s_mass) {
  M cur = base, peak = base;
  for (uint64_t rem = r; rem; rem &= rem - 1) {
    const int b = __ffsll(rem) - 1;
    cur += s_mass[b];
    peak = max(peak, cur);
    if (b + 1 >= T) break;
    const uint64_t later = b >= 63 ? 0ull : (~0ull << (b + 1));
    for (uint64_t f = (s_pmask[b] | (1ull << b)) & z & ~sn; f; f &= f - 1) {
      const int u = __ffsll(f) - 1;
      if (!(s_cons[u] & scan & later)) cur -= s_mass[u];
    }
  }
  return peak;
}

__device__ __forceinline__ void smem_max(int32_t* p, int32_t v) { atomicMax(p, v); }
__device__ __forceinline__ void smem_max(int64_t* p, int64_t v) {
  atomicMax(reinterpret_cast<long long*>(p), static_cast<long long>(v));
}

template <int MAXD>
struct Rows3 {  // rows of timestep t (R, S) and t+1 (Sn), passed by value to the rare paths
  uint64_t R[MAXD], S[MAXD], Sn[MAXD];
};

// EQ11 rows of timestep t (S(d,t+1,i) > S(d,t,i) + R(d,t,i)) and the EQ16_HI
// rows that fail with them (eval_cube_kernel.cuh eq16_hi).

template <int MAXD>
__device__ __noinline__ uint32_t eq11_flags(const Rows3<MAXD> rows, int D, int strict, const uint64_t* s_cons) {
  const uint64_t *R = rows.R, *S = rows.S, *Sn = rows.Sn;
  uint64_t allR = ~0ull;
  for (int d = 0; d < D; ++d) allR &= R[d];
  uint32_t fl = 0;
  for (int d = 0; d < D; ++d) {
    const uint64_t bad = Sn[d] & ~(R[d] | S[d]);
    if (!bad) continue;
    Row<1> Rd, Cd, B;
    Rd.w[0] = R[d];
    Cd.w[0] = strict ? allR : R[d];
    B.w[0] = bad;
    fl |= XE_F_EQ11 | eq16_hi<1>(Rd, Cd, B, s_cons);
  }
  return fl;
}


// decode(): a copy for a computation (dc, v <= t) comes from the lowest
// device holding the parent u; illegal when that device freed u at an
// earlier step of timestep t (schedule.cpp:52-71).
template <int MAXD>
__device__ __noinline__ uint32_t decode_freed(const Rows3<MAXD> rows, const Rows3<MAXD> need, uint64_t rany, int t,
                                              int D, int strict, const uint64_t* s_cons) {
  // by value: the caller's row arrays stay in registers (indexing them with a
  // runtime device index here would move them to local memory every step)
  const uint64_t *R = rows.R, *S = rows.S, *Sn = rows.Sn, *needD = need.R;
  uint64_t zany = 0;
  for (int d = 0; d < D; ++d) zany |= R[d] | S[d];
  const uint64_t le_t = t >= 63 ? ~0ull : ((2ull << t) - 1ull);
  for (int dc = 0; dc < D; ++dc) {
    for (uint64_t miss = needD[dc] & ~(R[dc] | S[dc]) & zany; miss; miss &= miss - 1) {
      const int u = __ffsll(miss) - 1;
      int sdev = 0;
      while (!(((R[sdev] | S[sdev]) >> u) & 1ull)) ++sdev;
      if ((Sn[sdev] >> u) & 1ull) continue;  // kept for t+1: never freed
      const uint64_t Rs = R[sdev], cu = s_cons[u];
      int fs = -1;
      const uint64_t cc = cu & (strict ? rany : Rs);
      if (cc) {
        const int mm = 63 - __clzll(cc);
        fs = ((Rs >> mm) & 1ull) ? mm : -1;
      } else if ((Rs >> u) & 1ull) {
        fs = u;
      }
      if (fs < 0) continue;
      const uint64_t vm = cu & R[dc] & le_t;
      const int vmax = vm ? 63 - __clzll(vm) : -1;
      if (fs < vmax || (fs == vmax && sdev < dc)) return XE_F_DECODE | XE_F_DECODE_FREED;
    }
  }
  return 0;
}

// M: integer type of tensor masses and memory sums (int32 when twice the
// save-all total fits, halving the table traffic; int64 otherwise).
// NBYTES: bytes of a bit row summed through the byte tables (4 for T <= 32,
// 6 for T <= 48, else 8; tables beyond the problem's bytes are zero), so
// every lookup is unconditional.
template <int MAXD, class M, int NBYTES>
__global__ void __launch_bounds__(kWarps * 32, MAXD <= 2 ? 3 : (MAXD <= 4 ? 2 : 1)) eval_il_kernel(const IlArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int NW = 1;
  const DevProblem& P = a.P;
  const int D = cube::ndev<MAXD>(P), T = P.T, E = P.E;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;

  // the hottest tables sit at compile-time offsets (immediate LDS offsets)
  M* s_mass = reinterpret_cast<M*>(smem + kOffMass);
  uint64_t* s_pmask = reinterpret_cast<uint64_t*>(smem + kOffPmask);
  uint64_t* s_cons = reinterpret_cast<uint64_t*>(smem + kOffCons);
  M* s_mtab = reinterpret_cast<M*>(smem + kOffMtab);
  double* s_tab = reinterpret_cast<double*>(smem + a.off_tab);
  int32_t* s_inptr = reinterpret_cast<int32_t*>(smem + a.off_inptr);
  int32_t* s_inedge = reinterpret_cast<int32_t*>(smem + a.off_inedge);
  int32_t* s_src = reinterpret_cast<int32_t*>(smem + a.off_src);
  int32_t* s_dst = reinterpret_cast<int32_t*>(smem + a.off_dst);
  uint64_t* s_ebad = reinterpret_cast<uint64_t*>(smem + a.off_ebad);
  double* s_q = reinterpret_cast<double*>(smem + a.off_q);

  // compute terms [D*T] then (energy) alpha*q terms [D*T] always in shared
  // memory; the copy terms [E*D*D] too when they fit, else read through L1
  const int n_dt = D * T, n_copy = E * D * D;
  for (int i = threadIdx.x; i < T; i += blockDim.x) {
    s_mass[i] = static_cast<M>(P.mass[i]);
    s_pmask[i] = P.pmask[i];
    s_cons[i] = P.cons[i];
  }
  for (int i = threadIdx.x; i < NBYTES * 256; i += blockDim.x)
    s_mtab[i] = i < P.NB * 256 ? static_cast<M>(P.mtab[i]) : M(0);
  for (int i = threadIdx.x; i < n_dt; i += blockDim.x) {
    s_tab[i] = P.table[i];
    if (a.energy) s_tab[n_dt + i] = P.table[n_dt + n_copy + i];
  }
  double* s_copy = s_tab + 2 * n_dt;
  if (a.copy_in_smem)
    for (int i = threadIdx.x; i < n_copy; i += blockDim.x) s_copy[i] = P.table[n_dt + i];
  for (int i = threadIdx.x; i <= T; i += blockDim.x) s_inptr[i] = P.in_ptr[i];
  for (int i = threadIdx.x; i < E; i += blockDim.x) {
    s_inedge[i] = P.in_edge[i];
    s_src[i] = P.src[i];
    s_dst[i] = P.dst[i];
  }
  if (a.energy) {
    for (int i = threadIdx.x; i < D; i += blockDim.x) s_ebad[i] = P.ebad[i];
    if (P.has_total)
      for (int i = threadIdx.x; i < n_dt; i += blockDim.x) s_q[i] = P.q[i];
  }
  PeakRow* queue = reinterpret_cast<PeakRow*>(smem + a.off_warp + wid * a.warp_bytes);
  M* s_pk = reinterpret_cast<M*>(queue + a.q_cap);  // [32][MAXD] deferred row peaks
  for (int i = lane; i < 32 * MAXD; i += 32) s_pk[i] = 0;
  __syncthreads();
  const double* copy_glob = P.table + n_dt;  // copy terms in global memory (large E*D*D)
  auto mass_bytes = [&](uint64_t x) {  // mass of a bit row through the byte tables
    M m = 0;
    const uint32_t lo = static_cast<uint32_t>(x), hi = static_cast<uint32_t>(x >> 32);
#pragma unroll
    for (int b = 0; b < NBYTES; ++b) m += s_mtab[b * 256 + (((b < 4 ? lo : hi) >> (8 * (b & 3))) & 0xffu)];
    return m;
  };
  int q_cnt = 0;  // warp-uniform
  auto drain = [&]() {
    __syncwarp();
#pragma unroll 1
    for (int k = lane; k < q_cnt; k += 32) {
      const PeakRow q = queue[k];
      const M rp = row_peak_nw1<M>(q.r, q.z, q.sn, q.scan, static_cast<M>(q.base), T, s_pmask, s_cons, s_mass);
      smem_max(&s_pk[q.owner], rp);
    }
    __syncwarp();
    q_cnt = 0;
  };

  const int64_t gwarp = static_cast<int64_t>(blockIdx.x) * kWarps + wid;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kWarps;
  const int64_t ngroups = (a.n + 31) / 32;
  const int K = 2 * D * T;
  const uint64_t valid = T >= 64 ? ~0ull : ((1ull << T) - 1ull);

  uint64_t best_key = ~0ull;
  int64_t best_idx = -1, n_valid = 0;

  for (int64_t g = gwarp; g < ngroups; g += nwarps) {
    const int64_t c = g * 32 + lane;
    const bool live = c < a.n;
    const uint64_t* cw = a.il + static_cast<size_t>(g) * K * 32 + lane;
    auto ldR = [&](int d, int t) { return __ldg(cw + static_cast<size_t>(d * T + t) * 32) & valid; };
    // device rows are T*32 words apart: offsets fixed per d, one base pointer per t
    const int64_t TS = static_cast<int64_t>(T) * 32;

    uint32_t fl = 0;
    double total = 0.0;
    M pk[MAXD];
#pragma unroll
    for (int d = 0; d < MAXD; ++d) pk[d] = 0;

    {  // padding lanes of the last group evaluate their zero rows; results are dropped
      // ================= pass B: compute terms, d-major =================
      uint64_t diag = 0, multi = 0;
      int eq9 = 0;
      for (int d = 0; d < D; ++d) {
        const uint64_t ebad = a.energy ? s_ebad[d] : 0ull;
        const double* ct = s_tab + d * T;
        // one R row of pass B: the first set bit is handled without a branch
        // (an empty row adds +0.0: the running total is never negative, so
        // that is the identity); further bits (recomputations) loop
        auto row_b = [&](uint64_t r, int tt) {
          const uint64_t above = tt >= 63 ? 0ull : (~0ull << (tt + 1));
          if (r & above) fl |= XE_F_FIXED_ZERO;
          const uint64_t on = (r >> tt) & 1ull;
          eq9 += static_cast<int>(on);
          multi |= diag & (on << tt);
          diag |= on << tt;
          if (r & ebad) fl |= XE_F_ENERGY_DEV;
          const double v0 = ct[r ? __ffsll(r) - 1 : 0];
          total = __dadd_rn(total, r ? v0 : 0.0);
          for (r &= r - 1; r; r &= r - 1) total = __dadd_rn(total, ct[__ffsll(r) - 1]);
        };
        int t = 0;
        for (; t + 4 <= T; t += 4) {
          uint64_t r4[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) r4[j] = ldR(d, t + j);
#pragma unroll
          for (int j = 0; j < 4; ++j) row_b(r4[j], t + j);
        }
        for (; t < T; ++t) row_b(ldR(d, t), t);
      }
      if (diag != valid || multi) fl |= XE_F_EQ8;
      if (eq9 != T) fl |= XE_F_EQ9;

      // ================= pass A: t-major =================
      // rows of t in R[], S[]; rows of t+1 prefetched into Rn[], Sn[]
      uint64_t R[MAXD], S[MAXD], Rn[MAXD], Sn[MAXD];
      const uint64_t* row = cw;  // word (R, d=0, t) of this lane's candidate
#pragma unroll
      for (int d = 0; d < MAXD; ++d) {
        Rn[d] = d < D ? __ldg(row + d * TS) & valid : 0ull;
        Sn[d] = d < D ? __ldg(row + (D + d) * TS) & valid : 0ull;
      }
      const bool by_dst = P.edges_by_dst != 0;
      for (int t = 0; t < T; ++t, row += 32) {
        const bool more = t + 1 < T;
        uint64_t rany = 0, zany = 0, sor = 0, bad = 0;
#pragma unroll
        for (int d = 0; d < MAXD; ++d) {
          R[d] = Rn[d];
          S[d] = Sn[d];
          Rn[d] = (d < D && more) ? __ldg(row + 32 + d * TS) & valid : 0ull;
          Sn[d] = (d < D && more) ? __ldg(row + 32 + (D + d) * TS) & valid : 0ull;
          rany |= R[d];
          zany |= R[d] | S[d];
          sor |= S[d];
          bad |= Sn[d] & ~(R[d] | S[d]);
        }
        if (sor & (t >= 64 ? 0ull : (~0ull << t))) fl |= XE_F_FIXED_ZERO;
        if (bad) {
          Rows3<MAXD> rows;
#pragma unroll
          for (int d = 0; d < MAXD; ++d) {
            rows.R[d] = R[d];
            rows.S[d] = S[d];
            rows.Sn[d] = Sn[d];
          }
          fl |= eq11_flags<MAXD>(rows, D, a.strict, s_cons);
        }

        // ---- U recurrence and per-device peaks (model.cpp:514-537)
#pragma unroll
        for (int d = 0; d < MAXD; ++d) {
          if (d >= D) continue;
          // mass of S(d,t) through the byte tables (branch-free; carrying it
          // across t with sparse bit loops measured 27% slower: divergence)
          const M base = mass_bytes(S[d]);
          const uint64_t r = R[d];
          const bool multi = (r & (r - 1)) != 0;
          const unsigned ballot = __ballot_sync(0xffffffffu, multi);
          if (multi) {
            PeakRow& q = queue[q_cnt + __popc(ballot & ((1u << lane) - 1u))];
            q.r = r;
            q.z = R[d] | S[d];
            q.sn = Sn[d];
            q.scan = a.strict ? rany : r;
            q.base = base;
            q.owner = lane * MAXD + d;
          }
          q_cnt += __popc(ballot);
          pk[d] = max(pk[d], r ? base + s_mass[__ffsll(r) - 1] : base);  // <= the deferred peak when multi
        }
        if (q_cnt > a.q_cap - 32 * D) drain();
        // ---- the computations of timestep t: dependencies (EQ12), decode's
        // copy sources, and (edges sorted by dst) the copy charges in
        // objective_value's (e, dc, ds) order (model.cpp:399-411)
        uint64_t need_all = 0, need_le = 0, needD[MAXD], elsewhere[MAXD];
        int busy = 0;  // devices computing something at t
#pragma unroll
        for (int d = 0; d < MAXD; ++d) {
          needD[d] = 0;
          elsewhere[d] = 0;
          busy += (d < D && R[d] != 0) ? 1 : 0;
#pragma unroll
          for (int x = 0; x < MAXD; ++x)
            if (x < D && x != d) elsewhere[d] |= R[x] | S[x];
        }
        bool copies_left = false;
        auto visit = [&](int v) {
          const uint64_t pm = s_pmask[v];
          need_all |= pm;
          const bool le = v <= t;
          if (le) need_le |= pm;
          bool cp = false;  // some parent of v is held by a device other than a computer of v
#pragma unroll
          for (int dc = 0; dc < MAXD; ++dc) {
            if (dc >= D || !((R[dc] >> v) & 1ull)) continue;
            if (le) needD[dc] |= pm;
            if (pm & elsewhere[dc]) cp = true;
          }
          if (!cp) return;
          if (!by_dst) {
            copies_left = true;
            return;
          }
          for (int k = s_inptr[v]; k < s_inptr[v + 1]; ++k) {
            const int e = s_inedge[k], u = s_src[e];
#pragma unroll
            for (int dc = 0; dc < MAXD; ++dc) {
              if (dc >= D || !((R[dc] >> v) & 1ull)) continue;
#pragma unroll
              for (int ds = 0; ds < MAXD; ++ds)
                if (ds < D && ds != dc && (((R[ds] | S[ds]) >> u) & 1ull)) {
                  const int idx = (e * D + ds) * D + dc;
                  total = __dadd_rn(total, a.copy_in_smem ? s_copy[idx] : __ldg(copy_glob + idx));
                }
            }
          }
        };
        // ascending op order is the copy-charge order; one call site keeps
        // the hot loop small (splitting off the diagonal op t measured equal)
        for (uint64_t rem = rany; rem; rem &= rem - 1) visit(__ffsll(rem) - 1);
        if (need_all & ~zany) fl |= XE_F_EQ12;
        if (need_le & ~zany) fl |= XE_F_DECODE;
        // a copy source can free its tensor within timestep t only if it
        // computes something at t, and it is never the device computing the
        // consumer: a copy can be illegal only when >= 2 devices compute
        if (busy >= 2) {
          uint64_t missing = 0;
#pragma unroll
          for (int d = 0; d < MAXD; ++d)
            if (d < D) missing |= needD[d] & ~(R[d] | S[d]) & zany;
          if (missing) {
            Rows3<MAXD> rows, need;
#pragma unroll
            for (int d = 0; d < MAXD; ++d) {
              rows.R[d] = R[d];
              rows.S[d] = S[d];
              rows.Sn[d] = Sn[d];
              need.R[d] = needD[d];
              need.S[d] = need.Sn[d] = 0;
            }
            fl |= decode_freed<MAXD>(rows, need, rany, t, D, a.strict, s_cons);
          }
        }
        if (copies_left) {  // edge order not monotone in dst: ordered walk
          TState<NW, MAXD> st;
          st.Rany.w[0] = rany;
          st.Zany.w[0] = zany;
#pragma unroll
          for (int d = 0; d < MAXD; ++d) {
            st.R[d].w[0] = R[d];
            st.S[d].w[0] = S[d];
            st.Sn[d].w[0] = Sn[d];
            st.Z[d].w[0] = R[d] | S[d];
          }
          for_copy_terms<NW, MAXD, true>(st, P, s_inptr, s_inedge, s_src, s_dst, [&](int idx) {
            total = __dadd_rn(total, a.copy_in_smem ? s_copy[idx - n_dt] : __ldg(copy_glob + idx - n_dt));
          });
        }
        // ---- ENERGY_TOTAL row of timestep t: sequential (d, i) sum
        if (a.energy && P.has_total) {
          double lhs = 0.0, scale = fmax(1.0, fabs(P.total_rhs));
          for (int d = 0; d < D; ++d) {
            for (uint64_t rr = R[d]; rr; rr &= rr - 1) {
              const double q = s_q[d * T + __ffsll(rr) - 1];
              if (q != 0.0) {
                lhs = __dadd_rn(lhs, q);
                scale = fmax(scale, fabs(q));
              }
            }
          }
          if (__dsub_rn(lhs, P.total_rhs) > 1e-6 * scale) fl |= XE_F_ENERGY_TOTAL;
        }
      }

      if (q_cnt) drain();
#pragma unroll
      for (int d = 0; d < MAXD; ++d) {
        pk[d] = max(pk[d], s_pk[lane * MAXD + d]);
        s_pk[lane * MAXD + d] = 0;
      }

      // ================= pass E: energy terms, d-major =================
      if (a.energy) {
        for (int d = 0; d < D; ++d) {
          const double* et = s_tab + n_dt + d * T;
          for (int t = 0; t < T; ++t)
            for (uint64_t r = ldR(d, t); r; r &= r - 1) total = __dadd_rn(total, et[__ffsll(r) - 1]);
        }
      }

#pragma unroll
      for (int d = 0; d < MAXD; ++d) {
        if (d >= D) continue;
        if (static_cast<int64_t>(pk[d]) > P.budget[d]) fl |= XE_F_BUDGET;
        if (static_cast<double>(pk[d]) > P.ubound[d]) fl |= XE_F_U_BOUND;
      }
      if (live && a.obj) a.obj[c] = total;
      if (live && a.flags) a.flags[c] = fl;
      if (live && a.peak)
#pragma unroll
        for (int d = 0; d < MAXD; ++d)
          if (d < D) a.peak[c * D + d] = static_cast<int64_t>(pk[d]);
      if (live && (fl & a.valid_mask) == 0) {
        ++n_valid;
        const uint64_t key = __double_as_longlong(total);
        if (key < best_key) {  // candidates of a lane ascend: strict < keeps the first
          best_key = key;
          best_idx = c;
        }
      }
    }
  }

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

int align16(int x) { return (x + 15) & ~15; }

template <int MAXD, class M>
int launch_m(const IlArgs& a, cudaStream_t s, int nsm) {
  auto k = a.P.T <= 32 ? eval_il_kernel<MAXD, M, 4> : a.P.T <= 48 ? eval_il_kernel<MAXD, M, 6> : eval_il_kernel<MAXD, M, 8>;
  XE_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, a.smem_bytes));
  int per_sm = 0;
  XE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kWarps * 32, a.smem_bytes));
  if (per_sm < 1) fail(XE_ERR_TOO_LARGE, "interleaved evaluator does not fit on an SM");
  const int64_t ngroups = (a.n + 31) / 32;
  const int64_t need = (ngroups + kWarps - 1) / kWarps;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, static_cast<int64_t>(nsm) * per_sm)));
  k<<<grid, kWarps * 32, a.smem_bytes, s>>>(a);
  XE_CUDA(cudaGetLastError());
  return grid;
}

template <int MAXD>
int launch(const IlArgs& a, cudaStream_t s, int nsm, bool m32) {
  return m32 ? launch_m<MAXD, int32_t>(a, s, nsm) : launch_m<MAXD, int64_t>(a, s, nsm);
}

}  // namespace il

void reduce_best_launch(const uint64_t* key, const int64_t* idx, const int64_t* valid, int n, uint64_t* out,
                        cudaStream_t s);

bool il_supported(const xe_problem* pr) { return pr->h.T <= 64 && pr->h.D <= 8; }

void eval_il_device(const xe_problem* pr, const xe_model_opts& opts, const uint64_t* il, int64_t n, double* obj,
                    int64_t* peak, uint32_t* flags, uint32_t valid_mask, uint64_t* best3, unsigned char* scratch,
                    cudaStream_t stream) {
  using namespace il;
  const HostProblem& h = pr->h;
  if (!h.missing_link.empty() && h.D > 1) fail(XE_ERR_MISSING_LINK, h.missing_link);
  if (!il_supported(pr)) fail(XE_ERR_TOO_LARGE, "interleaved cubes need T <= 64 and D <= 8");
  IlArgs a{};
  a.P = pr->view(opts.use_energy != 0);
  const DevProblem& P = a.P;
  a.il = il;
  a.n = n;
  a.obj = obj;
  a.peak = peak;
  a.flags = flags;
  a.strict = opts.strict_free ? 1 : 0;
  a.energy = (opts.use_energy && h.has_energy) ? 1 : 0;
  a.valid_mask = valid_mask;
  int off = kFixed;
  auto take = [&](int bytes) {
    int o = off;
    off = align16(off + bytes);
    return o;
  };
  // every U value is at most twice the save-all total (a tensor both saved
  // and recomputed in one row is counted twice, model.cpp:517-537)
  int64_t total_mass = 0;
  for (int64_t m : h.mass) total_mass += m;
  const bool m32 = total_mass < (int64_t{1} << 30);
  const int msz = m32 ? 4 : 8;
  const int n_dt = P.D * P.T, n_copy = P.E * P.D * P.D;
  a.off_mass = kOffMass;
  a.off_pmask = kOffPmask;
  a.off_cons = kOffCons;
  a.off_mtab = kOffMtab;
  a.off_inptr = take(4 * (P.T + 1));
  a.off_inedge = take(4 * std::max(1, P.E));
  a.off_src = take(4 * std::max(1, P.E));
  a.off_dst = take(4 * std::max(1, P.E));
  a.off_ebad = take(8 * P.D);
  a.off_q = take(a.energy && P.has_total ? 8 * n_dt : 8);
  a.copy_in_smem = (off + 8 * (2 * n_dt + n_copy) <= 64 * 1024) ? 1 : 0;
  a.off_tab = take(8 * (2 * n_dt + (a.copy_in_smem ? n_copy : 0)));
  a.off_warp = off;
  a.q_cap = queue_cap(P.D);
  const int maxd = P.D <= 4 ? P.D : 8;
  a.warp_bytes = align16(static_cast<int>(sizeof(PeakRow)) * a.q_cap + msz * 32 * maxd);
  a.smem_bytes = off + kWarps * a.warp_bytes;

  int nsm = 0;
  XE_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, pr->device));
  const size_t nw_max = static_cast<size_t>(nsm) * 8 * cube::kWarps;  // eval_scratch_bytes layout
  a.wbest_key = reinterpret_cast<uint64_t*>(scratch);
  a.wbest_idx = reinterpret_cast<int64_t*>(scratch + nw_max * 8);
  a.wvalid = reinterpret_cast<int64_t*>(scratch + nw_max * 16);
  int grid = 0;
  if (n > 0) {
    switch (P.D) {
      case 1: grid = launch<1>(a, stream, nsm, m32); break;
      case 2: grid = launch<2>(a, stream, nsm, m32); break;
      case 3: grid = launch<3>(a, stream, nsm, m32); break;
      case 4: grid = launch<4>(a, stream, nsm, m32); break;
      default: grid = launch<8>(a, stream, nsm, m32); break;
    }
    if (static_cast<size_t>(grid) * kWarps > nw_max) fail(XE_ERR_ARG, "evaluator scratch too small");
  }
  if (best3) {
    if (n > 0) {
      reduce_best_launch(a.wbest_key, a.wbest_idx, a.wvalid, grid * kWarps, best3, stream);
    } else {
      const uint64_t none[3] = {~0ull, ~0ull, 0ull};
      XE_CUDA(cudaMemcpyAsync(best3, none, sizeof none, cudaMemcpyHostToDevice, stream));
    }
  }
}

}  // namespace xe
