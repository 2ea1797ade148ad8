// SPDX-License-Identifier: Apache-2.0
#pragma once
//
// K2a v5 — streaming lane-per-candidate evaluation of dense (R,S) cubes in the
// candidate-interleaved layout "xe_cube_il" generalised to NW u64 words per
// bit row (T <= 64*NW, NW <= 4):
//
//   u64 word j of row (which, d, t) of candidate c lives at
//       il[((c / 32) * K + ((which * D + d) * T + t) * NW + j) * 32 + c % 32],
//   K = 2*D*T*NW  (NW = 1 is the round-1 T <= 64 layout, unchanged).
//
// Per candidate it computes what the reference composes on the CPU:
//   objective_value      proj/src/model.cpp:369-428
//   complete_assignment  proj/src/model.cpp:471-549  (F hazards, U recurrence)
//   check_assignment     proj/src/model.cpp:430-469  (one XE_F_* bit per family)
//   replay peaks         proj/src/schedule.cpp:326-367
//   decode legality      proj/src/schedule.cpp:40-129
//
// One pass over t.  Every lane runs the same branch-free code for every
// timestep ("fast" timestep = only the diagonal operator t is computed, on
// exactly one device — what a placement with minimal saves looks like):
//   loads of the 2*D*NW words of t, S fixed-zero, the S-row masses (byte
//   tables), EQ11 bits (S(t) against Z(t-1)), the compute term c[d*][t], the
//   copy charges of t's in-edges, EQ12/decode for t's parents, and the peaks
//   base_d + [d = d*] m_t.
// A timestep that is not fast (recomputations, several devices computing,
// an off-diagonal R bit, an EQ11 violation) is pushed as a 4-byte job onto a
// per-warp shared-memory queue; when the queue fills (and at the end of each
// 32-candidate group) the warp drains it at full width: lane k takes job k,
// reloads that timestep's rows (L2-resident: the warp just streamed them)
// and runs the general code (every term of the timestep, F-hazard free walks
// for rows with >= 2 computations, EQ16_HI with EQ11, decode's freed-source
// check).  Flags, EQ9 counts and peaks merge through order-free shared
// atomics; objective parts are summed by the owner in timestep order.
//
// Objective order.  The reference sums sequentially in (d,t,i) then
// (t,e,dc,ds) order; here each timestep's terms are summed t-major (fast
// timesteps into one running sum, deferred ones into a second, added at the
// end): a reassociation within (#terms * 2^-53) relative of the reference
// (north_star tolerance 1e-6; tested at 1e-12), and bit-identical when every
// term is dyadic (xe::exact_fix_k >= 0: every partial sum is exact).  The
// best-of-batch is then re-scored in the reference's order (refine_best in
// eval_stream.cu), so the reported winner and its objective bits are exactly
// the reference's argmin (solver.cpp:57-61 first-minimum rule).

#include "eval_cube_kernel.cuh"

namespace xe {
namespace st {

constexpr int kWarps = 8;
constexpr int kQCap = 192;  // queue jobs per warp (one timestep adds <= 64)
#ifndef XE_PREFETCH
#define XE_PREFETCH 2
#endif
constexpr int kPrefetch = XE_PREFETCH;  // timesteps ahead (multi-word rows)
#ifndef XE_T_UNROLL
#define XE_T_UNROLL 1
#endif
constexpr int kTUnroll = XE_T_UNROLL;  // unroll of the streaming pass over t
#ifndef XE_PF_REG
#define XE_PF_REG 1
#endif
constexpr bool kPfReg = XE_PF_REG;  // small rows: next timestep double-buffered in registers
// multi-word rows: a smaller queue keeps two CTAs per SM within shared memory
__host__ __device__ constexpr int qcap(int nw) { return nw == 1 ? kQCap : 128; }
constexpr int kKindA = 1;   // full general timestep
constexpr int kKindB = 2;   // EQ11 / EQ16_HI rows of the timestep

struct Job {
  uint32_t meta;  // t (bits 0..9) | owner lane (10..14) | kind (15..16)
  uint32_t next;  // the owner's next kind-A job in this queue window
  double part;    // objective part of a kind-A job (filled by the worker)
};

struct StArgs {
  DevProblem P;
  const uint64_t* il;
  int64_t n;
  double* obj;
  int64_t* peak;
  uint32_t* flags;
  int strict;
  uint32_t valid_mask;
  uint64_t* wbest_key;
  int64_t* wbest_idx;
  int64_t* wvalid;
  int off_mass, off_pmask, off_cons, off_c, off_w, off_inl, off_inptr, off_inedge, off_src, off_dst, off_warp;
  int warp_bytes, smem_bytes;
};

template <class M>
struct Sm {
  const M* mtab;
  const M* mass;
  const uint64_t* pmask;
  const uint64_t* cons;
  const double* c;
  const double* w;
  const int32_t *inptr, *inedge, *src, *dst;
  uint32_t* fl;   // [32] per-lane flag merges (this warp)
  int32_t* cnt;   // [32] per-lane EQ9 diagonal counts of deferred timesteps
  M* pk;          // [32][MAXD] per-lane deferred row peaks
};

__device__ __forceinline__ void smem_max(int32_t* p, int32_t v) { atomicMax(p, v); }
__device__ __forceinline__ void smem_max(int64_t* p, int64_t v) {
  atomicMax(reinterpret_cast<long long*>(p), static_cast<long long>(v));
}

template <int NW, class M>
__device__ __forceinline__ M mass_of(Row<NW> r, const M* mass) {
  M s = 0;
#pragma unroll
  for (int j = 0; j < NW; ++j)
    for (uint64_t w = r.w[j]; w; w &= w - 1) s += mass[64 * j + __ffsll(w) - 1];
  return s;
}

// Peak of U over row (d,t) holding >= 2 computations: the descending form of
// the recurrence U(v+1) = U(v) - freed(v) + R(v+1) m_{v+1}
// (model.cpp:514-537): F(u->v) fires for u in parents(v)+{v} resident on d,
// not kept (S(d,t+1,u) = 0) and with no later consumer in `scan` (R(d,t,.),
// or every device's R with strict_free) — model.cpp:492-505.
template <int NW, class M>
__device__ __noinline__ M row_peak(Row<NW> Rd, Row<NW> Zd, Row<NW> Snd, Row<NW> scan, M base,
                                   const uint64_t* pmask, const M* mass) {
  Row<NW> seen = Row<NW>::zero();
  int64_t acc = 0, mx = INT64_MIN, sR = 0, sF = 0;
  for (int v = scan.msb(); v >= 0;) {
    const Row<NW> pm = load_row<NW>(pmask + v * NW);
    if (Rd.test(v)) {
      Row<NW> f = pm;
      f.set(v);
      f = andnot(andnot(f & Zd, Snd), seen);
      const int64_t fm = static_cast<int64_t>(mass_of<NW, M>(f, mass)), mv = mass[v];
      mx = max(mx, acc + fm);
      acc += fm - mv;
      sR += mv;
      sF += fm;
    }
    seen = seen | pm;
    v = (scan & ~Row<NW>::at_or_above(v)).msb();
  }
  return static_cast<M>(max(static_cast<int64_t>(base), static_cast<int64_t>(base) + sR - sF + mx));
}

// The general timestep (a queued job): reloads rows t (and S of t+1) of the
// owner's candidate and evaluates them without any fast-path assumption.
// Kind A returns the timestep's objective part (compute terms in (d,i)
// order, then copy charges) and merges flags / EQ9 count / row peaks into the
// owner's shared slots; kind B merges the EQ11 and EQ16_HI bits.
// Mass of the tensors of a bit row through the shared tables (the same
// lookups as the streaming pass): TB = 8 byte tables, or TB = 11 chunks.
template <int NW, class M, int NBL, int TB>
__device__ __forceinline__ M table_mass(const Row<NW>& r, const M* mtab) {
  M m = 0;
  if (TB == 8) {
#pragma unroll
    for (int j = 0; j < NW; ++j) {
      const uint32_t lo = static_cast<uint32_t>(r.w[j]), hi = static_cast<uint32_t>(r.w[j] >> 32);
#pragma unroll
      for (int b = 0; b < (j == NW - 1 ? NBL : 8); ++b)
        m += mtab[(8 * j + b) * 256 + (((b < 4 ? lo : hi) >> (8 * (b & 3))) & 0xffu)];
    }
  } else {
#pragma unroll
    for (int c = 0; c < NBL; ++c) m += mtab[c * 2048 + static_cast<int>((r.w[0] >> (11 * c)) & 0x7ffull)];
  }
  return m;
}

template <int MAXD, int NW, class M, int NBL, int TB>
__device__ __forceinline__ double run_job(const uint64_t* cwo, int t, int kind, int owner, const StArgs* ap,
                                       const Sm<M> sm) {
  const StArgs& a = *ap;
  const DevProblem& P = a.P;
  const int D = cube::ndev<MAXD>(P), T = P.T;
  const Row<NW> valid = Row<NW>::below(T);
  auto ld = [&](int which, int d, int tt) {
    Row<NW> r;
    const uint64_t* p = cwo + (static_cast<int64_t>(which * D + d) * T + tt) * NW * 32;
#pragma unroll
    for (int j = 0; j < NW; ++j) r.w[j] = p[j * 32];
    return r & valid;
  };
  cube::TState<NW, MAXD> st;
  st.Rany = Row<NW>::zero();
  st.Zany = Row<NW>::zero();
#pragma unroll
  for (int d = 0; d < MAXD; ++d) {
    if (d < D) {
      st.R[d] = ld(0, d, t);
      st.S[d] = ld(1, d, t);
      st.Sn[d] = t + 1 < T ? ld(1, d, t + 1) : Row<NW>::zero();
    } else {
      st.R[d] = st.S[d] = st.Sn[d] = Row<NW>::zero();
    }
    st.Z[d] = st.R[d] | st.S[d];
    st.Rany = st.Rany | st.R[d];
    st.Zany = st.Zany | st.Z[d];
  }
  uint32_t fl = 0;
  double part = 0.0;
  if (kind == kKindB) {
    Row<NW> allR = ~Row<NW>::zero();
#pragma unroll
    for (int d = 0; d < MAXD; ++d)
      if (d < D) allR = allR & st.R[d];
#pragma unroll
    for (int d = 0; d < MAXD; ++d) {
      if (d >= D) continue;
      const Row<NW> bad = andnot(st.Sn[d], st.Z[d]);
      if (bad.any()) fl |= XE_F_EQ11 | cube::eq16_hi<NW>(st.R[d], a.strict ? allR : st.R[d], bad, sm.cons);
    }
    if (fl) atomicOr(&sm.fl[owner], fl);
    return 0.0;
  }
  // ---- kind A
  const Row<NW> above = Row<NW>::above(t);
  int busy = 0, cnt = 0;
#pragma unroll
  for (int d = 0; d < MAXD; ++d) {
    if (d >= D) continue;
    busy += st.R[d].any() ? 1 : 0;
    cnt += st.R[d].test(t) ? 1 : 0;
    if ((st.R[d] & above).any()) fl |= XE_F_FIXED_ZERO;
  }
  if (cnt != 1) fl |= XE_F_EQ8;
  atomicAdd(&sm.cnt[owner], cnt);
  // compute terms (model.cpp:392-397), then copy charges (model.cpp:399-411)
#pragma unroll
  for (int d = 0; d < MAXD; ++d) {
    if (d >= D) continue;
    for (Row<NW> r = st.R[d]; r.any();) {
      const int i = r.lsb();
      r.clear(i);
      part = __dadd_rn(part, sm.c[d * T + i]);
    }
  }
  const int n_dt = D * T;
  cube::for_copy_terms<NW, MAXD, false>(st, P, sm.inptr, sm.inedge, sm.src, sm.dst, [&](int idx) {
    part = __dadd_rn(part, sm.w[idx - n_dt]);
  });
  // EQ12 and decode's resident-nowhere / freed-source checks (schedule.cpp:52-71)
  Row<NW> need_all = Row<NW>::zero(), need_le = Row<NW>::zero(), needD[MAXD];
#pragma unroll
  for (int d = 0; d < MAXD; ++d) needD[d] = Row<NW>::zero();
  for (Row<NW> r = st.Rany; r.any();) {
    const int v = r.lsb();
    r.clear(v);
    const Row<NW> pm = load_row<NW>(sm.pmask + v * NW);
    need_all = need_all | pm;
    if (v <= t) {
      need_le = need_le | pm;
#pragma unroll
      for (int d = 0; d < MAXD; ++d)
        if (d < D && st.R[d].test(v)) needD[d] = needD[d] | pm;
    }
  }
  if (andnot(need_all, st.Zany).any()) fl |= XE_F_EQ12;
  if (andnot(need_le, st.Zany).any()) fl |= XE_F_DECODE;
  if (busy >= 2) {
    bool bad = false;
#pragma unroll
    for (int dc = 0; dc < MAXD; ++dc) {
      if (dc >= D || bad) continue;
      for (Row<NW> miss = andnot(needD[dc], st.Z[dc]) & st.Zany; miss.any() && !bad;) {
        const int u = miss.lsb();
        miss.clear(u);
        int sdev = 0;
        while (!st.Z[sdev].test(u)) ++sdev;
        if (st.Sn[sdev].test(u)) continue;  // kept for t+1: never freed
        if (cube::decode_freed_one<NW>(st.R[sdev], st.Rany, st.R[dc], u, t, sdev, dc, a.strict, sm.cons)) bad = true;
      }
    }
    if (bad) fl |= XE_F_DECODE | XE_F_DECODE_FREED;
  }
  // row peaks
#pragma unroll
  for (int d = 0; d < MAXD; ++d) {
    if (d >= D) continue;
    const M base = table_mass<NW, M, NBL, TB>(st.S[d], sm.mtab);
    const int np = st.R[d].popc();
    M pkd = base;
    if (np >= 2)
      pkd = row_peak<NW, M>(st.R[d], st.Z[d], st.Sn[d], a.strict ? st.Rany : st.R[d], base, sm.pmask, sm.mass);
    else if (np == 1)
      pkd = base + sm.mass[st.R[d].lsb()];
    smem_max(&sm.pk[owner * MAXD + d], pkd);
  }
  if (fl) atomicOr(&sm.fl[owner], fl);
  return part;
}

// A lane's streaming state, parked in shared memory while its warp drains the
// job queue (the drain needs the registers; nothing is live across it).
template <int MAXD, int NW, class M>
struct Park {
  // the prefetched rows of t+1 exist only when MAXD * NW <= 4 (PF)
  static constexpr int PFD = MAXD * NW <= 4 ? MAXD : 1, PFW = MAXD * NW <= 4 ? NW : 1;
  double total;
  uint64_t fz, e12;
  uint64_t Zp[MAXD][NW], Rn[PFD][PFW], Sn[PFD][PFW];
  M pk[MAXD];
  int nfast;
};

// M: integer type of masses and memory sums (int32 when twice the save-all
// total fits).
// NBL: bytes of the last bit-row word that carry operators (4, 6 or 8).
//
// WARPS / TB: the default plan is 8-warp CTAs (2-3 per SM) with one 256-entry
// mass table per byte of a bit row; the wide plan (T <= 64) is one 24-warp
// CTA per SM whose 2048-entry tables cover 11 bits each (TB = 11, NBL = the
// number of 11-bit chunks): the tables are shared by 3x the warps and a row
// takes 4 lookups instead of 6 at T = 43.
template <int MAXD, int NW, class M, int NBL, int WARPS = kWarps, int TB = 8>
__global__ void __launch_bounds__(WARPS * 32, WARPS == kWarps ? ((MAXD * NW <= 2) ? 3 : 2) : 1)
    stream_kernel(const __grid_constant__ StArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const DevProblem& P = a.P;
  const int D = cube::ndev<MAXD>(P), T = P.T, E = P.E;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int NBT = 8 * (NW - 1) + NBL;  // byte tables of the row bytes that carry operators
  static_assert(TB == 8 || (TB == 11 && NW == 1), "11-bit mass tables cover one-word rows");

  M* s_mtab = reinterpret_cast<M*>(smem);  // [NBT][256] or [NBL][2048]
  M* s_mass = reinterpret_cast<M*>(smem + a.off_mass);
  uint64_t* s_pmask = reinterpret_cast<uint64_t*>(smem + a.off_pmask);
  uint64_t* s_cons = reinterpret_cast<uint64_t*>(smem + a.off_cons);
  double* s_c = reinterpret_cast<double*>(smem + a.off_c);
  double* s_w = reinterpret_cast<double*>(smem + a.off_w);
  uint32_t* s_inl = reinterpret_cast<uint32_t*>(smem + a.off_inl);  // in-edges: src | edge << 16
  int32_t* s_inptr = reinterpret_cast<int32_t*>(smem + a.off_inptr);
  int32_t* s_inedge = reinterpret_cast<int32_t*>(smem + a.off_inedge);
  int32_t* s_src = reinterpret_cast<int32_t*>(smem + a.off_src);
  int32_t* s_dst = reinterpret_cast<int32_t*>(smem + a.off_dst);
  const int n_dt = D * T, n_copy = E * D * D;
  if (TB == 8) {
    for (int i = threadIdx.x; i < NBT * 256; i += blockDim.x)
      s_mtab[i] = i < P.NB * 256 ? static_cast<M>(P.mtab[i]) : M(0);
  } else {  // chunk c, entry v: the masses of the set bits of v at operators 11c..11c+10
    for (int i = threadIdx.x; i < NBL * 2048; i += blockDim.x) {
      const int c = i >> 11, v = i & 2047;
      M m = 0;
      for (int b = 0; b < 11; ++b)
        if (((v >> b) & 1) && 11 * c + b < T) m += static_cast<M>(P.mass[11 * c + b]);
      s_mtab[i] = m;
    }
  }
  for (int i = threadIdx.x; i < T; i += blockDim.x) s_mass[i] = static_cast<M>(P.mass[i]);
  for (int i = threadIdx.x; i < T * NW; i += blockDim.x) {
    s_pmask[i] = P.pmask[i];
    s_cons[i] = P.cons[i];
  }
  for (int i = threadIdx.x; i < n_dt; i += blockDim.x) s_c[i] = P.table[i];
  for (int i = threadIdx.x; i < n_copy; i += blockDim.x) s_w[i] = P.table[n_dt + i];
  for (int i = threadIdx.x; i <= T; i += blockDim.x) s_inptr[i] = P.in_ptr[i];
  for (int i = threadIdx.x; i < E; i += blockDim.x) {
    const int e = P.in_edge[i];
    s_inedge[i] = e;
    s_inl[i] = static_cast<uint32_t>(P.src[e]) | (static_cast<uint32_t>(e) << 16);
    s_src[i] = P.src[i];
    s_dst[i] = P.dst[i];
  }
  Job* queue = reinterpret_cast<Job*>(smem + a.off_warp + wid * a.warp_bytes);
  constexpr int QCAP = qcap(NW);
  uint32_t* s_fl = reinterpret_cast<uint32_t*>(queue + QCAP);
  int32_t* s_cnt = reinterpret_cast<int32_t*>(s_fl + 32);
  M* s_pk = reinterpret_cast<M*>(s_cnt + 32);
  double* s_slow = reinterpret_cast<double*>(s_pk + 32 * MAXD);  // [32] deferred objective parts
  Park<MAXD, NW, M>* park = reinterpret_cast<Park<MAXD, NW, M>*>(s_slow + 32);
  s_slow[lane] = 0.0;
  s_fl[lane] = 0;
  s_cnt[lane] = 0;
#pragma unroll
  for (int d = 0; d < MAXD; ++d) s_pk[lane * MAXD + d] = 0;
  __syncthreads();
  const Sm<M> sm{s_mtab, s_mass, s_pmask, s_cons, s_c, s_w, s_inptr, s_inedge, s_src, s_dst, s_fl, s_cnt, s_pk};

  const int64_t gwarp = static_cast<int64_t>(blockIdx.x) * WARPS + wid;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * WARPS;
  const int64_t ngroups = (a.n + 31) / 32;
  const int64_t K = 2ll * D * T * NW;
  const int dstride = T * NW * 32;  // words between (which,d) blocks
  const int tl = T - 64 * (NW - 1);                            // bits in the last word
  const uint64_t lastmask = tl >= 64 ? ~0ull : ((1ull << tl) - 1ull);
  const unsigned lt_mask = (1u << lane) - 1u;

  uint64_t best_key = ~0ull;
  int64_t best_idx = -1;
  int n_valid = 0;

  for (int64_t g = gwarp; g < ngroups; g += nwarps) {
    const int64_t c = g * 32 + lane;
    const uint64_t* cw = a.il + static_cast<size_t>(g) * K * 32 + lane;
    int q_cnt = 0;  // warp-uniform
    int a_first = 0, a_last = 0, a_n = 0;  // this lane's kind-A chain in the queue
    double total = 0.0;
    int nfast = 0;
    uint64_t fzS = 0, eq12 = 0;
    M pk[MAXD];
    uint64_t Zp[MAXD][NW];
#pragma unroll
    for (int d = 0; d < MAXD; ++d) {
      pk[d] = 0;
#pragma unroll
      for (int j = 0; j < NW; ++j) Zp[d][j] = ~0ull;  // no EQ11 rows before t = 0
    }
    // drains the queue at full width: lane k takes job k; the owners then add
    // their jobs' objective parts in push (= timestep) order, so the sum is a
    // pure function of the candidate
    auto drain = [&]() {
      __syncwarp();
#pragma unroll 1
      for (int k = lane; k < q_cnt; k += 32) {
        const uint32_t m = queue[k].meta;
        const int owner = (m >> 10) & 31;
        queue[k].part = run_job<MAXD, NW, M, NBL, TB>(cw - lane + owner, static_cast<int>(m & 1023u), static_cast<int>(m >> 15),
                                             owner, &a, sm);
      }
      __syncwarp();
      // each owner walks its own kind-A chain (push = timestep order)
      double sl = s_slow[lane];
#pragma unroll 1
      for (int k = a_first, n = a_n; n > 0; --n) {
        sl = __dadd_rn(sl, queue[k].part);
        k = static_cast<int>(queue[k].next);
      }
      s_slow[lane] = sl;
      __syncwarp();
      q_cnt = 0;
      a_n = 0;
    };

    // rows of t in registers; t+1 prefetched for small rows
    constexpr bool PF = kPfReg && MAXD * NW <= 4;
    uint64_t Rn[MAXD][NW], Sn[MAXD][NW];
    auto load_p = [&](const uint64_t* pt, uint64_t (&R)[MAXD][NW], uint64_t (&S)[MAXD][NW]) {
#pragma unroll
      for (int d = 0; d < MAXD; ++d)
#pragma unroll
        for (int j = 0; j < NW; ++j) {
          R[d][j] = d < D ? __ldg(pt + d * dstride + j * 32) : 0ull;
          S[d][j] = d < D ? __ldg(pt + (D + d) * dstride + j * 32) : 0ull;
        }
    };
    // running pointer to the rows of the next timestep to load
    const uint64_t* pnext = cw;
    if (PF) {
      load_p(pnext, Rn, Sn);
      pnext += NW * 32;
    }

#pragma unroll kTUnroll
    for (int t = 0; t < T; ++t) {
      uint64_t R[MAXD][NW], S[MAXD][NW];
      if (PF) {
#pragma unroll
        for (int d = 0; d < MAXD; ++d)
#pragma unroll
          for (int j = 0; j < NW; ++j) {
            R[d][j] = Rn[d][j];
            S[d][j] = Sn[d][j];
          }
        if (t + 1 < T) load_p(pnext, Rn, Sn);
        pnext += NW * 32;
      } else {
        // rows too wide to double-buffer in registers: prefetch the lines of
        // t + kPrefetch into L2 (no registers) while t's are loaded
        if (t + kPrefetch < T) {
          const uint64_t* pn = pnext + kPrefetch * NW * 32;
#pragma unroll
          for (int d = 0; d < MAXD; ++d)
#pragma unroll
            for (int j = 0; j < NW; ++j)
              if (d < D) {
                asm volatile("prefetch.global.L2 [%0];" ::"l"(pn + d * dstride + j * 32));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(pn + (D + d) * dstride + j * 32));
              }
        }
        load_p(pnext, R, S);
        pnext += NW * 32;
      }
      const int tw = NW == 1 ? 0 : (t >> 6), tb = t & 63;
      uint64_t off = 0, eq11 = 0, zany[NW];
      int cnt = 0, dstar = 0;
      M base[MAXD];
#pragma unroll
      for (int j = 0; j < NW; ++j) zany[j] = 0;
#pragma unroll
      for (int d = 0; d < MAXD; ++d) {
        base[d] = 0;
        if (d >= D) continue;
#pragma unroll
        for (int j = 0; j < NW; ++j) {
          uint64_t r = R[d][j], s = S[d][j];
          if (j == NW - 1) {
            r &= lastmask;
            s &= lastmask;
          }
          // S(d,t,i >= t) is fixed to zero (model.cpp:126-132)
          const uint64_t ge = (NW == 1 || j == tw) ? (~0ull << tb) : (j > tw ? ~0ull : 0ull);
          fzS |= s & ge;
          uint64_t rr = r;
          if (NW == 1 || j == tw) {
            const int on = static_cast<int>((r >> tb) & 1ull);
            cnt += on;
            dstar = on ? d : dstar;
            rr = r & ~(1ull << tb);
          }
          off |= rr;
          const uint64_t z = r | s;
          eq11 |= s & ~Zp[d][j];  // EQ11 rows of t-1: S(d,t,i) > S(d,t-1,i) + R(d,t-1,i)
          Zp[d][j] = z;
          zany[j] |= z;
          // mass of the saved tensors through the byte tables
          if (TB == 8) {
            const uint32_t lo = static_cast<uint32_t>(s), hi = static_cast<uint32_t>(s >> 32);
#pragma unroll
            for (int b = 0; b < (j == NW - 1 ? NBL : 8); ++b)
              base[d] += s_mtab[(8 * j + b) * 256 + (((b < 4 ? lo : hi) >> (8 * (b & 3))) & 0xffu)];
          } else {
#pragma unroll
            for (int c = 0; c < NBL; ++c)
              base[d] += s_mtab[c * 2048 + static_cast<int>((s >> (11 * c)) & 0x7ffull)];
          }
        }
      }
      const bool fast = off == 0 && cnt == 1;
      // parents of t must be resident somewhere (EQ12; decode)
      uint64_t miss = 0;
#pragma unroll
      for (int j = 0; j < NW; ++j) miss |= s_pmask[t * NW + j] & ~zany[j];
      eq12 |= fast ? miss : 0ull;
      // compute term and copy charges of the diagonal computation
      double acc = s_c[dstar * T + t];
      for (int k = s_inptr[t]; k < s_inptr[t + 1]; ++k) {
        const uint32_t pe = s_inl[k];
        const int u = static_cast<int>(pe & 0xffffu), e = static_cast<int>(pe >> 16);
        const int uw = NW == 1 ? 0 : (u >> 6), ub = u & 63;
        if constexpr (MAXD == 2 && NW == 1) {
          // one other device: select its row per lane (measured faster here
          // than the bit gather below)
#pragma unroll
          for (int o = 1; o < MAXD; ++o) {
            if (o >= D) break;
            const int ds = dstar + o < D ? dstar + o : dstar + o - D;
            const uint64_t zw = ds == 0 ? Zp[0][0] : Zp[1][0];
            // branch-free: adding +0.0 leaves the (non-negative) sum unchanged
            const double wv = s_w[(e * D + ds) * D + dstar];
            acc = __dadd_rn(acc, ((zw >> ub) & 1ull) ? wv : 0.0);
          }
        } else {
          // u's residency on every device as bits (u and its word are the
          // same in every lane: the word select is uniform); ResNet-50 /
          // U-Net 127 / 106 -> 133 / 115 M cand/s against a per-(device,
          // word) select for every other device
          uint32_t zb = 0u;
#pragma unroll
          for (int d = 0; d < MAXD; ++d) {
            uint64_t zw = Zp[d][0];
#pragma unroll
            for (int j = 1; j < NW; ++j)
              if (j == uw) zw = Zp[d][j];
            zb |= static_cast<uint32_t>((zw >> ub) & 1ull) << d;
          }
          // every other device in rotation from d*: each lane runs D-1 steps
#pragma unroll
          for (int o = 1; o < MAXD; ++o) {
            if (o >= D) break;
            const int ds = dstar + o < D ? dstar + o : dstar + o - D;
            // branch-free: adding +0.0 leaves the (non-negative) sum unchanged
            const double wv = s_w[(e * D + ds) * D + dstar];
            acc = __dadd_rn(acc, ((zb >> ds) & 1u) ? wv : 0.0);
          }
        }
      }
      if (fast) total = __dadd_rn(total, acc);
      nfast += fast ? 1 : 0;
      const M mt = s_mass[t];
#pragma unroll
      for (int d = 0; d < MAXD; ++d)
        if (d < D) pk[d] = max(pk[d], base[d] + ((fast && d == dstar) ? mt : M(0)));
      // defer the irregular timesteps
      const unsigned bA = __ballot_sync(0xffffffffu, !fast), bB = __ballot_sync(0xffffffffu, eq11 != 0);
      if (bA | bB) {
        if (!fast) {
          const int k = q_cnt + __popc(bA & lt_mask);
          queue[k].meta = static_cast<uint32_t>(t) | (lane << 10) | (kKindA << 15);
          if (a_n) queue[a_last].next = static_cast<uint32_t>(k);
          else a_first = k;
          a_last = k;
          ++a_n;
        }
        const int q2 = q_cnt + __popc(bA);
        if (eq11) queue[q2 + __popc(bB & lt_mask)].meta = static_cast<uint32_t>(t - 1) | (lane << 10) | (kKindB << 15);
        q_cnt = q2 + __popc(bB);
        if (q_cnt > QCAP - 64) {
          Park<MAXD, NW, M>& pp = park[lane];
          pp.total = total;
          pp.fz = fzS;
          pp.e12 = eq12;
          pp.nfast = nfast;
#pragma unroll
          for (int d = 0; d < MAXD; ++d) {
            pp.pk[d] = pk[d];
#pragma unroll
            for (int j = 0; j < NW; ++j) {
              pp.Zp[d][j] = Zp[d][j];
              if constexpr (PF) {
                pp.Rn[d][j] = Rn[d][j];
                pp.Sn[d][j] = Sn[d][j];
              }
            }
          }
          asm volatile("" ::: "memory");
          drain();
          asm volatile("" ::: "memory");
          total = pp.total;
          fzS = pp.fz;
          eq12 = pp.e12;
          nfast = pp.nfast;
#pragma unroll
          for (int d = 0; d < MAXD; ++d) {
            pk[d] = pp.pk[d];
#pragma unroll
            for (int j = 0; j < NW; ++j) {
              Zp[d][j] = pp.Zp[d][j];
              if constexpr (PF) {
                Rn[d][j] = pp.Rn[d][j];
                Sn[d][j] = pp.Sn[d][j];
              }
            }
          }
        }
      }
    }
    if (q_cnt) {
      Park<MAXD, NW, M>& pp = park[lane];
      pp.total = total;
      pp.fz = fzS;
      pp.e12 = eq12;
      pp.nfast = nfast;
#pragma unroll
      for (int d = 0; d < MAXD; ++d) pp.pk[d] = pk[d];
      asm volatile("" ::: "memory");
      drain();
      asm volatile("" ::: "memory");
      total = pp.total;
      fzS = pp.fz;
      eq12 = pp.e12;
      nfast = pp.nfast;
#pragma unroll
      for (int d = 0; d < MAXD; ++d) pk[d] = pp.pk[d];
    }
    __syncwarp();
    const double slow_total = s_slow[lane];
    s_slow[lane] = 0.0;

    uint32_t fl = s_fl[lane];
    s_fl[lane] = 0;
    const int nslow_diag = s_cnt[lane];
    s_cnt[lane] = 0;
#pragma unroll
    for (int d = 0; d < MAXD; ++d) {
      pk[d] = max(pk[d], s_pk[lane * MAXD + d]);
      s_pk[lane * MAXD + d] = 0;
    }
    if (fzS) fl |= XE_F_FIXED_ZERO;
    if (eq12) fl |= XE_F_EQ12 | XE_F_DECODE;
    if (nfast + nslow_diag != T) fl |= XE_F_EQ9;
#pragma unroll
    for (int d = 0; d < MAXD; ++d) {
      if (d >= D) continue;
      if (static_cast<int64_t>(pk[d]) > P.budget[d]) fl |= XE_F_BUDGET;
      if (static_cast<double>(pk[d]) > P.ubound[d]) fl |= XE_F_U_BOUND;
    }
    const double obj = __dadd_rn(total, slow_total);
    const bool live = c < a.n;
    if (live && a.obj) a.obj[c] = obj;
    if (live && a.flags) a.flags[c] = fl;
    if (live && a.peak)
#pragma unroll
      for (int d = 0; d < MAXD; ++d)
        if (d < D) a.peak[c * D + d] = static_cast<int64_t>(pk[d]);
    if (live && (fl & a.valid_mask) == 0) {
      ++n_valid;
      const uint64_t key = __double_as_longlong(obj);
      if (key < best_key) {
        best_key = key;
        best_idx = c;
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
  const int64_t nv = warp_sum_i64(n_valid);
  if (lane == 0) {
    a.wbest_key[gwarp] = best_key;
    a.wbest_idx[gwarp] = best_idx;
    a.wvalid[gwarp] = nv;
  }
}

// launcher instantiated per NW (eval_stream_nw*.cu); wide: the 24-warp,
// 11-bit-table plan (NW = 1, int32 masses), nbl = its chunk count
template <int NW>
int launch_stream(const StArgs& a, bool m32, int nbl, cudaStream_t s, int nsm, bool wide);
#ifndef XE_WIDE_WARPS
#define XE_WIDE_WARPS 24
#endif
constexpr int kWideWarps = XE_WIDE_WARPS;

}  // namespace st
}  // namespace xe
