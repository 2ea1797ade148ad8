// SPDX-License-Identifier: Apache-2.0
#pragma once
//
// K2a kernel, v3: two lane mappings per candidate.
//
//   pass A — one lane per (d,t) ROW, rows in d-major order (the order of
//            objective_value's first loop, model.cpp:393-398): fixed-zero,
//            EQ11 (+EQ16_HI), ENERGY_DEV, the U recurrence / row peak, and the
//            R (+ alpha*q) terms of the serial objective, whose list positions
//            are then a single running exclusive scan over rows.
//   pass B — one lane per TIMESTEP t (all devices' rows of t): EQ8/EQ9, the
//            dependency masks (EQ12, decode's resident-nowhere and
//            freed-copy-source checks), the copy charges (model.cpp:399-411)
//            and ENERGY_TOTAL.
//
// Helpers (row loads, mass tables, the general row peak, EQ16_HI, decode,
// the over-capacity objective) are shared with eval_cube_kernel.cuh.

#include "eval_cube_kernel.cuh"

namespace xe {
namespace cube {

constexpr int kCopyScratch = 8;  // copy terms per lane per timestep before the slow path

template <int NW, int MAXD, bool EXACT>
__global__ void __launch_bounds__(kWarps * 32, 2) eval_cube_v3(const EvalArgs a) {
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

  unsigned char* wreg = smem + a.off_warp + wid * a.warp_bytes;
  uint32_t* stage_buf = reinterpret_cast<uint32_t*>(wreg + a.off_w_stage);
  uint64_t* bars = reinterpret_cast<uint64_t*>(wreg + a.off_w_bar);
  uint16_t* terms = reinterpret_cast<uint16_t*>(wreg + a.off_w_terms);
  uint16_t* terms2 = reinterpret_cast<uint16_t*>(wreg + a.off_w_terms2);
  double* slot_obj = reinterpret_cast<double*>(wreg + a.off_w_slot);
  uint32_t* slot_flags = reinterpret_cast<uint32_t*>(slot_obj + kSlots);
  int32_t* slot_cnt = reinterpret_cast<int32_t*>(slot_flags + kSlots);
  int32_t* slot_cnt2 = slot_cnt + kSlots;
  int64_t* slot_peak = reinterpret_cast<int64_t*>(slot_cnt2 + kSlots);      // [kSlots][D]
  uint16_t* cscr = reinterpret_cast<uint16_t*>(slot_peak + kSlots * D);     // [32][kCopyScratch]

  if (lane == 0)
    for (int s = 0; s < a.stages; ++s) mbar_init(&bars[s], 1);
  fence_mbar_init();
  __syncthreads();

  const int64_t gwarp = static_cast<int64_t>(blockIdx.x) * a.warps + wid;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * a.warps;
  const int64_t nblocks = (a.n + kSlots - 1) / kSlots;
  const uint32_t cube_bytes = a.cube_words * 4u;
  const int nrows = D * T;
  const Row<NW> valid = Row<NW>::below(T);
  const int eb = D * T + E * D * D;  // energy terms base in the term table

  uint64_t best_key = ~0ull;
  int64_t best_idx = -1, n_valid = 0;

  auto cand_of = [&](int64_t k) -> int64_t {
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
      const int64_t next_c = ((k + 1) % kSlots == 0) ? cand_of(k + 1) : (s + 1 < nslot ? first + s + 1 : a.n);
      if (a.stages > 1) issue(next_c, static_cast<int>((k + 1) % a.stages));  // prefetch into the other buffer
      if (a.use_bulk) {
        mbar_wait(&bars[stage], (phase_bits >> stage) & 1u);
        phase_bits ^= 1u << stage;
      }
      const uint32_t* cw = stage_buf + static_cast<size_t>(stage) * a.cube_words;
      uint16_t* list = terms + s * a.cap;
      uint16_t* list2 = terms2 + s * a.cap2;

      uint32_t fl = 0;
      int64_t pk[MAXD];
#pragma unroll
      for (int d = 0; d < MAXD; ++d) pk[d] = 0;
      int64_t fix = 0;
      int run = 0;  // serial: running count of R terms (d-major rows)
      bool overflow = false;

      // ================= pass A: one lane per (d,t) row =================
      for (int r0 = 0; r0 < nrows; r0 += 32) {
        const int r = r0 + lane;
        const bool act = r < nrows;
        const int d = act ? r / T : 0;
        const int t = act ? r - d * T : 0;
        Row<NW> R = Row<NW>::zero(), S = Row<NW>::zero(), Sn = Row<NW>::zero();
        if (act) {
          R = cube_row<NW>(cw, P.W32, D, T, 0, d, t) & valid;
          S = cube_row<NW>(cw, P.W32, D, T, 1, d, t) & valid;
          if (t + 1 < T) Sn = cube_row<NW>(cw, P.W32, D, T, 1, d, t + 1) & valid;
          const Row<NW> Z = R | S;
          if ((R & Row<NW>::above(t)).any() || (S & Row<NW>::at_or_above(t)).any()) fl |= XE_F_FIXED_ZERO;
          const Row<NW> bad = andnot(Sn, Z);  // EQ11
          if (bad.any()) {
            Row<NW> Cd = R;
            if (a.strict)
              for (int x = 0; x < D; ++x) Cd = Cd & cube_row<NW>(cw, P.W32, D, T, 0, x, t);
            fl |= XE_F_EQ11 | eq16_hi<NW>(R, Cd, bad, s_cons);
          }
          if (a.energy && (R & load_row<NW>(s_ebad + d * NW)).any()) fl |= XE_F_ENERGY_DEV;
          // U recurrence of row (d,t): base = saved tensors; at most one
          // computation -> peak base + m_v, else the general free walk
          const int64_t base = mass_bytes<NW>(S, s_mtab, P.NB);
          const int c = R.popc();
          int64_t rp = base;
          if (c == 1) {
            rp = base + s_mass[R.lsb()];
          } else if (c > 1) {
            Row<NW> scan = R;
            if (a.strict)
              for (int x = 0; x < D; ++x) scan = scan | cube_row<NW>(cw, P.W32, D, T, 0, x, t);
            rp = row_peak_general<NW>(R, Z, Sn, scan & valid, base, s_pmask, s_mass);
          }
#pragma unroll
          for (int x = 0; x < MAXD; ++x)
            if (x == d) pk[x] = max(pk[x], rp);
        }
        if (EXACT) {
          for (Row<NW> rr = R; rr.any();) {
            const int i = rr.lsb();
            rr.clear(i);
            fix += s_tfix[d * T + i];
            if (a.energy) fix += s_tfix[eb + d * T + i];
          }
        } else {
          int chunk_tot;
          int pos = run + warp_excl_scan(R.popc(), lane, &chunk_tot);
          run += chunk_tot;
          if (run > a.cap || (a.energy && run > a.cap2)) {
            overflow = true;
          } else {
            for (Row<NW> rr = R; rr.any(); ++pos) {
              const int i = rr.lsb();
              rr.clear(i);
              list[pos] = static_cast<uint16_t>(d * T + i);
              if (a.energy) list2[pos] = static_cast<uint16_t>(eb + d * T + i);
            }
          }
        }
      }
      const int sumR = run;

      // ================= pass B: one lane per timestep =================
      int eq9 = 0, runC = 0;
      for (int t0 = 0; t0 < T; t0 += 32) {
        const int t = t0 + lane;
        const bool act = t < T;
        TState<NW, MAXD> st;
        load_t<NW, MAXD>(st, cw, P, t, act);
        bool has_copy = false;
        Row<NW> needAllD[MAXD];
#pragma unroll
        for (int x = 0; x < MAXD; ++x) needAllD[x] = Row<NW>::zero();
        if (act) {
          int nd = 0;
#pragma unroll
          for (int x = 0; x < MAXD; ++x)
            if (x < D) nd += st.R[x].test(t);
          if (nd != 1) fl |= XE_F_EQ8;
          eq9 += nd;
          Row<NW> need_all = Row<NW>::zero(), need_le = Row<NW>::zero(), needD[MAXD];
#pragma unroll
          for (int x = 0; x < MAXD; ++x) needD[x] = Row<NW>::zero();
          for (Row<NW> rem = st.Rany; rem.any();) {
            const int v = rem.lsb();
            rem.clear(v);
            const Row<NW> pm = load_row<NW>(s_pmask + v * NW);
            need_all = need_all | pm;
            const bool le = v <= t;
            if (le) need_le = need_le | pm;
#pragma unroll
            for (int x = 0; x < MAXD; ++x)
              if (x < D && st.R[x].test(v)) {
                needAllD[x] = needAllD[x] | pm;
                if (le) needD[x] = needD[x] | pm;
              }
          }
          if (andnot(need_all, st.Zany).any()) fl |= XE_F_EQ12;
          if (andnot(need_le, st.Zany).any()) fl |= XE_F_DECODE;
          // a copy source can free its tensor within timestep t only if it
          // computes something at t, and it never computes the consumer: an
          // illegal copy needs >= 2 devices computing at t
          int busy = 0;
#pragma unroll
          for (int x = 0; x < MAXD; ++x) busy += (x < D && st.R[x].any()) ? 1 : 0;
#pragma unroll
          for (int dc = 0; dc < MAXD; ++dc) {
            if (dc >= D) continue;
            // parents of dc's computations held by another device -> copies
            Row<NW> others = Row<NW>::zero();
#pragma unroll
            for (int ds = 0; ds < MAXD; ++ds)
              if (ds < D && ds != dc) others = others | st.Z[ds];
            if ((needAllD[dc] & others).any()) has_copy = true;
            // decode: copy source = lowest holder; illegal if it freed u earlier
            Row<NW> miss = busy >= 2 ? andnot(needD[dc], st.Z[dc]) & st.Zany : Row<NW>::zero();
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
              if (keep) continue;
              const Row<NW> cu = load_row<NW>(s_cons + u * NW);
              int fs = -1;
              const Row<NW> cc = cu & (a.strict ? st.Rany : Rs);
              if (cc.any()) {
                const int mm = cc.msb();
                fs = Rs.test(mm) ? mm : -1;
              } else if (Rs.test(u)) {
                fs = u;
              }
              if (fs < 0) continue;
              const int vmax = (cu & st.R[dc] & ~Row<NW>::above(t)).msb();
              if (fs < vmax || (fs == vmax && sdev < dc)) fl |= XE_F_DECODE | XE_F_DECODE_FREED;
            }
          }
          if (a.energy && P.has_total) {
            double lhs = 0.0, scale = fmax(1.0, fabs(P.total_rhs));
            for (int x = 0; x < D; ++x) {
              Row<NW> rr = cube_row<NW>(cw, P.W32, D, T, 0, x, t) & valid;
              for (int i = rr.lsb(); i >= 0; rr.clear(i), i = rr.lsb()) {
                const double q = s_q[x * T + i];
                if (q != 0.0) {
                  lhs = __dadd_rn(lhs, q);
                  scale = fmax(scale, fabs(q));
                }
              }
            }
            if (__dsub_rn(lhs, P.total_rhs) > 1e-6 * scale) fl |= XE_F_ENERGY_TOTAL;
          }
        }
        // ---- copy charges of timestep t
        if (EXACT) {
          if (has_copy)
            for_copy_terms<NW, MAXD, false>(st, P, s_inptr, s_inedge, s_src, s_dst,
                                            [&](int idx) { fix += s_tfix[idx]; });
        } else if (__any_sync(0xffffffffu, has_copy)) {
          int c = 0;
          uint16_t* mine = cscr + lane * kCopyScratch;
          if (has_copy)
            for_copy_terms<NW, MAXD, true>(st, P, s_inptr, s_inedge, s_src, s_dst, [&](int idx) {
              if (c < kCopyScratch) mine[c] = static_cast<uint16_t>(idx);
              ++c;
            });
          if (__any_sync(0xffffffffu, c > kCopyScratch)) overflow = true;
          int chunk_tot;
          int pos = sumR + runC + warp_excl_scan(c, lane, &chunk_tot);
          runC += chunk_tot;
          if (sumR + runC > a.cap) overflow = true;
          if (!overflow)
            for (int j = 0; j < c; ++j) list[pos + j] = mine[j];
        }
      }

      // ---- per-candidate reductions
      fl = __reduce_or_sync(0xffffffffu, fl);
      eq9 = __reduce_add_sync(0xffffffffu, eq9);
      if (eq9 != T) fl |= XE_F_EQ9;
#pragma unroll
      for (int x = 0; x < MAXD; ++x) {
        if (x >= D) continue;
        const int64_t pv = warp_max_u63(pk[x]);
        if (pv > P.budget[x]) fl |= XE_F_BUDGET;
        if (static_cast<double>(pv) > P.ubound[x]) fl |= XE_F_U_BOUND;
        if (lane == 0) slot_peak[s * D + x] = pv;
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
      if (a.stages == 1) issue(next_c, 0);  // single buffer: refill once this candidate is done
    }

    // ---- chain phase: lane s replays slot s's term list (serial mode)
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
int launch3_t(const EvalArgs& a, int grid_cap, int smem, cudaStream_t s, int nsm) {
  auto k = eval_cube_v3<NW, MAXD, EXACT>;
  XE_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 0;
  XE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, a.warps * 32, smem));
  if (per_sm < 1) fail(XE_ERR_TOO_LARGE, "evaluator does not fit on an SM");
  const int grid = std::max(1, std::min(grid_cap, nsm * per_sm));
  k<<<grid, a.warps * 32, smem, s>>>(a);
  XE_CUDA(cudaGetLastError());
  return grid;
}

template <int NW, int MAXD>
int launch3_m(const EvalArgs& a, int grid, int smem, cudaStream_t s, int nsm) {
  if (a.P.fix_k >= 0) return launch3_t<NW, MAXD, true>(a, grid, smem, s, nsm);
  return launch3_t<NW, MAXD, false>(a, grid, smem, s, nsm);
}

template <int NW>
int launch3_d(const EvalArgs& a, int grid, int smem, cudaStream_t s, int nsm) {
  switch (a.P.D) {
    case 1: return launch3_m<NW, 1>(a, grid, smem, s, nsm);
    case 2: return launch3_m<NW, 2>(a, grid, smem, s, nsm);
    case 3: return launch3_m<NW, 3>(a, grid, smem, s, nsm);
    case 4: return launch3_m<NW, 4>(a, grid, smem, s, nsm);
    default: return launch3_m<NW, 8>(a, grid, smem, s, nsm);
  }
}

}  // namespace cube
}  // namespace xe
