// SPDX-License-Identifier: Apache-2.0
//
// Problem upload: the resolved host problem becomes the device tables the
// K1/K2/K4 kernels read (bit masks of parents/consumers, byte tables of
// tensor masses, the objective term table).  Host-side precomputation only;
// every number the kernels combine is taken verbatim from the reference's
// inputs (output_bytes, costs_ms, copy_cost values).

#include <algorithm>
#include <cmath>
#include <cstring>

#include "xe_internal.hpp"

namespace xe {

// Smallest k >= 0 such that every table entry is an integer multiple of
// 2^-k and the largest possible objective (each (d,t,i) compute and each
// (t,e,ds,dc) copy charged at most once per timestep) stays below 2^52
// units.  Then every partial sum of objective_value's sequential loop
// (model.cpp:392-427) is exactly representable, any summation order gives
// the same double, and the kernels may accumulate in int64 fixed point.
// Returns -1 when no such k exists (the kernels then reproduce the
// reference's summation order term by term).
// Same rule with an explicit bound on the largest possible total.
int exact_fix_k_bound(const std::vector<double>& table, long double bound) {
  int k = 0;
  for (double v : table) {
    if (!std::isfinite(v)) return -1;
    if (v == 0.0) continue;
    int e = 0;
    double m = std::frexp(std::fabs(v), &e);                  // v = m * 2^e, m in [0.5,1)
    uint64_t M = static_cast<uint64_t>(std::ldexp(m, 53));    // exact 53-bit mantissa
    int tz = __builtin_ctzll(M);
    int need = -(e - 53 + tz);                                 // fractional bits
    k = std::max(k, need);
  }
  if (k > 60) return -1;
  if (std::ldexp(bound, k) >= std::ldexp(1.0L, 52)) return -1;
  return k;
}

int exact_fix_k(const std::vector<double>& table, int T) {
  long double bound = 0.0L;
  for (double v : table) bound += std::fabs(static_cast<long double>(v));
  return exact_fix_k_bound(table, bound * static_cast<long double>(T));
}

DevProblem xe_problem_view_impl(const xe_problem* p, bool energy);

}  // namespace xe

xe::DevProblem xe_problem::view(bool energy) const {
  xe::DevProblem v = dev;
  if (energy && h.has_energy) {
    v.has_energy = 1;
    v.fix_k = fix_k_energy;
    v.tfix = d_tfix.p;
  } else {
    v.has_energy = 0;
    v.fix_k = fix_k_plain;
    v.tfix = d_tfix_noenergy.p;
    v.has_total = 0;
  }
  return v;
}

namespace xe {

void upload_problem(xe_problem* pr) {
  const HostProblem& h = pr->h;
  const int D = h.D, T = h.T, E = h.E;
  const int NW = (T + 63) / 64, WE = std::max(1, (E + 63) / 64), NB = (T + 7) / 8;
  cudaStream_t s = pr->stream;

  std::vector<uint64_t> pmask(static_cast<size_t>(T) * NW, 0), cons(static_cast<size_t>(T) * NW, 0);
  std::vector<int32_t> in_ptr(static_cast<size_t>(T) + 1, 0), in_edge(static_cast<size_t>(E));
  for (int e = 0; e < E; ++e) {
    int u = h.src[static_cast<size_t>(e)], v = h.dst[static_cast<size_t>(e)];
    pmask[static_cast<size_t>(v) * NW + u / 64] |= 1ull << (u % 64);
    cons[static_cast<size_t>(u) * NW + v / 64] |= 1ull << (v % 64);
    in_ptr[static_cast<size_t>(v) + 1]++;
  }
  for (int v = 0; v < T; ++v) in_ptr[static_cast<size_t>(v) + 1] += in_ptr[static_cast<size_t>(v)];
  {
    std::vector<int32_t> fill(in_ptr.begin(), in_ptr.end() - 1);
    for (int e = 0; e < E; ++e) in_edge[static_cast<size_t>(fill[static_cast<size_t>(h.dst[static_cast<size_t>(e)])]++)] = e;
  }
  int by_dst = 1;
  for (int e = 1; e < E; ++e)
    if (h.dst[static_cast<size_t>(e)] < h.dst[static_cast<size_t>(e) - 1]) by_dst = 0;

  // byte tables: mtab[b][x] = sum of output_bytes[8b + j] over the set bits j of x
  std::vector<int64_t> mtab(static_cast<size_t>(NB) * 256, 0);
  for (int b = 0; b < NB; ++b)
    for (int x = 0; x < 256; ++x) {
      int64_t sum = 0;
      for (int j = 0; j < 8; ++j)
        if (((x >> j) & 1) && 8 * b + j < T) sum += h.mass[static_cast<size_t>(8 * b + j)];
      mtab[static_cast<size_t>(b) * 256 + x] = sum;
    }

  // U upper bound of check_assignment: val > b*(1+tol)+tol (model.cpp:441-445)
  std::vector<double> ub(static_cast<size_t>(D));
  for (int d = 0; d < D; ++d) {
    double b = static_cast<double>(h.budget[static_cast<size_t>(d)]);
    ub[static_cast<size_t>(d)] = b * (1.0 + 1e-6) + 1e-6;
  }

  // objective term table: cost[d][i] | copy w[e][ds][dc] | alpha*q[d][i]
  const int n_table = D * T + E * D * D + D * T;
  pr->table.assign(static_cast<size_t>(n_table), 0.0);
  for (int i = 0; i < D * T; ++i) pr->table[static_cast<size_t>(i)] = h.cost[static_cast<size_t>(i)];
  for (int i = 0; i < E * D * D; ++i) pr->table[static_cast<size_t>(D * T + i)] = h.w.empty() ? 0.0 : h.w[static_cast<size_t>(i)];
  for (int i = 0; i < D * T; ++i)
    pr->table[static_cast<size_t>(D * T + E * D * D + i)] = h.has_energy ? h.alpha * h.q[static_cast<size_t>(i)] : 0.0;
  {
    std::vector<double> plain(pr->table.begin(), pr->table.begin() + D * T + E * D * D);
    pr->fix_k_plain = exact_fix_k(plain, T);
    // a placement computes each op once and charges each edge at most once
    // (save_all_assignment, solver.cpp:30-42): a much smaller worst case
    long double pb = 0.0L;
    for (int i = 0; i < T; ++i) {
      double mx = 0.0;
      for (int d = 0; d < D; ++d) mx = std::max(mx, std::fabs(h.cost[static_cast<size_t>(d) * T + i]));
      pb += mx;
    }
    for (int e = 0; e < E; ++e) {
      double mx = 0.0;
      for (int k2 = 0; k2 < D * D; ++k2) mx = std::max(mx, std::fabs(pr->table[static_cast<size_t>(D * T + e * D * D + k2)]));
      pb += mx;
    }
    pr->fix_k_place = exact_fix_k_bound(plain, pb);
    pr->fix_k_energy = h.has_energy ? exact_fix_k(pr->table, T) : pr->fix_k_plain;
  }
  auto fixed = [&](int k, bool with_energy) {
    std::vector<int64_t> f(static_cast<size_t>(n_table), 0);
    if (k < 0) return f;
    for (int i = 0; i < n_table; ++i) {
      if (!with_energy && i >= D * T + E * D * D) break;
      f[static_cast<size_t>(i)] = static_cast<int64_t>(std::ldexp(pr->table[static_cast<size_t>(i)], k));
    }
    return f;
  };

  // energy: ENERGY_DEV row (q*R <= lim) violated by R(d,t,i)=1 exactly when
  // q - lim > 1e-6 * max(1, |lim|, |q|) (model.cpp:451-466)
  std::vector<uint64_t> ebad(static_cast<size_t>(D) * NW, 0);
  if (h.has_energy)
    for (int d = 0; d < D; ++d) {
      if (!h.has_lim[static_cast<size_t>(d)]) continue;
      double lim = h.lim[static_cast<size_t>(d)];
      for (int i = 0; i < T; ++i) {
        double q = h.q[static_cast<size_t>(d) * T + i];
        double scale = std::max({1.0, std::fabs(lim), std::fabs(q)});
        if (q - lim > 1e-6 * scale) ebad[static_cast<size_t>(d) * NW + i / 64] |= 1ull << (i % 64);
      }
    }

  pr->d_mass.upload(h.mass, s);
  pr->d_mtab.upload(mtab, s);
  pr->d_budget.upload(h.budget, s);
  pr->d_pmask.upload(pmask, s);
  pr->d_cons.upload(cons, s);
  pr->d_ebad.upload(ebad, s);
  pr->d_src.upload(h.src, s);
  pr->d_dst.upload(h.dst, s);
  pr->d_in_ptr.upload(in_ptr, s);
  pr->d_in_edge.upload(in_edge, s);
  pr->d_ubound.upload(ub, s);
  pr->d_table.upload(pr->table, s);
  pr->d_q.upload(h.q.empty() ? std::vector<double>(static_cast<size_t>(D) * T, 0.0) : h.q, s);
  pr->d_cost.upload(h.cost, s);
  pr->d_w.upload(h.w.empty() ? std::vector<double>(1, 0.0) : h.w, s);
  pr->d_tfix.upload(fixed(pr->fix_k_energy, true), s);
  pr->d_tfix_noenergy.upload(fixed(pr->fix_k_plain, false), s);
  pr->d_tfix_place.upload(fixed(pr->fix_k_place, false), s);
  XE_CUDA(cudaStreamSynchronize(s));

  DevProblem& v = pr->dev;
  v.D = D;
  v.T = T;
  v.E = E;
  v.W32 = (T + 31) / 32;
  v.NW = NW;
  v.WE = WE;
  v.NB = NB;
  v.edges_by_dst = by_dst;
  v.mass = pr->d_mass.p;
  v.pmask = pr->d_pmask.p;
  v.cons = pr->d_cons.p;
  v.mtab = pr->d_mtab.p;
  v.src = pr->d_src.p;
  v.dst = pr->d_dst.p;
  v.in_ptr = pr->d_in_ptr.p;
  v.in_edge = pr->d_in_edge.p;
  v.budget = pr->d_budget.p;
  v.ubound = pr->d_ubound.p;
  v.table = pr->d_table.p;
  v.tfix = pr->d_tfix_noenergy.p;
  v.n_table = n_table;
  v.fix_k = pr->fix_k_plain;
  v.has_energy = 0;
  v.ebad = pr->d_ebad.p;
  v.q = pr->d_q.p;
  v.has_total = h.has_energy && h.has_total ? 1 : 0;
  v.total_rhs = h.total_limit - h.board;
}

}  // namespace xe
