// SPDX-License-Identifier: Apache-2.0
//
// Best-schedule search as one native call (xe_search): K1 -> K3 -> K4
// rounding -> K2, then the R-space local-search population (K4 moves + K2),
// all on the device of the problem handle, host code only for control.
//
// The reference reaches its schedules through solve_exact (memoised DFS,
// proj/src/solver.cpp:449-489, D*T <= 64) or solve_external (MPS -> an
// external MILP solver, solver.cpp:501-561); neither is a data-parallel
// path.  This is the GPU counterpart: every candidate is scored exactly with
// the reference's semantics (objective_value of the completion,
// check_assignment families, integer budgets, decode legality), the rounding
// incumbent is the first minimum in global index order (solver.cpp:57-61),
// and the local search only replaces it when strictly better.
//
//   rounding:  round `rounds` blocks of `n_per_round` candidates, block r
//              of rank k at global index first + (r*world + k)*n_per_round;
//              canonical saves (xe_move_cubes, no move); evaluate; keep the
//              best `chains` distinct objectives as the starting population
//   local search: each iteration evaluates `chain_n` neighbours of every
//              chain (1..max_moves R-space moves + canonical saves), a chain
//              moves to its best neighbour when it improves, or after
//              `stall` iterations without improvement (a kick)
// Scores: a valid schedule scores its objective; one that fails only on
// memory (BUDGET / U_BOUND) scores kOverBudget + its relative excess
// sum_d max(0, peak_d - b_d) / b_d, so chains seeded from over-budget
// candidates (tight budgets where the rounding finds no valid schedule)
// first descend to feasibility; anything else is never accepted.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "csr.hpp"

namespace xe {
bool move_supported(const xe_problem* pr);  // round.cu
namespace {

constexpr double kOverBudget = 1e200;  // above any schedule's objective
constexpr uint32_t kMemFlags = XE_F_BUDGET | XE_F_U_BOUND;

__host__ __device__ inline double score(double obj, uint32_t flags, uint32_t mask, const int64_t* peak,
                                        const int64_t* budget, int D) {
  if ((flags & mask) == 0u) return obj;
  if ((flags & mask & ~kMemFlags) != 0u) return INFINITY;
  double ex = 0.0;
  for (int d = 0; d < D; ++d)
    if (peak[d] > budget[d]) ex += static_cast<double>(peak[d] - budget[d]) / static_cast<double>(budget[d] > 0 ? budget[d] : 1);
  return kOverBudget + ex;
}

// scores of a rounding batch as sortable keys (non-negative doubles order as
// their bit patterns), with their indices
__global__ void score_keys_kernel(const double* __restrict__ obj, const uint32_t* __restrict__ flags,
                                  const int64_t* __restrict__ peak, const int64_t* __restrict__ budget, int D,
                                  uint32_t mask, int64_t n, uint64_t* __restrict__ key, int32_t* __restrict__ idx) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    key[i] = static_cast<uint64_t>(__double_as_longlong(score(obj[i], flags[i], mask, peak + i * D, budget, D)));
    idx[i] = static_cast<int32_t>(i);
  }
}

// best-scoring neighbour of every chain: one warp per chain, lowest index on ties
__global__ void chain_select_kernel(const double* __restrict__ obj, const uint32_t* __restrict__ flags,
                                    const int64_t* __restrict__ peak, const int64_t* __restrict__ budget, int D,
                                    uint32_t mask, int P, int M, double* __restrict__ vbest,
                                    int32_t* __restrict__ jbest) {
  const int lane = threadIdx.x & 31;
  const int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (p >= P) return;
  double bv = INFINITY;
  int bj = -1;
  for (int j = lane; j < M; j += 32) {
    const int64_t k = static_cast<int64_t>(p) * M + j;
    const double v = score(obj[k], flags[k], mask, peak + k * D, budget, D);
    if (v < bv) bv = v, bj = j;  // ascending j per lane: strict < keeps the first
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
    if (ov < bv || (ov == bv && oj >= 0 && (bj < 0 || oj < bj))) bv = ov, bj = oj;
  }
  if (lane == 0) {
    vbest[p] = bv;
    jbest[p] = bj;
  }
}

// accept: a chain takes its best neighbour when it improves, or after `stall`
// iterations without improvement when it has a valid neighbour
__global__ void chain_accept_kernel(const uint32_t* __restrict__ nb, const double* __restrict__ vbest,
                                    const int32_t* __restrict__ jbest, int M, int words, int stall,
                                    uint32_t* __restrict__ bases, double* __restrict__ cur,
                                    int32_t* __restrict__ stalled) {
  const int p = blockIdx.x;
  __shared__ int take;
  if (threadIdx.x == 0) {
    const double v = vbest[p];
    const bool better = v < cur[p];
    take = (better || (stalled[p] >= stall && isfinite(v))) ? 1 : 0;
    if (take) {
      cur[p] = v;
      stalled[p] = 0;
    } else {
      stalled[p] += 1;
    }
  }
  __syncthreads();
  if (!take) return;
  const uint32_t* src = nb + (static_cast<int64_t>(p) * M + jbest[p]) * words;
  uint32_t* dst = bases + static_cast<int64_t>(p) * words;
  for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
}

void check_rc(int rc) {
  if (rc != XE_OK) fail(rc, xe_last_error());
}

struct Cand {
  double obj;
  int64_t slot;  // position in the batch
};

}  // namespace

void search_device(const xe_problem* pr, const xe_model_opts& mo, const xe_search_opts& so, xe_search_result* res,
                   uint32_t* cube_host, int64_t* peaks_host, cudaStream_t s) {
  const HostProblem& h = pr->h;
  const auto t_start = std::chrono::steady_clock::now();
  auto out_of_time = [&] {
    if (so.time_limit_ms <= 0) return false;
    const auto ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t_start);
    return ms.count() >= so.time_limit_ms;
  };
  const int words = 2 * h.D * h.T * ((h.T + 31) / 32);
  const bool movable = move_supported(pr);  // the move kernel's cube fits shared memory
  const bool canonical = so.canonical && movable;
  const int chains = movable ? so.chains : 0;
  const uint32_t mask = so.valid_mask;
  std::memset(res, 0, sizeof *res);
  res->objective = res->rounding_objective = INFINITY;
  res->index = -1;
  res->lp_bound = res->lp_value = NAN;
  res->lp_certified = 1;

  // ---- K1 + K3: LP relaxation, its x on the device for the rounding
  DevBuf<double> x;
  if (so.use_lp) {
    xe_csr* m = nullptr;
    check_rc(xe_build_csr(pr, &mo, &m));
    struct Free {
      xe_csr* m;
      ~Free() { xe_csr_destroy(m); }
    } guard_m{m};
    xe_pdhg_opts po{};
    po.max_iters = 400000;
    po.tol_rel = so.lp_tol > 0 ? so.lp_tol : 1e-6;
    xe_pdhg_result lr{};
    xe_csr_info info{};
    check_rc(xe_csr_get_info(m, &info));
    std::vector<double> xh(static_cast<size_t>(info.n_cols));
    check_rc(xe_pdhg_solve(m, &po, &lr, xh.data(), nullptr));
    x.upload(xh, s);
    res->has_lp = 1;
    // the Lagrangian dual value b'y + sum_j min over [lb_j, ub_j] of the
    // reduced-cost term (every column is boxed, y is sign-projected) is a
    // lower bound of the presolved LP for ANY iterate, converged or not; it
    // bounds the full LP (and so the MILP) only when the prohibitive-cost
    // fixing is certified by the same duals
    res->lp_value = lr.primal_obj;
    res->lp_converged = lr.status == 0;
    res->lp_certified = lr.certified;
    res->lp_bound = lr.certified ? std::min(lr.dual_obj, lr.primal_obj) : -INFINITY;
  }

  // ---- rounding rounds
  const int64_t n = so.n_per_round;
  DevBuf<uint32_t> cubes;
  DevBuf<double> obj;
  DevBuf<uint32_t> flags;
  DevBuf<int64_t> peak;
  cubes.alloc(static_cast<size_t>(std::max<int64_t>(1, n)) * words);
  obj.alloc(std::max<int64_t>(1, n));
  flags.alloc(std::max<int64_t>(1, n));
  if (chains > 0) peak.alloc(static_cast<size_t>(std::max<int64_t>(1, n)) * h.D);
  std::vector<double> pool_obj;  // the population: best distinct objectives
  DevBuf<uint32_t> pool;
  pool.alloc(static_cast<size_t>(std::max(1, chains)) * words);
  DevBuf<uint64_t> keys, keys_out;
  DevBuf<int32_t> kidx, kidx_out;
  DevBuf<unsigned char> sort_tmp;
  auto candidates = [&](int64_t lo, int64_t cnt, uint32_t* out) {
    check_rc(xe_round_cubes(pr, so.use_lp ? x.p : nullptr, so.seed, lo, cnt, so.edits, 0.0, out, s));
    if (canonical) check_rc(xe_move_cubes(pr, out, cnt, 0, 0, cnt, 0, out, s));
  };
  for (int r = 0; r < so.rounds && n > 0; ++r) {
    if (r > 0 && out_of_time()) {
      res->time_limited = 1;
      break;
    }
    const int64_t lo = so.first + (static_cast<int64_t>(r) * so.world + so.rank) * n;
    candidates(lo, n, cubes.p);
    xe_eval_out eo{obj.p, chains > 0 ? peak.p : nullptr, flags.p};
    xe_best b{};
    check_rc(xe_eval_cubes(pr, &mo, cubes.p, n, &eo, mask, &b, s));
    res->n_valid += b.n_valid;
    res->n_evaluated += n;
    if (b.index >= 0 && b.obj < res->rounding_objective) {  // blocks ascend in index: strict <
      res->rounding_objective = b.obj;
      res->index = lo + b.index;
    }
    if (chains <= 0) continue;
    // merge the batch's best distinct scores into the population: scores
    // sorted on the device (stable radix sort: ties keep index order), only
    // the head comes back
    {
      keys.reserve(static_cast<size_t>(n));
      keys_out.reserve(static_cast<size_t>(n));
      kidx.reserve(static_cast<size_t>(n));
      kidx_out.reserve(static_cast<size_t>(n));
      const int g = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 16));
      score_keys_kernel<<<g, 256, 0, s>>>(obj.p, flags.p, peak.p, pr->d_budget.p, h.D, mask, n, keys.p, kidx.p);
      XE_CUDA(cudaGetLastError());
      size_t tb = 0;
      XE_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.p, keys_out.p, kidx.p, kidx_out.p,
                                              static_cast<int>(n), 0, 64, s));
      sort_tmp.reserve(std::max<size_t>(1, tb));
      XE_CUDA(cub::DeviceRadixSort::SortPairs(sort_tmp.p, tb, keys.p, keys_out.p, kidx.p, kidx_out.p,
                                              static_cast<int>(n), 0, 64, s));
    }
    // enough of the head for `chains` distinct scores (rounding repeats schedules)
    const int64_t head = std::min<int64_t>(n, 256 * static_cast<int64_t>(chains));
    std::vector<uint64_t> hk(static_cast<size_t>(head));
    std::vector<int32_t> hi(static_cast<size_t>(head));
    XE_CUDA(cudaMemcpyAsync(hk.data(), keys_out.p, head * 8, cudaMemcpyDeviceToHost, s));
    XE_CUDA(cudaMemcpyAsync(hi.data(), kidx_out.p, head * 4, cudaMemcpyDeviceToHost, s));
    XE_CUDA(cudaStreamSynchronize(s));
    std::vector<Cand> c;
    for (int i = 0; i < static_cast<int>(pool_obj.size()); ++i) c.push_back({pool_obj[static_cast<size_t>(i)], -1 - i});
    for (int64_t q = 0; q < head; ++q) {
      double v;
      std::memcpy(&v, &hk[static_cast<size_t>(q)], 8);
      if (!(v < INFINITY)) break;
      c.push_back({v, hi[static_cast<size_t>(q)]});
    }
    // pool entries first among equal objectives (they are older, lower index)
    std::stable_sort(c.begin(), c.end(), [](const Cand& a, const Cand& b) { return a.obj < b.obj; });
    DevBuf<uint32_t> next;
    next.alloc(static_cast<size_t>(chains) * words);
    std::vector<double> next_obj;
    for (const Cand& k : c) {
      if (static_cast<int>(next_obj.size()) == chains) break;
      if (!next_obj.empty() && k.obj == next_obj.back()) continue;
      const uint32_t* src = k.slot >= 0 ? cubes.p + k.slot * words : pool.p + (-1 - k.slot) * words;
      XE_CUDA(cudaMemcpyAsync(next.p + next_obj.size() * words, src, words * 4, cudaMemcpyDeviceToDevice, s));
      next_obj.push_back(k.obj);
    }
    XE_CUDA(cudaStreamSynchronize(s));
    pool = std::move(next);
    pool_obj = std::move(next_obj);
  }
  DevBuf<uint32_t> inc;
  inc.alloc(words);
  bool have = res->index >= 0;
  if (have) {
    res->objective = res->rounding_objective;
    candidates(res->index, 1, inc.p);
  }

  // ---- local-search population
  if (chains > 0 && !pool_obj.empty()) {
    const int P = chains, M = std::max(1, so.chain_n);
    const int64_t PM = static_cast<int64_t>(P) * M;
    DevBuf<uint32_t> bases, nb;
    DevBuf<double> cur, vbest, nobj;
    DevBuf<int32_t> jbest, stalled;
    DevBuf<uint32_t> nflags;
    DevBuf<int64_t> npeak;
    bases.alloc(static_cast<size_t>(P) * words);
    std::vector<double> cur_h(static_cast<size_t>(P));
    for (int p = 0; p < P; ++p) {
      const size_t q = static_cast<size_t>(p) % pool_obj.size();
      XE_CUDA(cudaMemcpyAsync(bases.p + static_cast<size_t>(p) * words, pool.p + q * words, words * 4,
                              cudaMemcpyDeviceToDevice, s));
      cur_h[static_cast<size_t>(p)] = pool_obj[q];
    }
    cur.upload(cur_h, s);
    stalled.upload(std::vector<int32_t>(static_cast<size_t>(P), 0), s);
    vbest.alloc(P);
    jbest.alloc(P);
    nb.alloc(static_cast<size_t>(PM) * words);
    nobj.alloc(PM);
    nflags.alloc(PM);
    npeak.alloc(static_cast<size_t>(PM) * h.D);
    const auto mi0 = std::min_element(cur_h.begin(), cur_h.end());
    double gbest = *mi0;
    DevBuf<uint32_t> gcube;
    gcube.alloc(words);
    // the population's best chain is the local search's incumbent until a
    // chain improves on it (its score may sit an ulp below the exact
    // rounding objective: the streaming evaluator's reassociation)
    XE_CUDA(cudaMemcpyAsync(gcube.p, bases.p + static_cast<size_t>(mi0 - cur_h.begin()) * words, words * 4,
                            cudaMemcpyDeviceToDevice, s));
    const uint64_t ls_seed = (so.seed * 1000003ull + static_cast<uint64_t>(so.rank)) & 0xFFFFFFFFFFFFull;
    for (int it = 0; it < so.chain_iters; ++it) {
      if (out_of_time()) {
        res->time_limited = 1;
        break;
      }
      check_rc(xe_move_cubes(pr, bases.p, P, ls_seed, static_cast<int64_t>(it) * PM, PM, so.max_moves, nb.p, s));
      xe_eval_out eo{nobj.p, npeak.p, nflags.p};
      check_rc(xe_eval_cubes(pr, &mo, nb.p, PM, &eo, mask, nullptr, s));
      chain_select_kernel<<<(P * 32 + 255) / 256, 256, 0, s>>>(nobj.p, nflags.p, npeak.p, pr->d_budget.p, h.D, mask,
                                                                P, M, vbest.p, jbest.p);
      chain_accept_kernel<<<P, 256, 0, s>>>(nb.p, vbest.p, jbest.p, M, words, so.stall, bases.p, cur.p, stalled.p);
      XE_CUDA(cudaGetLastError());
      XE_CUDA(cudaMemcpyAsync(cur_h.data(), cur.p, P * 8, cudaMemcpyDeviceToHost, s));
      XE_CUDA(cudaStreamSynchronize(s));
      res->n_evaluated += PM;
      const auto mi = std::min_element(cur_h.begin(), cur_h.end());
      if (*mi < gbest) {  // first chain holding the minimum
        gbest = *mi;
        XE_CUDA(cudaMemcpyAsync(gcube.p, bases.p + static_cast<size_t>(mi - cur_h.begin()) * words, words * 4,
                                cudaMemcpyDeviceToDevice, s));
        res->improvements += 1;
      }
    }
    if (gbest < kOverBudget && gbest < res->objective) {
      res->objective = gbest;
      XE_CUDA(cudaMemcpyAsync(inc.p, gcube.p, words * 4, cudaMemcpyDeviceToDevice, s));
      have = true;
    }
  }
  if (!have) return;  // no valid schedule: objective stays inf

  // ---- the incumbent re-scored alone: objective bits and peaks
  DevBuf<double> o1;
  DevBuf<int64_t> p1;
  DevBuf<uint32_t> f1;
  o1.alloc(1);
  p1.alloc(h.D);
  f1.alloc(1);
  xe_eval_out eo{o1.p, p1.p, f1.p};
  xe_best b{};
  check_rc(xe_eval_cubes(pr, &mo, inc.p, 1, &eo, mask, &b, s));
  // the batch scores may be the streaming evaluator's reassociated sums (within
  // #terms * 2^-53 relative); the single re-score is the reference's order
  if (b.index != 0 || !(std::fabs(b.obj - res->objective) <= 1e-9 * std::max(1.0, std::fabs(b.obj))))
    fail(XE_ERR_ARG, "search: incumbent re-evaluation mismatch");
  res->objective = b.obj;
  if (cube_host) XE_CUDA(cudaMemcpyAsync(cube_host, inc.p, words * 4, cudaMemcpyDeviceToHost, s));
  if (peaks_host) XE_CUDA(cudaMemcpyAsync(peaks_host, p1.p, h.D * 8, cudaMemcpyDeviceToHost, s));
  XE_CUDA(cudaStreamSynchronize(s));
}

}  // namespace xe

extern "C" void xe_search_opts_default(xe_search_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof *o);
  o->n_per_round = 1 << 18;
  o->rounds = 4;
  o->edits = 3;
  o->seed = 1;
  o->use_lp = 1;
  o->lp_tol = 1e-6;
  o->valid_mask = XE_F_CHECK_MASK | XE_F_BUDGET | XE_F_DECODE;
  o->canonical = 1;
  o->chains = 256;
  o->chain_n = 1024;
  o->chain_iters = 200;
  o->max_moves = 4;
  o->stall = 15;
  o->first = 0;
  o->rank = 0;
  o->world = 1;
  o->time_limit_ms = 0;
}

extern "C" int xe_search(const xe_problem* p, const xe_model_opts* opts, const xe_search_opts* so,
                         xe_search_result* res, uint32_t* cube_host, int64_t* peaks_host, void* stream) {
  return xe::guard([&] {
    if (!p || !res) xe::fail(XE_ERR_ARG, "null argument");
    xe::require_uploaded(p);
    xe_search_opts o;
    xe_search_opts_default(&o);
    if (so) o = *so;
    if (o.n_per_round < 0 || o.rounds < 0 || o.edits < 0 || o.chains < 0 || o.chain_n < 1 || o.chain_iters < 0 ||
        o.max_moves < 1 || o.stall < 1 || o.world < 1 || o.rank < 0 || o.rank >= o.world)
      xe::fail(XE_ERR_ARG, "bad search options");
    xe_model_opts mo{};
    if (opts) mo = *opts;
    xe::search_device(p, mo, o, res, cube_host, peaks_host, static_cast<cudaStream_t>(stream));
  });
}
