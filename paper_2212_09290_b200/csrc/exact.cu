// SPDX-License-Identifier: Apache-2.0
//
// solve_exact on the GPU (xe_solve_exact): the reference's exact search
// (proj/src/solver.cpp:101-489, the memoised DFS "Search") restated as a
// level-synchronous dynamic program over the same states and transitions,
// expanded in parallel.
//
// The reference's search space, per timestep t and entry state (one saved
// set per device, the memo key `(t, OR_d exit_d << d*T)`, solver.cpp:408-417):
//   * a computation set: operator t on exactly one device (cells, v == t,
//     solver.cpp:332-352) and, for every v < t, an optional non-empty device
//     subset recomputing v, allowed only when some consumer of v is computed
//     at t (solver.cpp:354-356), every device within its energy cap (cap_ok);
//   * legal when every computed operator's parents are available (entry or
//     computed) and the per-timestep energy total holds (leaf, :300-305);
//     step cost = the compute costs + every copy charge (:306-318);
//   * an exit subset per device among the resident tensors with a later
//     consumer (maxreach > t, :323-328), kept when the device's memory
//     trajectory stays within budget (mem_ok, :224-252).
// The optimum is the minimum under tail_less = (cost, sum R, sum S, bit
// string) (:87-92) of (step + child tail) — the composition is monotone in
// every key, so the principle of optimality holds exactly and the DP over
// (t, mask) returns the same tail as the memoised DFS.  Two keys compare
// a step's strings: both encode the step's computation and exit sets
// completely, so among different choices the string order is decided by the
// step's own bits (bit position d*T+i first ⇔ lowest set bit of the XOR).
//
// Phases: forward (level t -> t+1: every (state, computation set) pair is a
// GPU thread; children deduplicated by a device sort, keeping the cheapest
// prefix cost g), then backward (t = T-1 .. 0: the best tail of every kept
// state, one CTA per (state, configuration block), block reductions under
// tail_less).  Forward pruning: a child is dropped when g + lb[t+1] exceeds
// an upper bound known to be attained inside the search space (lb =
// solver.cpp:195-203's cheapest completion) — every dropped path costs more
// than the optimum, so the optimum and all its ties survive.  The step
// cost is summed in the reference's order (compute terms as cells adds them,
// then the copy charges of leaf); tails fold right (cand.cost = step_cost +
// child.cost, :284); for dyadic costs (every fixture and test problem) every
// partial sum is exact, otherwise the reference's own DFS arithmetic
// (f.cost += add ... -= add) drifts by rounding and the two agree to ~1 ulp
// per term.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <functional>
#include <limits>
#include <vector>

#include <thrust/binary_search.h>
#include <thrust/execution_policy.h>
#include <thrust/functional.h>
#include <thrust/reduce.h>
#include <thrust/sort.h>

#include "xe_internal.hpp"

namespace xe {
namespace ex {

constexpr int kB = 128;  // threads per block

// A computation set of one timestep: per-device masks packed at d*T, the
// compute cost as cells accumulates it, the number of computations.
struct Conf {
  uint64_t comp;
  double cost;
  int64_t r;
};

struct ExArgs {
  int D, T, E, strict, energy, t;
  double total_cap, ub;
  uint64_t pmask[64], cons[64], reach_gt[64];
  int64_t mass[64], bud[64];
  double lb[65];
  const double *c, *q, *devcap, *w;
  const int32_t *in_ptr, *in_src, *in_e;
  // level t
  const uint64_t* states;
  const double* g;
  int64_t nstates;
  const Conf* conf;  // the computation sets of timestep t
  uint64_t nconf;
  int64_t lo, hi;  // forward: flattened (state, configuration) range
  // forward outputs
  uint64_t* ch_mask;
  double* ch_g;
  unsigned long long* ch_cnt;
  int64_t ch_cap;
  unsigned long long* nodes;
  int* overflow;
  // backward: level t+1 and its tails
  const uint64_t* nstates_mask;
  int64_t n_next;
  const double* next_cost;
  const int32_t *next_r, *next_s;
  uint64_t conf_per_block;
  int groups;
};

// tail_less key of a candidate (cost, sum_r, sum_s, then the step's bits)
struct Key {
  double cost;
  int32_t r, s;
  uint64_t comp, exits;  // packed d*T+i
};

__host__ __device__ inline uint64_t brev64(uint64_t x) {
#ifdef __CUDA_ARCH__
  return __brevll(x);
#else
  uint64_t r = 0;
  for (int i = 0; i < 64; ++i) r |= ((x >> i) & 1ull) << (63 - i);
  return r;
#endif
}

// a < b under tail_less; strings compare position d*T+i first ('0' < '1')
__host__ __device__ inline bool key_less(const Key& a, const Key& b) {
  if (a.cost != b.cost) return a.cost < b.cost;
  if (a.r != b.r) return a.r < b.r;
  if (a.s != b.s) return a.s < b.s;
  if (a.comp != b.comp) return brev64(a.comp) < brev64(b.comp);
  return brev64(a.exits) < brev64(b.exits);
}

__device__ __forceinline__ bool cap_ok(const ExArgs& a, int d, int i) {
  return !a.energy || a.q[d * a.T + i] <= a.devcap[d];
}

__device__ __forceinline__ uint64_t above(int v) { return v >= 63 ? 0ull : (~0ull << (v + 1)); }

// Frame (t, entry) with computation set `cf` (state-independent: built on
// the host in cells' order, solver.cpp:325-398): false when some computed
// operator's parent is unavailable (leaf, :300-303); else the step cost =
// the computation set's cost + the copy charges of leaf (:306-318).
template <int MAXD>
__device__ bool frame_comp(const ExArgs& a, const uint64_t* entry, uint64_t entry_any, const Conf& cf,
                           uint64_t* comp, uint64_t& comp_any, double& step) {
  const int D = a.D, T = a.T;
  const uint64_t tmask = T >= 64 ? ~0ull : ((1ull << T) - 1ull);
  comp_any = 0;
  for (int d = 0; d < D; ++d) {
    comp[d] = (cf.comp >> (d * T)) & tmask;
    comp_any |= comp[d];
  }
  const uint64_t avail = entry_any | comp_any;
  for (uint64_t m = comp_any; m; m &= m - 1)
    if (a.pmask[__ffsll(m) - 1] & ~avail) return false;
  double wsum = 0.0;
  for (uint64_t m = comp_any; m; m &= m - 1) {
    const int o = __ffsll(m) - 1;
    for (int dc = 0; dc < D; ++dc) {
      if (!((comp[dc] >> o) & 1ull)) continue;
      for (int k2 = a.in_ptr[o]; k2 < a.in_ptr[o + 1]; ++k2) {
        const int src = a.in_src[k2], e = a.in_e[k2];
        for (int ds = 0; ds < D; ++ds) {
          if (ds == dc) continue;
          if (((entry[ds] | comp[ds]) >> src) & 1ull) wsum += a.w[(e * D + ds) * D + dc];
        }
      }
    }
  }
  step = cf.cost + wsum;
  return true;
}

// mem_ok (solver.cpp:224-252) of device d with exit set ex
__device__ bool mem_ok(const ExArgs& a, uint64_t en, uint64_t cm, uint64_t comp_any, uint64_t ex, int d) {
  const int T = a.T;
  const uint64_t scan = a.strict ? comp_any : cm;
  int64_t u = 0;
  for (uint64_t m = en; m; m &= m - 1) u += a.mass[__ffsll(m) - 1];
  if (cm & 1ull) u += a.mass[0];
  if (u > a.bud[d]) return false;
  const uint64_t res = en | cm;
  for (int v = 0; v + 1 < T; ++v) {
    if ((cm >> v) & 1ull) {
      for (int k2 = a.in_ptr[v]; k2 < a.in_ptr[v + 1]; ++k2) {
        const int src = a.in_src[k2];
        if (((res >> src) & 1ull) && !((ex >> src) & 1ull) && !(a.cons[src] & above(v) & scan)) u -= a.mass[src];
      }
      if (!((ex >> v) & 1ull) && !(a.cons[v] & above(v) & scan)) u -= a.mass[v];
    }
    if ((cm >> (v + 1)) & 1ull) u += a.mass[v + 1];
    if (u > a.bud[d]) return false;
  }
  return true;
}

constexpr int kMaxExitBits = 20;  // candidate saves per device and frame (2^20 exit sets)

// Calls fn(nmask) for every exit combination of a legal frame: an odometer
// over the devices, each digit stepping through its legal exit sets (subsets
// of its candidates passing mem_ok, which depends on that device alone).
// Returns false when a device has more than 2^kMaxExitBits exit sets.
template <int MAXD, class F>
__device__ bool for_exits(const ExArgs& a, const uint64_t* entry, const uint64_t* comp, uint64_t comp_any, F&& fn) {
  const int D = a.D, T = a.T, t = a.t;
  uint64_t cand[MAXD], cur[MAXD];
  for (int d = 0; d < D; ++d) {
    cand[d] = t + 1 < T ? ((entry[d] | comp[d]) & a.reach_gt[t]) : 0ull;
    if (__popcll(cand[d]) > kMaxExitBits) return false;
  }
  // first legal exit set of device d at or after s (descending subset order)
  auto first = [&](int d, uint64_t s, uint64_t& out) {
    for (;;) {
      if (mem_ok(a, entry[d], comp[d], comp_any, s, d)) {
        out = s;
        return true;
      }
      if (s == 0) return false;
      s = (s - 1) & cand[d];
    }
  };
  for (int d = 0; d < D; ++d)
    if (!first(d, cand[d], cur[d])) return true;  // no legal exit set on d: no child
  for (;;) {
    uint64_t nmask = 0;
    for (int d = 0; d < D; ++d) nmask |= cur[d] << (d * T);
    fn(nmask);
    int d = D - 1;
    for (; d >= 0; --d) {
      if (cur[d] != 0 && first(d, (cur[d] - 1) & cand[d], cur[d])) break;
      first(d, cand[d], cur[d]);  // wrap: exists (found before)
    }
    if (d < 0) return true;
  }
}

template <int MAXD>
__device__ __forceinline__ void unpack_entry(const ExArgs& a, uint64_t mask, uint64_t* entry, uint64_t& any) {
  const uint64_t tmask = a.T >= 64 ? ~0ull : ((1ull << a.T) - 1ull);
  any = 0;
  for (int d = 0; d < a.D; ++d) {
    entry[d] = (mask >> (d * a.T)) & tmask;
    any |= entry[d];
  }
}

template <int MAXD>
__global__ void __launch_bounds__(kB) forward_kernel(const __grid_constant__ ExArgs a) {
  unsigned long long my_nodes = 0;
  for (int64_t idx = a.lo + blockIdx.x * static_cast<int64_t>(kB) + threadIdx.x; idx < a.hi;
       idx += static_cast<int64_t>(gridDim.x) * kB) {
    const int64_t si = idx / static_cast<int64_t>(a.nconf);
    const uint64_t k = static_cast<uint64_t>(idx - si * static_cast<int64_t>(a.nconf));
    uint64_t entry[MAXD], comp[MAXD], entry_any, comp_any;
    unpack_entry<MAXD>(a, a.states[si], entry, entry_any);
    double step;
    if (!frame_comp<MAXD>(a, entry, entry_any, a.conf[k], comp, comp_any, step)) continue;
    ++my_nodes;
    const double gn = a.g[si] + step;
    if (gn + a.lb[a.t + 1] > a.ub) continue;  // every completion costs more than a known schedule
    const bool ok = for_exits<MAXD>(a, entry, comp, comp_any, [&](uint64_t nmask) {
      const unsigned long long pos = atomicAdd(a.ch_cnt, 1ull);
      if (pos < static_cast<unsigned long long>(a.ch_cap)) {
        a.ch_mask[pos] = nmask;
        a.ch_g[pos] = gn;
      }
    });
    if (!ok) atomicExch(a.overflow, 1);
  }
  atomicAdd(a.nodes, my_nodes);
}

template <int MAXD>
__global__ void __launch_bounds__(kB) backward_kernel(const __grid_constant__ ExArgs a, Key* partial) {
  const int64_t si = blockIdx.x / a.groups;
  const int grp = blockIdx.x % a.groups;
  Key best{INFINITY, 0, 0, 0, 0};
  uint64_t entry[MAXD], comp[MAXD], entry_any, comp_any;
  unpack_entry<MAXD>(a, a.states[si], entry, entry_any);
  const double gs = a.g[si];
  const uint64_t k0 = static_cast<uint64_t>(grp) * a.conf_per_block;
  const uint64_t k1 = a.nconf < k0 + a.conf_per_block ? a.nconf : k0 + a.conf_per_block;
  for (uint64_t k = k0 + threadIdx.x; k < k1; k += kB) {
    double step;
    const Conf cf = a.conf[k];
    if (!frame_comp<MAXD>(a, entry, entry_any, cf, comp, comp_any, step)) continue;
    if (gs + step + a.lb[a.t + 1] > a.ub) continue;  // as in the forward pass
    const uint64_t cpack = cf.comp;
    const int r = static_cast<int>(cf.r);
    for_exits<MAXD>(a, entry, comp, comp_any, [&](uint64_t nmask) {
      // the child's tail (level T: the empty tail)
      double cc = 0.0;
      int cr = 0, cs = 0;
      if (a.t + 1 < a.T) {
        int64_t lo = 0, hi = a.n_next;
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (a.nstates_mask[mid] < nmask) lo = mid + 1;
          else hi = mid;
        }
        if (lo >= a.n_next || a.nstates_mask[lo] != nmask) return;
        cc = a.next_cost[lo];
        if (!(cc < INFINITY)) return;
        cr = a.next_r[lo];
        cs = a.next_s[lo];
      }
      const Key kk{step + cc, r + cr, __popcll(nmask) + cs, cpack, nmask};
      if (key_less(kk, best)) best = kk;
    });
  }
  __shared__ Key sk[kB];
  sk[threadIdx.x] = best;
  __syncthreads();
  for (int o = kB / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o && key_less(sk[threadIdx.x + o], sk[threadIdx.x])) sk[threadIdx.x] = sk[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sk[0];
}

__global__ void reduce_tails_kernel(const Key* partial, int groups, int64_t n, double* cost, int32_t* r, int32_t* s,
                                    uint64_t* comp, uint64_t* exits) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  Key b = partial[i * groups];
  for (int gq = 1; gq < groups; ++gq)
    if (key_less(partial[i * groups + gq], b)) b = partial[i * groups + gq];
  cost[i] = b.cost;
  r[i] = b.r;
  s[i] = b.s;
  comp[i] = b.comp;
  exits[i] = b.exits;
}

struct MinG {
  __host__ __device__ double operator()(double x, double y) const { return x < y ? x : y; }
};

struct Level {
  DevBuf<uint64_t> mask;
  DevBuf<double> g;
  DevBuf<double> cost;
  DevBuf<int32_t> r, s;
  DevBuf<uint64_t> comp, exits;
  int64_t n = 0;
};

template <int MAXD>
void launch_forward(const ExArgs& a, int grid, cudaStream_t st) {
  forward_kernel<MAXD><<<grid, kB, 0, st>>>(a);
}
template <int MAXD>
void launch_backward(const ExArgs& a, int64_t blocks, Key* part, cudaStream_t st) {
  backward_kernel<MAXD><<<static_cast<unsigned>(blocks), kB, 0, st>>>(a, part);
}

}  // namespace ex

using ex::ExArgs;
using ex::Key;
using ex::Level;

// Host: builds the static tables, runs forward + backward, reconstructs.
void solve_exact_device(const xe_problem* pr, const xe_model_opts& mo, const xe_exact_opts& eo, xe_exact_result* res,
                        uint32_t* cube_host, cudaStream_t s) {
  const auto t0 = std::chrono::steady_clock::now();
  const HostProblem& h = pr->h;
  const int D = h.D, T = h.T, E = h.E;
  std::memset(res, 0, sizeof *res);
  res->objective = std::numeric_limits<double>::quiet_NaN();
  res->status = 2;
  if (D * T > 64) fail(XE_ERR_TOO_LARGE, "state space exceeds 64 residency bits");
  int64_t maxbud = 0;
  for (int64_t b : h.budget) maxbud = std::max(maxbud, b);
  for (int64_t m : h.mass)
    if (m > maxbud) {
      res->status = 1;  // solver.cpp:463-468
      return;
    }
  auto elapsed_ms = [&] {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  };
  auto out_of_time = [&] { return eo.time_limit_ms >= 0 && elapsed_ms() >= static_cast<double>(eo.time_limit_ms); };

  ExArgs a{};
  a.D = D;
  a.T = T;
  a.E = E;
  a.strict = mo.strict_free ? 1 : 0;
  a.energy = (mo.use_energy && h.has_energy) ? 1 : 0;
  a.total_cap = (a.energy && h.has_total) ? h.total_limit - h.board : INFINITY;
  std::vector<double> c(static_cast<size_t>(D) * T), q(static_cast<size_t>(D) * T, 0.0), devcap(D, INFINITY);
  for (int d = 0; d < D; ++d)
    for (int i = 0; i < T; ++i) {
      double v = h.cost[static_cast<size_t>(d) * T + i];
      if (a.energy) {
        q[static_cast<size_t>(d) * T + i] = h.q[static_cast<size_t>(d) * T + i];
        v += h.alpha * h.q[static_cast<size_t>(d) * T + i];  // solver.cpp:160-166
      }
      c[static_cast<size_t>(d) * T + i] = v;
    }
  if (a.energy)
    for (int d = 0; d < D; ++d)
      if (h.has_lim[static_cast<size_t>(d)]) devcap[static_cast<size_t>(d)] = h.lim[static_cast<size_t>(d)];
  std::vector<int32_t> in_ptr(T + 1, 0), in_src, in_e;
  std::vector<std::vector<int>> cons(T);
  for (int e = 0; e < E; ++e) {
    const int u = h.src[static_cast<size_t>(e)], v = h.dst[static_cast<size_t>(e)];
    a.pmask[v] |= 1ull << u;
    a.cons[u] |= 1ull << v;
    cons[static_cast<size_t>(u)].push_back(v);
    in_ptr[static_cast<size_t>(v) + 1]++;
  }
  for (int v = 0; v < T; ++v) in_ptr[static_cast<size_t>(v) + 1] += in_ptr[static_cast<size_t>(v)];
  in_src.assign(static_cast<size_t>(std::max(1, E)), 0);
  in_e.assign(static_cast<size_t>(std::max(1, E)), 0);
  {
    std::vector<int32_t> fillp(in_ptr.begin(), in_ptr.end() - 1);
    for (int e = 0; e < E; ++e) {  // pedges: edge order per destination (solver.cpp:174-180)
      const int v = h.dst[static_cast<size_t>(e)];
      in_src[static_cast<size_t>(fillp[static_cast<size_t>(v)])] = h.src[static_cast<size_t>(e)];
      in_e[static_cast<size_t>(fillp[static_cast<size_t>(v)]++)] = e;
    }
  }
  std::vector<int> maxreach(T, -1);
  for (int v = T - 1; v >= 0; --v)
    for (int x : cons[static_cast<size_t>(v)])
      maxreach[static_cast<size_t>(v)] =
          std::max({maxreach[static_cast<size_t>(v)], x, maxreach[static_cast<size_t>(x)]});
  for (int t = 0; t < T; ++t)
    for (int i = 0; i <= t; ++i)
      if (maxreach[static_cast<size_t>(i)] > t) a.reach_gt[t] |= 1ull << i;
  for (int i = 0; i < T; ++i) a.mass[i] = h.mass[static_cast<size_t>(i)];
  for (int d = 0; d < D; ++d) a.bud[d] = h.budget[static_cast<size_t>(d)];
  a.lb[T] = 0.0;
  for (int t = T - 1; t >= 0; --t) {  // solver.cpp:195-203
    double m = INFINITY;
    for (int d = 0; d < D; ++d)
      if (!a.energy || q[static_cast<size_t>(d) * T + t] <= devcap[static_cast<size_t>(d)])
        m = std::min(m, c[static_cast<size_t>(d) * T + t]);
    a.lb[t] = a.lb[t + 1] + m;
  }
  std::vector<double> w(static_cast<size_t>(std::max(1, E)) * D * D, 0.0);
  for (size_t i = 0; i < h.w.size(); ++i) w[i] = h.w[i];
  DevBuf<double> dc, dq, dcap, dw;
  DevBuf<int32_t> dinp, dins, dine;
  dc.upload(c, s);
  dq.upload(q, s);
  dcap.upload(devcap, s);
  dw.upload(w, s);
  dinp.upload(in_ptr, s);
  dins.upload(in_src, s);
  dine.upload(in_e, s);
  a.c = dc.p;
  a.q = dq.p;
  a.devcap = dcap.p;
  a.w = dw.p;
  a.in_ptr = dinp.p;
  a.in_src = dins.p;
  a.in_e = dine.p;
  if (D > 16) fail(XE_ERR_TOO_LARGE, "solve_exact: more than 16 devices");
  const int maxd = D <= 2 ? 2 : D <= 4 ? 4 : D <= 8 ? 8 : 16;
  // the computation sets of every timestep, in cells' order (solver.cpp:
  // 325-398): operator t on one device within its energy cap, then for v =
  // t-1 .. 0 either nothing or (when something computed here consumes v) a
  // non-empty device subset; compute and energy sums accumulated as cells
  // does (f.cost += add), the per-timestep energy total filtered (leaf :305)
  constexpr size_t kMaxConfs = size_t{1} << 24;
  auto cap_ok_h = [&](int d, int i) {
    return !a.energy || q[static_cast<size_t>(d) * T + i] <= devcap[static_cast<size_t>(d)];
  };
  std::vector<DevBuf<ex::Conf>> confs(static_cast<size_t>(T));
  std::vector<int64_t> nconfs(static_cast<size_t>(T), 0);
  for (int t = 0; t < T; ++t) {
    std::vector<ex::Conf> out;
    std::vector<uint64_t> comp(static_cast<size_t>(D), 0);
    std::function<void(int, uint64_t, double, double, int64_t)> cells = [&](int v, uint64_t any, double cost,
                                                                            double qq, int64_t r) {
      if (v < 0) {
        if (a.energy && qq > a.total_cap) return;
        uint64_t pk = 0;
        for (int d = 0; d < D; ++d) pk |= comp[static_cast<size_t>(d)] << (d * T);
        if (out.size() >= kMaxConfs) fail(XE_ERR_TOO_LARGE, "solve_exact: more than 2^24 computation sets in a timestep");
        out.push_back({pk, cost, r});
        return;
      }
      cells(v - 1, any, cost, qq, r);  // not recomputed
      if (!(a.cons[v] & any)) return;
      for (unsigned sig = 1; sig < (1u << D); ++sig) {
        bool ok = true;
        double add = 0, qadd = 0;
        for (int d = 0; d < D; ++d)
          if ((sig >> d) & 1u) {
            if (!cap_ok_h(d, v)) {
              ok = false;
              break;
            }
            add += c[static_cast<size_t>(d) * T + v];
            if (a.energy) qadd += q[static_cast<size_t>(d) * T + v];
          }
        if (!ok) continue;
        for (int d = 0; d < D; ++d)
          if ((sig >> d) & 1u) comp[static_cast<size_t>(d)] |= 1ull << v;
        cells(v - 1, any | (1ull << v), cost + add, qq + qadd, r + __builtin_popcount(sig));
        for (int d = 0; d < D; ++d)
          if ((sig >> d) & 1u) comp[static_cast<size_t>(d)] &= ~(1ull << v);
      }
    };
    for (int d = 0; d < D; ++d) {
      if (!cap_ok_h(d, t)) continue;
      comp[static_cast<size_t>(d)] = 1ull << t;
      const double add = c[static_cast<size_t>(d) * T + t];
      cells(t - 1, 1ull << t, 0.0 + add, a.energy ? 0.0 + q[static_cast<size_t>(d) * T + t] : 0.0, 1);
      comp[static_cast<size_t>(d)] = 0;
    }
    nconfs[static_cast<size_t>(t)] = static_cast<int64_t>(out.size());
    confs[static_cast<size_t>(t)].upload(out, s);
  }

  DevBuf<unsigned long long> cnt;  // [0] children, [1] nodes
  DevBuf<int> ovf;
  cnt.alloc(2);
  ovf.alloc(1);
  XE_CUDA(cudaMemsetAsync(ovf.p, 0, sizeof(int), s));
  a.nodes = cnt.p + 1;
  a.overflow = ovf.p;
  auto pol = thrust::cuda::par.on(s);

  struct DpOut {
    int status = 2;  // 0 optimal (within the run's space), 1 infeasible, 2 limit
    bool found = false;
    Key root{};
    std::vector<uint64_t> comps, exits;
  };
  int64_t nodes = 0, states = 0;
  const int64_t kChunk = 1ll << 22;           // frames per launch
  const int64_t kMaxChildren = 1ll << 27;      // raw children buffered before a dedup

  // One dynamic program over the search space: beam > 0 keeps the `beam`
  // cheapest-prefix states per timestep (a heuristic dive whose winner is a
  // schedule of the search space: an upper bound); beam == 0 is exact.
  auto run_dp = [&](int64_t beam, double ubv) -> DpOut {
    DpOut out;
    a.ub = std::isfinite(ubv) ? ubv + 1e-9 * std::max(1.0, std::fabs(ubv)) : INFINITY;
    std::vector<Level> lv(static_cast<size_t>(T) + 1);
    lv[0].mask.upload(std::vector<uint64_t>{0ull}, s);
    lv[0].g.upload(std::vector<double>{0.0}, s);
    lv[0].n = 1;
    states += 1;
    DevBuf<uint64_t> chm, tm;
    DevBuf<double> chg, tg;
    int64_t cap = 1 << 20;
    chm.alloc(static_cast<size_t>(cap));
    chg.alloc(static_cast<size_t>(cap));
    // sort + keep the cheapest prefix per distinct child, in place
    auto compact = [&](int64_t n) -> int64_t {
      if (n <= 1) return n;
      tm.reserve(static_cast<size_t>(n));
      tg.reserve(static_cast<size_t>(n));
      thrust::sort_by_key(pol, chm.p, chm.p + n, chg.p);
      auto ends = thrust::reduce_by_key(pol, chm.p, chm.p + n, chg.p, tm.p, tg.p, thrust::equal_to<uint64_t>(),
                                        ex::MinG());
      const int64_t m = ends.first - tm.p;
      XE_CUDA(cudaMemcpyAsync(chm.p, tm.p, m * 8, cudaMemcpyDeviceToDevice, s));
      XE_CUDA(cudaMemcpyAsync(chg.p, tg.p, m * 8, cudaMemcpyDeviceToDevice, s));
      return m;
    };
    // ---- forward: reachable states with their cheapest prefix cost
    for (int t = 0; t < T; ++t) {
      Level& cur = lv[static_cast<size_t>(t)];
      a.t = t;
      a.states = cur.mask.p;
      a.g = cur.g.p;
      a.nstates = cur.n;
      a.conf = confs[static_cast<size_t>(t)].p;
      a.nconf = static_cast<uint64_t>(nconfs[static_cast<size_t>(t)]);
      const long double total = static_cast<long double>(cur.n) * static_cast<long double>(a.nconf);
      if (total > 9.0e18L) fail(XE_ERR_TOO_LARGE, "solve_exact: frame count overflows");
      const int64_t nflat = cur.n * static_cast<int64_t>(a.nconf);
      int64_t nch = 0, chunk = kChunk;
      bool compacted = true;
      for (int64_t lo = 0; lo < nflat;) {
        if (out_of_time()) return out;
        int64_t ch = chunk;
        if (eo.node_limit >= 0) {
          if (nodes > eo.node_limit) return out;
          ch = std::min<int64_t>(ch, eo.node_limit - nodes + 1);
        }
        const int64_t hi = std::min(nflat, lo + ch);
        const unsigned long long c2[2] = {static_cast<unsigned long long>(nch), static_cast<unsigned long long>(nodes)};
        XE_CUDA(cudaMemcpyAsync(cnt.p, c2, 16, cudaMemcpyHostToDevice, s));
        a.lo = lo;
        a.hi = hi;
        a.ch_mask = chm.p;
        a.ch_g = chg.p;
        a.ch_cnt = cnt.p;
        a.ch_cap = cap;
        const int grid = static_cast<int>(std::min<int64_t>((hi - lo + ex::kB - 1) / ex::kB, 148 * 16));
        switch (maxd) {
          case 2: ex::launch_forward<2>(a, grid, s); break;
          case 4: ex::launch_forward<4>(a, grid, s); break;
          case 8: ex::launch_forward<8>(a, grid, s); break;
          default: ex::launch_forward<16>(a, grid, s); break;
        }
        XE_CUDA(cudaGetLastError());
        unsigned long long hc[2];
        int hov = 0;
        XE_CUDA(cudaMemcpyAsync(hc, cnt.p, 16, cudaMemcpyDeviceToHost, s));
        XE_CUDA(cudaMemcpyAsync(&hov, ovf.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        XE_CUDA(cudaStreamSynchronize(s));
        if (hov) fail(XE_ERR_TOO_LARGE, "solve_exact: more than 2^20 exit sets in one frame");
        if (hc[0] > static_cast<unsigned long long>(cap)) {
          // children overflowed: deduplicate what earlier chunks wrote, grow
          // the buffer up to its limit, else split the chunk; then redo it
          if (!compacted) {
            nch = compact(nch);
            compacted = true;
          }
          if (cap < kMaxChildren) {
            const int64_t ncap = std::min<int64_t>(kMaxChildren, std::max<int64_t>(2 * cap, nch + (hi - lo)));
            DevBuf<uint64_t> m2;
            DevBuf<double> g2;
            m2.alloc(static_cast<size_t>(ncap));
            g2.alloc(static_cast<size_t>(ncap));
            if (nch) {
              XE_CUDA(cudaMemcpyAsync(m2.p, chm.p, nch * 8, cudaMemcpyDeviceToDevice, s));
              XE_CUDA(cudaMemcpyAsync(g2.p, chg.p, nch * 8, cudaMemcpyDeviceToDevice, s));
            }
            chm = std::move(m2);
            chg = std::move(g2);
            cap = ncap;
          } else if (hi - lo > 1) {
            chunk = std::max<int64_t>(1, (hi - lo) / 4);
          } else {
            fail(XE_ERR_TOO_LARGE, "solve_exact: one frame has more than 2^27 exit combinations");
          }
          continue;
        }
        nodes = static_cast<int64_t>(hc[1]);
        nch = static_cast<int64_t>(hc[0]);
        compacted = false;
        if (nch > cap / 2) {
          nch = compact(nch);
          compacted = true;
        }
        if (eo.node_limit >= 0 && nodes > eo.node_limit) return out;
        lo = hi;
        chunk = std::min<int64_t>(kChunk, 2 * chunk);
      }
      // level t+1 = the distinct children, cheapest prefix kept
      Level& nx = lv[static_cast<size_t>(t) + 1];
      if (t + 1 < T) {
        int64_t m = compacted ? nch : compact(nch);
        if (beam > 0 && m > beam) {  // the beam: cheapest prefixes, then back to mask order
          thrust::sort_by_key(pol, chg.p, chg.p + m, chm.p);
          m = beam;
          thrust::sort_by_key(pol, chm.p, chm.p + m, chg.p);
        }
        nx.mask.alloc(static_cast<size_t>(std::max<int64_t>(1, m)));
        nx.g.alloc(static_cast<size_t>(std::max<int64_t>(1, m)));
        if (m) {
          XE_CUDA(cudaMemcpyAsync(nx.mask.p, chm.p, m * 8, cudaMemcpyDeviceToDevice, s));
          XE_CUDA(cudaMemcpyAsync(nx.g.p, chg.p, m * 8, cudaMemcpyDeviceToDevice, s));
        }
        nx.n = m;
        states += m;
        if (m > eo.max_states) return out;
        if (m == 0) break;  // nothing reaches t+1
      } else {
        nx.n = nch > 0 ? 1 : 0;  // the terminal state
      }
    }
    chm.release();
    chg.release();
    tm.release();
    tg.release();

    // ---- backward: the best tail of every kept state
    bool feasible = true;
    for (int t = T - 1; t >= 0; --t) {
      Level& cur = lv[static_cast<size_t>(t)];
      const size_t nn = static_cast<size_t>(std::max<int64_t>(1, cur.n));
      cur.cost.alloc(nn);
      cur.r.alloc(nn);
      cur.s.alloc(nn);
      cur.comp.alloc(nn);
      cur.exits.alloc(nn);
      if (cur.n == 0) continue;
      if (lv[static_cast<size_t>(t) + 1].n == 0) {
        feasible = false;
        break;
      }
      if (out_of_time()) return out;
      a.t = t;
      a.states = cur.mask.p;
      a.g = cur.g.p;
      a.nstates = cur.n;
      a.conf = confs[static_cast<size_t>(t)].p;
      a.nconf = static_cast<uint64_t>(nconfs[static_cast<size_t>(t)]);
      a.conf_per_block = std::max<uint64_t>(ex::kB, std::min<uint64_t>(a.nconf, 1ull << 12));
      a.groups = static_cast<int>((a.nconf + a.conf_per_block - 1) / a.conf_per_block);
      if (t + 1 < T) {
        const Level& nx = lv[static_cast<size_t>(t) + 1];
        a.nstates_mask = nx.mask.p;
        a.n_next = nx.n;
        a.next_cost = nx.cost.p;
        a.next_r = nx.r.p;
        a.next_s = nx.s.p;
      } else {
        a.nstates_mask = nullptr;
        a.n_next = 0;
      }
      const int64_t blocks = cur.n * a.groups;
      if (blocks > 0x7fffffffLL) fail(XE_ERR_TOO_LARGE, "solve_exact: too many states in one timestep");
      DevBuf<Key> part;
      part.alloc(static_cast<size_t>(blocks));
      switch (maxd) {
        case 2: ex::launch_backward<2>(a, blocks, part.p, s); break;
        case 4: ex::launch_backward<4>(a, blocks, part.p, s); break;
        case 8: ex::launch_backward<8>(a, blocks, part.p, s); break;
        default: ex::launch_backward<16>(a, blocks, part.p, s); break;
      }
      XE_CUDA(cudaGetLastError());
      ex::reduce_tails_kernel<<<static_cast<unsigned>((cur.n + 127) / 128), 128, 0, s>>>(
          part.p, a.groups, cur.n, cur.cost.p, cur.r.p, cur.s.p, cur.comp.p, cur.exits.p);
      XE_CUDA(cudaGetLastError());
      XE_CUDA(cudaStreamSynchronize(s));
    }
    out.status = 1;
    if (!feasible || lv[0].n == 0) return out;
    XE_CUDA(cudaMemcpyAsync(&out.root.cost, lv[0].cost.p, 8, cudaMemcpyDeviceToHost, s));
    XE_CUDA(cudaMemcpyAsync(&out.root.r, lv[0].r.p, 4, cudaMemcpyDeviceToHost, s));
    XE_CUDA(cudaMemcpyAsync(&out.root.s, lv[0].s.p, 4, cudaMemcpyDeviceToHost, s));
    XE_CUDA(cudaStreamSynchronize(s));
    if (!(out.root.cost < INFINITY)) return out;
    // the chain of best choices from the root
    out.comps.assign(static_cast<size_t>(T), 0);
    out.exits.assign(static_cast<size_t>(T), 0);
    int64_t idx = 0;
    for (int t = 0; t < T; ++t) {
      const Level& cur = lv[static_cast<size_t>(t)];
      XE_CUDA(cudaMemcpyAsync(&out.comps[static_cast<size_t>(t)], cur.comp.p + idx, 8, cudaMemcpyDeviceToHost, s));
      XE_CUDA(cudaMemcpyAsync(&out.exits[static_cast<size_t>(t)], cur.exits.p + idx, 8, cudaMemcpyDeviceToHost, s));
      XE_CUDA(cudaStreamSynchronize(s));
      if (t + 1 < T) {
        const Level& nx = lv[static_cast<size_t>(t) + 1];
        idx = thrust::lower_bound(pol, nx.mask.p, nx.mask.p + nx.n, out.exits[static_cast<size_t>(t)]) - nx.mask.p;
      }
    }
    out.status = 0;
    out.found = true;
    return out;
  };

  // an upper bound inside the search space: the caller's, else beam dives
  double ubv = eo.upper_bound;
  DpOut inc;
  if (!std::isfinite(ubv)) {
    for (int64_t beam : {int64_t{64}, int64_t{4096}}) {
      DpOut b = run_dp(beam, INFINITY);
      if (b.found) {
        inc = std::move(b);
        ubv = inc.root.cost;
        break;
      }
      if (b.status == 2) break;  // out of budget already
    }
  }
  DpOut fin = run_dp(0, ubv);
  res->nodes = nodes;
  res->states = states;
  const DpOut* best = nullptr;
  if (fin.status == 2) {  // limits: LimitReached with the dive's schedule, if any
    res->status = 2;
    if (inc.found) best = &inc;
  } else if (fin.status == 1) {
    // nothing at or below the bound: infeasible only without one (the dive's
    // schedule is itself feasible and would have been found)
    res->status = inc.found ? 0 : 1;
    if (inc.found) best = &inc;
  } else {
    res->status = 0;
    best = &fin;
  }
  res->ms = elapsed_ms();
  if (!best) return;
  res->found = 1;
  res->objective = best->root.cost;
  res->sum_r = best->root.r;
  res->sum_s = best->root.s;
  if (cube_host) {
    const int W = (T + 31) / 32;
    std::memset(cube_host, 0, static_cast<size_t>(2) * D * T * W * 4);
    const uint64_t tmask = T >= 64 ? ~0ull : ((1ull << T) - 1ull);
    for (int t = 0; t < T; ++t)
      for (int d = 0; d < D; ++d) {
        const uint64_t rc = (best->comps[static_cast<size_t>(t)] >> (d * T)) & tmask;
        const uint64_t se = (best->exits[static_cast<size_t>(t)] >> (d * T)) & tmask;
        for (int i = 0; i < T; ++i) {
          if ((rc >> i) & 1ull) cube_host[((static_cast<size_t>(0) * D + d) * T + t) * W + i / 32] |= 1u << (i % 32);
          if (t + 1 < T && ((se >> i) & 1ull))
            cube_host[((static_cast<size_t>(1) * D + d) * T + t + 1) * W + i / 32] |= 1u << (i % 32);
        }
      }
  }
}

}  // namespace xe

extern "C" void xe_exact_opts_default(xe_exact_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof *o);
  o->node_limit = -1;
  o->time_limit_ms = -1;
  o->upper_bound = INFINITY;
  o->max_states = 1ll << 26;
}

extern "C" int xe_solve_exact(const xe_problem* p, const xe_model_opts* opts, const xe_exact_opts* eo,
                              xe_exact_result* res, uint32_t* cube_host, void* stream) {
  return xe::guard([&] {
    if (!p || !res) xe::fail(XE_ERR_ARG, "null argument");
    xe::require_uploaded(p);
    xe_exact_opts o;
    xe_exact_opts_default(&o);
    if (eo) o = *eo;
    xe_model_opts mo{};
    if (opts) mo = *opts;
    xe::solve_exact_device(p, mo, o, res, cube_host, static_cast<cudaStream_t>(stream));
  });
}
