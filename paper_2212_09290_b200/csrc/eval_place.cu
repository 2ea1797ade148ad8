// SPDX-License-Identifier: Apache-2.0
//
// K2b — batched evaluation of device placements, and the assignment oracle.
//
// A placement candidate is dev[T] (uint8): op i computed once, at timestep i,
// on dev[i].  policy 0 is the reference's save-all family
// (save_all_assignment, proj/src/solver.cpp:30-42): every output stays saved
// on its device afterwards.  policy 1 (minimal-save) keeps a tensor only
// until its last consumer and never saves a tensor without consumers.
// On these cubes the completion has closed forms (verified
// against complete_assignment/objective_value/check_assignment):
//   objective = sum_d sum_{t: dev_t = d} c[d][t]              (R terms, d-major)
//             + sum over edges e=(u->v) in (v, e) order with dev_u != dev_v
//               of w[e][dev_u][dev_v]                         (copy terms)
//   save-all peak_d    = sum_{i: dev_i = d} m_i
//   minimal-save peak_d = max_t ( sum_{u < t <= last(u), dev_u = d} m_u + [dev_t = d] m_t )
// and only BUDGET / U_BOUND can fail (EQ8/11/12/16 and decode hold).
//
// One warp per candidate: the placement is staged in shared memory; lanes
// stride over ops and edges; EXACT mode sums int64 fixed point (any order),
// serial mode reproduces objective_value's sequential FP64 order on lane 0.
//
// assignment_oracle (solver.cpp:44-75): one thread per odometer index
// (op 0 most significant), save-all objective in the reference's order,
// first strict minimum = lowest index among equal objective bits.

#include <climits>
#include <cstdlib>
#include <cstring>

#include "bits.cuh"
#include "xe_internal.hpp"

namespace xe {
namespace place {

constexpr int kWarps = 8;

struct Args {
  int D, T, E, policy, fix_k;
  const int64_t* mass;
  const double* cost;     // [D][T]
  const double* w;        // [E][D][D]
  const int64_t* tfix;    // [D*T + E*D*D] fixed point
  const int64_t* tfix_edge;  // [E] when every cross-device copy of an edge costs the same (else null)
  const int64_t* tfix_op;    // [T][D] fixed-point compute costs, op-major (sliced kernel)
  const int32_t* src;
  const int32_t* dst;
  const int32_t* eorder;  // edges sorted by (dst, e)
  const int32_t* last;    // last consumer of each op, -1 if none
  const int32_t* lv_ptr;  // [T+1] ops grouped by last consumer
  const int32_t* lv_ops;
  const int64_t* budget;
  const double* ubound;
  const uint8_t* dev;
  int64_t n;
  double* obj;
  int64_t* peak;
  uint32_t* flags;
  uint32_t valid_mask;
  uint64_t* wbest_key;
  int64_t* wbest_idx;
  int64_t* wvalid;
};

template <bool EXACT>
__global__ void __launch_bounds__(kWarps * 32) place_kernel(const Args a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int T = a.T, D = a.D, E = a.E;
  const int tb = (T + 15) & ~15;
  // edge endpoints packed (src | dst << 16) in shared memory, then one
  // placement buffer per warp
  uint32_t* s_edge = reinterpret_cast<uint32_t*>(smem);
  const int eb = (4 * E + 15) & ~15;
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    s_edge[e] = static_cast<uint32_t>(a.src[e]) | (static_cast<uint32_t>(a.dst[e]) << 16);
  // the placement buffers, then per-lane peak accumulators [8][32] per warp
  // (the per-edge cost table stays in L1: staging it in shared memory halves
  // the resident warps, A/B: 84.5 M/s staged)
  const int teb = 0;
  uint8_t* sdev = smem + eb + teb + wid * tb;
  int64_t* s_acc = reinterpret_cast<int64_t*>(smem + eb + teb + kWarps * tb) + wid * 8 * 32;
  __syncthreads();
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * kWarps + wid;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * kWarps;
  uint64_t best_key = ~0ull;
  int64_t best_idx = -1, n_valid = 0;
  const bool vec = (T % 16) == 0 && (reinterpret_cast<uintptr_t>(a.dev) % 16) == 0;

  for (int64_t c = gw; c < a.n; c += nw) {
    const uint8_t* g = a.dev + c * T;
    if (vec) {  // 16-byte loads: one warp instruction moves 512 bytes
      for (int i = lane; i < T / 16; i += 32)
        reinterpret_cast<uint4*>(sdev)[i] = __ldg(reinterpret_cast<const uint4*>(g) + i);
    } else {
      for (int i = lane; i < T; i += 32) sdev[i] = g[i];
    }
    __syncwarp();
    // ---- objective
    double obj = 0.0;
    if (EXACT) {
      int64_t fix = 0;
      for (int i = lane; i < T; i += 32) fix += a.tfix[sdev[i] * T + i];
      const int base = D * T;
      if (a.tfix_edge) {  // one cost per edge: an 8E-byte table that stays in L1
#pragma unroll 4
        for (int e = lane; e < E; e += 32) {
          const uint32_t sd = s_edge[e];
          if (sdev[sd & 0xffffu] != sdev[sd >> 16]) fix += __ldg(a.tfix_edge + e);
        }
      } else {
#pragma unroll 4
        for (int e = lane; e < E; e += 32) {
          const uint32_t sd = s_edge[e];
          const int du = sdev[sd & 0xffffu], dv = sdev[sd >> 16];
          if (du != dv) fix += __ldg(a.tfix + base + (e * D + du) * D + dv);
        }
      }
      fix = warp_sum_i64(fix);
      obj = ldexp(static_cast<double>(fix), -a.fix_k);
    } else if (lane == 0) {  // objective_value's order (model.cpp:392-411)
      double total = 0.0;
      for (int d = 0; d < D; ++d)
        for (int t = 0; t < T; ++t)
          if (sdev[t] == d) total = __dadd_rn(total, a.cost[d * T + t]);
      for (int k = 0; k < E; ++k) {
        const int e = a.eorder[k];
        const int du = sdev[a.src[e]], dv = sdev[a.dst[e]];
        if (du != dv) total = __dadd_rn(total, a.w[(e * D + du) * D + dv]);
      }
      obj = total;
    }
    // ---- peaks
    int64_t pk[8];
#pragma unroll
    for (int d = 0; d < 8; ++d) pk[d] = 0;
    if (a.policy == 0) {
      // save-all peak_d = sum of the masses placed on d: lane-private shared
      // accumulators (acc[d][lane], conflict-free) instead of an 8-way select
#pragma unroll
      for (int x = 0; x < 8; ++x) s_acc[x * 32 + lane] = 0;
      for (int i = lane; i < T; i += 32) s_acc[sdev[i] * 32 + lane] += a.mass[i];
#pragma unroll
      for (int x = 0; x < 8; ++x)
        if (x < D) pk[x] = warp_sum_i64(s_acc[x * 32 + lane]);
    } else {
      // exact sequential sweep (lane 0): live sets per device
      if (lane == 0) {
        int64_t live[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) live[x] = 0;
        for (int t = 0; t < T; ++t) {
          if (t >= 1) {
            const int u = t - 1;
            if (a.last[u] >= t) {
              const int d = sdev[u];
#pragma unroll
              for (int x = 0; x < 8; ++x)
                if (x == d) live[x] += a.mass[u];
            }
          }
          const int dt = sdev[t];
#pragma unroll
          for (int x = 0; x < 8; ++x) {
            const int64_t v = live[x] + (x == dt ? a.mass[t] : 0);
            pk[x] = max(pk[x], v);
          }
          // tensors whose last consumer is t are not saved into t+1
          for (int k = a.lv_ptr[t]; k < a.lv_ptr[t + 1]; ++k) {
            const int u = a.lv_ops[k];
            if (u >= t) continue;
            const int d = sdev[u];
#pragma unroll
            for (int x = 0; x < 8; ++x)
              if (x == d) live[x] -= a.mass[u];
          }
        }
      }
#pragma unroll
      for (int x = 0; x < 8; ++x) pk[x] = __shfl_sync(0xffffffffu, pk[x], 0);
    }
    obj = __shfl_sync(0xffffffffu, obj, 0);
    uint32_t fl = 0;
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      if (x >= D) continue;
      if (pk[x] > a.budget[x]) fl |= XE_F_BUDGET;
      if (static_cast<double>(pk[x]) > a.ubound[x]) fl |= XE_F_U_BOUND;
    }
    if (lane == 0) {
      if (a.obj) a.obj[c] = obj;
      if (a.flags) a.flags[c] = fl;
      if (a.peak)
        for (int x = 0; x < D; ++x) a.peak[c * D + x] = pk[x];
      if ((fl & a.valid_mask) == 0) {
        ++n_valid;
        const uint64_t key = __double_as_longlong(obj);
        if (key < best_key || (key == best_key && c < best_idx)) {
          best_key = key;
          best_idx = c;
        }
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    a.wbest_key[gw] = best_key;
    a.wbest_idx[gw] = best_idx;
    a.wvalid[gw] = n_valid;
  }
}

// Save-all placements, fixed-point objective, one copy cost per edge (the
// compact tfix_edge table): the bit-sliced kernel.  A CTA takes 32
// placements at a time, one per lane.  Phase 1 (ops, split over the warps in
// 16-op blocks): lane k reads 16 device bytes of its placement, adds its
// compute terms and save-all masses, and the warp ballots the device bits into
// bit planes — plane b of op i holds bit b of dev_i of all 32 placements.
// Phase 2 (edges, split over the warps): per edge (u, v) one broadcast
// 8-byte load of its plane offsets and 32-bit cost, two broadcast 16-byte
// plane loads that give the 32-placement mask of dev_u != dev_v in up to
// three LOP3s, and each lane adds the cost when its bit is set: the per-edge
// gathers of the warp-per-placement kernel become broadcasts.  Config 5
// (T = 2000, E = 5987, D = 8): 82.5 -> 101 M placements/s (A/B: 16-warp
// CTAs 93, shared atomics for the masses 91, edge costs from L1 95).
#ifndef XE_SL_WARPS
#define XE_SL_WARPS 8
#endif
constexpr int kSlWarps = XE_SL_WARPS;

template <int NB>
__global__ void __launch_bounds__(kSlWarps * 32) place_sliced_kernel(const Args a, int acc32) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int T = a.T, D = a.D, E = a.E;
  uint4* planes = reinterpret_cast<uint4*>(smem);                          // [T]
  // per edge: plane byte offsets 16 src | 16 dst << 16, and its 32-bit cost
  uint2* s_edge = reinterpret_cast<uint2*>(planes + T);                    // [E]
  int64_t* s_acc = reinterpret_cast<int64_t*>(s_edge + ((E + 1) & ~1));    // [warps][8][32] save-all masses
  int64_t* s_fix = s_acc + kSlWarps * 8 * 32;                              // [warps][32]
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    s_edge[e] = make_uint2((16u * static_cast<uint32_t>(a.src[e])) | ((16u * static_cast<uint32_t>(a.dst[e])) << 16),
                           static_cast<uint32_t>(a.tfix_edge[e]));
  const unsigned char* pbase = reinterpret_cast<const unsigned char*>(planes);
  const bool vec = (T % 16) == 0 && (reinterpret_cast<uintptr_t>(a.dev) % 16) == 0;
  const int nblk = (T + 15) >> 4;
  const int e_per = (E + kSlWarps - 1) / kSlWarps;
  const int e0 = min(E, wid * e_per), e1 = min(E, e0 + e_per);
  uint64_t best_key = ~0ull;
  int64_t best_idx = -1, n_valid = 0;
  const int64_t ngroups = (a.n + 31) / 32;
  __syncthreads();
  for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
    const int64_t c = g * 32 + lane;
    const bool live = c < a.n;
    const uint8_t* row = a.dev + (live ? c : 0) * T;
    int64_t fix = 0;
#pragma unroll
    for (int x = 0; x < 8; ++x) s_acc[(wid * 8 + x) * 32 + lane] = 0;
    // ---- phase 1: ops, kG blocks of 16 per warp at a time: their bytes are
    // loaded together, then consumed (the loads of a group overlap)
    constexpr int kG = 4;
    for (int b0 = wid; b0 < nblk; b0 += kG * kSlWarps) {
      uint4 vg[kG];
#pragma unroll
      for (int g = 0; g < kG; ++g) {
        const int b = b0 + g * kSlWarps;
        if (vec) {
          vg[g] = (live && b < nblk) ? __ldg(reinterpret_cast<const uint4*>(row) + b) : make_uint4(0, 0, 0, 0);
        } else {
          uint32_t w4[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t x = 0;
#pragma unroll
            for (int y = 0; y < 4; ++y) {
              const int i = 16 * b + 4 * q + y;
              if (live && b < nblk && i < T) x |= static_cast<uint32_t>(row[i]) << (8 * y);
            }
            w4[q] = x;
          }
          vg[g] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
        }
      }
#pragma unroll
      for (int g = 0; g < kG; ++g) {
        const int b = b0 + g * kSlWarps;
        if (b >= nblk) break;  // warp-uniform
        const uint32_t wv[4] = {vg[g].x, vg[g].y, vg[g].z, vg[g].w};
        const int jn = min(16, T - 16 * b);  // warp-uniform
        const int64_t* tf = a.tfix_op + static_cast<int64_t>(16 * b) * D;
        const int64_t* ms = a.mass + 16 * b;
        // op j of the block: bit b of its device byte by an immediate mask
        auto op = [&](int j) {
          const uint32_t x = wv[j >> 2];
          const int sh = 8 * (j & 3);
          const int d = static_cast<int>((x >> sh) & 0xffu);
          const unsigned p0 = __ballot_sync(0xffffffffu, x & (1u << sh));
          const unsigned p1 = NB > 1 ? __ballot_sync(0xffffffffu, x & (2u << sh)) : 0u;
          const unsigned p2 = NB > 2 ? __ballot_sync(0xffffffffu, x & (4u << sh)) : 0u;
          if (lane == 0) planes[16 * b + j] = make_uint4(p0, p1, p2, 0u);
          fix += __ldg(tf + j * D + d);
          s_acc[(wid * 8 + d) * 32 + lane] += __ldg(ms + j);
        };
        if (jn == 16) {
#pragma unroll
          for (int j = 0; j < 16; ++j) op(j);
        } else {
          for (int j = 0; j < jn; ++j) op(j);
        }
      }
    }
    __syncthreads();
    // ---- phase 2: edges
    // a warp's edge costs sum in 32 bits when they cannot overflow
    // (acc32, checked on the host), else in 64
    auto edges = [&](auto acc) {
#pragma unroll 4
      for (int e = e0; e < e1; ++e) {
        const uint2 ed = s_edge[e];
        const uint32_t sd = ed.x;
        const uint4 pu = *reinterpret_cast<const uint4*>(pbase + (sd & 0xffffu));
        const uint4 pv = *reinterpret_cast<const uint4*>(pbase + (sd >> 16));
        unsigned diff = pu.x ^ pv.x;
        if (NB > 1) diff |= pu.y ^ pv.y;
        if (NB > 2) diff |= pu.z ^ pv.z;
        if ((diff >> lane) & 1u) acc += static_cast<decltype(acc)>(ed.y);
      }
      return acc;
    };
    if (acc32) fix += static_cast<int64_t>(edges(0u));
    else fix += edges(int64_t(0));
    s_fix[wid * 32 + lane] = fix;
    __syncthreads();
    // ---- warp 0: totals, flags, outputs
    if (wid == 0) {
      int64_t f = 0;
#pragma unroll
      for (int w = 0; w < kSlWarps; ++w) f += s_fix[w * 32 + lane];
      const double obj = ldexp(static_cast<double>(f), -a.fix_k);
      uint32_t fl = 0;
      int64_t pk[8];
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        int64_t v = 0;
#pragma unroll
        for (int w = 0; w < kSlWarps; ++w) v += s_acc[(w * 8 + x) * 32 + lane];
        pk[x] = v;
        if (x < D) {
          if (v > a.budget[x]) fl |= XE_F_BUDGET;
          if (static_cast<double>(v) > a.ubound[x]) fl |= XE_F_U_BOUND;
        }
      }
      if (live) {
        if (a.obj) a.obj[c] = obj;
        if (a.flags) a.flags[c] = fl;
        if (a.peak)
#pragma unroll
          for (int x = 0; x < 8; ++x)
            if (x < D) a.peak[c * D + x] = pk[x];
        if ((fl & a.valid_mask) == 0) {
          ++n_valid;
          const uint64_t key = __double_as_longlong(obj);
          if (key < best_key || (key == best_key && c < best_idx)) {
            best_key = key;
            best_idx = c;
          }
        }
      }
    }
    __syncthreads();  // planes, accumulators and partial sums are reused
  }
  if (wid == 0) {
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
      a.wbest_key[blockIdx.x] = best_key;
      a.wbest_idx[blockIdx.x] = best_idx;
      a.wvalid[blockIdx.x] = nv;
    }
  }
}

// op-major copy of the [D][T] fixed-point compute costs
__global__ void transpose_fix_kernel(const int64_t* tfix, int D, int T, int64_t* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < D * T) out[(k % T) * D + k / T] = tfix[k];
}

// ---- assignment oracle: thread per odometer index -------------------------
struct OracleArgs {
  int D, T, E;
  const double* cost;
  const double* w;
  const int32_t* src;
  const int32_t* dst;
  const int32_t* eorder;
  int64_t first, n;
  uint64_t* bkey;
  int64_t* bidx;
};

__global__ void oracle_kernel(const OracleArgs a) {
  __shared__ uint64_t sk[256];
  __shared__ int64_t si[256];
  uint64_t bk = ~0ull;
  int64_t bi = -1;
  uint8_t dev[64];
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < a.n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t idx = a.first + k, r = idx;
    for (int t = a.T - 1; t >= 0; --t) {
      dev[t] = static_cast<uint8_t>(r % a.D);
      r /= a.D;
    }
    double total = 0.0;  // objective_value order on the save-all cube
    for (int d = 0; d < a.D; ++d)
      for (int t = 0; t < a.T; ++t)
        if (dev[t] == d) total = __dadd_rn(total, a.cost[d * a.T + t]);
    for (int q = 0; q < a.E; ++q) {
      const int e = a.eorder[q];
      const int du = dev[a.src[e]], dv = dev[a.dst[e]];
      if (du != dv) total = __dadd_rn(total, a.w[(e * a.D + du) * a.D + dv]);
    }
    const uint64_t key = __double_as_longlong(total);
    if (key < bk || (key == bk && idx < bi)) {
      bk = key;
      bi = idx;
    }
  }
  sk[threadIdx.x] = bk;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const uint64_t ok = sk[threadIdx.x + s];
      const int64_t oi = si[threadIdx.x + s];
      if (oi >= 0 && (ok < sk[threadIdx.x] || (ok == sk[threadIdx.x] && (si[threadIdx.x] < 0 || oi < si[threadIdx.x])))) {
        sk[threadIdx.x] = ok;
        si[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    a.bkey[blockIdx.x] = sk[0];
    a.bidx[blockIdx.x] = si[0];
  }
}

}  // namespace place

namespace {

std::vector<int32_t> edges_by_dst(const HostProblem& h) {
  std::vector<int32_t> o(static_cast<size_t>(h.E));
  for (int e = 0; e < h.E; ++e) o[static_cast<size_t>(e)] = e;
  std::stable_sort(o.begin(), o.end(), [&](int a, int b) { return h.dst[static_cast<size_t>(a)] < h.dst[static_cast<size_t>(b)]; });
  return o;
}

}  // namespace

void eval_placements_device(const xe_problem* pr, const uint8_t* dev, int64_t n, int policy, double* obj,
                            int64_t* peak, uint32_t* flags, uint32_t valid_mask, uint64_t* best3,
                            unsigned char* scratch, cudaStream_t s) {
  const HostProblem& h = pr->h;
  if (!h.missing_link.empty() && h.D > 1) fail(XE_ERR_MISSING_LINK, h.missing_link);
  if (h.D > 8) fail(XE_ERR_TOO_LARGE, "placement evaluation supports D <= 8");
  if (policy != 0 && policy != 1) fail(XE_ERR_ARG, "policy must be 0 (save-all) or 1 (minimal-save)");
  DevBuf<int32_t> eorder, last;
  eorder.upload(h.E ? edges_by_dst(h) : std::vector<int32_t>(1, 0), s);
  std::vector<int32_t> lst(static_cast<size_t>(h.T), -1);
  for (int e = 0; e < h.E; ++e)
    lst[static_cast<size_t>(h.src[static_cast<size_t>(e)])] =
        std::max(lst[static_cast<size_t>(h.src[static_cast<size_t>(e)])], h.dst[static_cast<size_t>(e)]);
  last.upload(lst, s);
  std::vector<int32_t> lvp(static_cast<size_t>(h.T) + 1, 0), lvo;
  for (int u = 0; u < h.T; ++u)
    if (lst[static_cast<size_t>(u)] >= 0) lvp[static_cast<size_t>(lst[static_cast<size_t>(u)]) + 1]++;
  for (int t = 0; t < h.T; ++t) lvp[static_cast<size_t>(t) + 1] += lvp[static_cast<size_t>(t)];
  lvo.assign(static_cast<size_t>(std::max(1, lvp.back())), 0);
  {
    std::vector<int32_t> fill(lvp.begin(), lvp.end() - 1);
    for (int u = 0; u < h.T; ++u)
      if (lst[static_cast<size_t>(u)] >= 0) lvo[static_cast<size_t>(fill[static_cast<size_t>(lst[static_cast<size_t>(u)])]++)] = u;
  }
  DevBuf<int32_t> lv_ptr, lv_ops;
  lv_ptr.upload(lvp, s);
  lv_ops.upload(lvo, s);
  place::Args a{};
  a.D = h.D;
  a.T = h.T;
  a.E = h.E;
  a.policy = policy;
  a.fix_k = pr->fix_k_place;
  a.mass = pr->d_mass.p;
  a.cost = pr->d_cost.p;
  a.w = pr->d_w.p;
  a.tfix = pr->d_tfix_place.p;
  // copy cost uniform over device pairs per edge (a single link model, the
  // config-5 generator): the compact per-edge table
  DevBuf<int64_t> tedge;
  bool tedge32 = false;
  int64_t tedge_max = 0;
  if (pr->fix_k_place >= 0 && h.D > 1) {
    bool uniform = true;
    std::vector<int64_t> te(static_cast<size_t>(h.E));
    for (int e = 0; e < h.E && uniform; ++e) {
      const double w0 = h.w[(static_cast<size_t>(e) * h.D + 0) * h.D + 1];
      for (int x = 0; x < h.D && uniform; ++x)
        for (int y = 0; y < h.D; ++y)
          if (x != y && h.w[(static_cast<size_t>(e) * h.D + x) * h.D + y] != w0) {
            uniform = false;
            break;
          }
      te[static_cast<size_t>(e)] = static_cast<int64_t>(std::ldexp(w0, pr->fix_k_place));
    }
    if (uniform && h.E > 0) {
      tedge.upload(te, s);
      a.tfix_edge = tedge.p;
      tedge32 = std::all_of(te.begin(), te.end(), [](int64_t v) { return v >= INT32_MIN && v <= INT32_MAX; });
      for (int64_t v : te) tedge_max = std::max(tedge_max, v);
    }
  }
  a.src = pr->d_src.p;
  a.dst = pr->d_dst.p;
  a.eorder = eorder.p;
  a.last = last.p;
  a.lv_ptr = lv_ptr.p;
  a.lv_ops = lv_ops.p;
  a.budget = pr->d_budget.p;
  a.ubound = pr->d_ubound.p;
  a.dev = dev;
  a.n = n;
  a.obj = obj;
  a.peak = peak;
  a.flags = flags;
  a.valid_mask = valid_mask;
  int nsm = 0;
  XE_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, pr->device));
  const size_t nw_max = static_cast<size_t>(nsm) * 8 * 8;
  a.wbest_key = reinterpret_cast<uint64_t*>(scratch);
  a.wbest_idx = reinterpret_cast<int64_t*>(scratch + nw_max * 8);
  a.wvalid = reinterpret_cast<int64_t*>(scratch + nw_max * 16);
  const int tb = (h.T + 15) & ~15;
  if (h.T > 65535) fail(XE_ERR_TOO_LARGE, "placement evaluation supports T <= 65535");
  const char* sl_env = std::getenv("XE_PLACE_SLICED");
  if (policy == 0 && a.tfix_edge && tedge32 && h.T <= 4095 && !(sl_env && sl_env[0] == '0')) {
    // bit-sliced save-all kernel (one lane per placement)
    const size_t smem_sl = static_cast<size_t>(h.T) * 16 + static_cast<size_t>((h.E + 1) & ~1) * 8 +
                           static_cast<size_t>(place::kSlWarps) * (8 * 32 * 8 + 32 * 8);
    int dev_smem = 0;
    XE_CUDA(cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, pr->device));
    if (smem_sl <= static_cast<size_t>(dev_smem)) {
      DevBuf<int64_t> top;
      top.alloc(static_cast<size_t>(h.T) * h.D);
      place::transpose_fix_kernel<<<std::max(1, (h.T * h.D + 255) / 256), 256, 0, s>>>(a.tfix, h.D, h.T, top.p);
      XE_CUDA(cudaGetLastError());
      a.tfix_op = top.p;
      auto ks = h.D <= 2 ? place::place_sliced_kernel<1> : h.D <= 4 ? place::place_sliced_kernel<2>
                                                                     : place::place_sliced_kernel<3>;
      XE_CUDA(cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_sl)));
      int per_sm = 0;
      XE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ks, place::kSlWarps * 32, smem_sl));
      const int64_t groups = (n + 31) / 32;
      // one best slot per CTA; the scratch holds nsm * 64 slots
      const int grid = static_cast<int>(std::max<int64_t>(
          1, std::min<int64_t>(groups, static_cast<int64_t>(nsm) * std::max(1, std::min(per_sm, 8)))));
      if (n > 0) {
        // 32-bit edge sums when a warp's share of the edges cannot overflow them
        const int64_t cmax = tedge_max;
        const int64_t per_warp = (h.E + place::kSlWarps - 1) / place::kSlWarps;
        const int acc32 = cmax * per_warp < (int64_t(1) << 32) ? 1 : 0;
        ks<<<grid, place::kSlWarps * 32, smem_sl, s>>>(a, acc32);
        XE_CUDA(cudaGetLastError());
      }
      if (best3) {
        extern void reduce_best_launch(const uint64_t* key, const int64_t* idx, const int64_t* valid, int n,
                                       uint64_t* out, cudaStream_t s);
        if (n > 0) {
          reduce_best_launch(a.wbest_key, a.wbest_idx, a.wvalid, grid, best3, s);
        } else {
          const uint64_t none[3] = {~0ull, ~0ull, 0ull};
          XE_CUDA(cudaMemcpyAsync(best3, none, sizeof none, cudaMemcpyHostToDevice, s));
        }
      }
      XE_CUDA(cudaStreamSynchronize(s));
      return;
    }
  }
  const int smem = ((4 * h.E + 15) & ~15) + place::kWarps * tb + place::kWarps * 8 * 32 * 8;
  const bool exact = pr->fix_k_place >= 0;
  auto k = exact ? place::place_kernel<true> : place::place_kernel<false>;
  XE_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 0;
  XE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, place::kWarps * 32, smem));
  const int64_t want = (n + place::kWarps - 1) / place::kWarps;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, static_cast<int64_t>(nsm) * std::max(1, std::min(per_sm, 8)))));
  if (n > 0) {
    k<<<grid, place::kWarps * 32, smem, s>>>(a);
    XE_CUDA(cudaGetLastError());
  }
  if (best3) {
    extern void reduce_best_launch(const uint64_t* key, const int64_t* idx, const int64_t* valid, int n,
                                   uint64_t* out, cudaStream_t s);
    if (n > 0) {
      reduce_best_launch(a.wbest_key, a.wbest_idx, a.wvalid, grid * place::kWarps, best3, s);
    } else {
      const uint64_t none[3] = {~0ull, ~0ull, 0ull};
      XE_CUDA(cudaMemcpyAsync(best3, none, sizeof none, cudaMemcpyHostToDevice, s));
    }
  }
  XE_CUDA(cudaStreamSynchronize(s));  // the order/last tables are call-local
}

void assignment_oracle_device(const xe_problem* pr, double* best_obj, int32_t* best_dev, int64_t* n_eval,
                              cudaStream_t s) {
  const HostProblem& h = pr->h;
  if (!h.missing_link.empty() && h.D > 1) fail(XE_ERR_MISSING_LINK, h.missing_link);
  if (h.T > 64) fail(XE_ERR_TOO_LARGE, "placement family too large to enumerate");
  double combos = 1.0;
  for (int i = 0; i < h.T; ++i) combos *= h.D;
  // the reference stops at 4e6 (solver.cpp:49); the sweep goes to 2^40
  if (combos > 1099511627776.0) fail(XE_ERR_TOO_LARGE, "placement family too large to enumerate");
  const int64_t n = static_cast<int64_t>(combos);
  DevBuf<int32_t> eorder;
  eorder.upload(h.E ? edges_by_dst(h) : std::vector<int32_t>(1, 0), s);
  place::OracleArgs a{};
  a.D = h.D;
  a.T = h.T;
  a.E = h.E;
  a.cost = pr->d_cost.p;
  a.w = pr->d_w.p;
  a.src = pr->d_src.p;
  a.dst = pr->d_dst.p;
  a.eorder = eorder.p;
  int nsm = 0;
  XE_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, pr->device));
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, nsm * 16)));
  DevBuf<uint64_t> bk;
  DevBuf<int64_t> bi;
  bk.alloc(static_cast<size_t>(grid));
  bi.alloc(static_cast<size_t>(grid));
  a.first = 0;
  a.n = n;
  a.bkey = bk.p;
  a.bidx = bi.p;
  place::oracle_kernel<<<grid, 256, 0, s>>>(a);
  XE_CUDA(cudaGetLastError());
  std::vector<uint64_t> hk(static_cast<size_t>(grid));
  std::vector<int64_t> hi(static_cast<size_t>(grid));
  XE_CUDA(cudaMemcpyAsync(hk.data(), bk.p, grid * 8, cudaMemcpyDeviceToHost, s));
  XE_CUDA(cudaMemcpyAsync(hi.data(), bi.p, grid * 8, cudaMemcpyDeviceToHost, s));
  XE_CUDA(cudaStreamSynchronize(s));
  uint64_t key = ~0ull;
  int64_t idx = -1;
  for (int g = 0; g < grid; ++g)
    if (hi[static_cast<size_t>(g)] >= 0 &&
        (hk[static_cast<size_t>(g)] < key || (hk[static_cast<size_t>(g)] == key && hi[static_cast<size_t>(g)] < idx))) {
      key = hk[static_cast<size_t>(g)];
      idx = hi[static_cast<size_t>(g)];
    }
  std::memcpy(best_obj, &key, 8);
  int64_t r = idx;
  for (int t = h.T - 1; t >= 0; --t) {
    best_dev[t] = static_cast<int32_t>(r % h.D);
    r /= h.D;
  }
  *n_eval = n;
}

}  // namespace xe
