// SPDX-License-Identifier: Apache-2.0
//
// The executable reading of schedules on the GPU (proj/src/schedule.cpp):
//
//   decode    schedule.cpp:40-129   per (candidate, timestep) thread: the
//             action list of the timestep (copies from the lowest device
//             holding the tensor, the compute, the fired frees; then the
//             end-of-timestep drops) — timesteps are independent, slots
//             restart at 0 — counted, prefix-summed, then written; the
//             first IllegalAssignment in the reference's order is reported
//   validate  schedule.cpp:131-240  per schedule: the residency / memory
//             simulation through the action list, every violation
//   replay    schedule.cpp:261-369  per schedule: total action cost, the
//             Eq. 1 objective rebuilt from availability, and the per-slot
//             memory series (one sample per (device, t, v)) with its peaks
//
// Input bits per candidate, from canonical (R, S) cubes completed with
// complete_assignment's semantics (model.cpp:471-549: Z = R|S, F hazards) or
// read from a dense assignment vector (x > 0.5, the map's own values):
//   R, S, Z  [D][T][NW] u64 rows;  F  [D][T][NWF] u64 (edge ordinals, then E+v self)
// The batch unit is the top-K of an evaluated candidate set: the schedules a
// caller turns into artifacts (format_schedule / trace_csv, schedule_text.cpp).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include <thrust/execution_policy.h>
#include <thrust/scan.h>

#include "xe_internal.hpp"

namespace xe {
namespace sch {

struct Bits {
  int D, T, E, NW, NWF;
  uint64_t* R;  // [n][D][T][NW]
  uint64_t* S;
  uint64_t* Z;
  uint64_t* F;  // [n][D][T][NWF]
  __device__ size_t row(int64_t c, int d, int t) const { return ((static_cast<size_t>(c) * D + d) * T + t) * NW; }
  __device__ size_t frow(int64_t c, int d, int t) const { return ((static_cast<size_t>(c) * D + d) * T + t) * NWF; }
  __device__ bool r(int64_t c, int d, int t, int i) const { return (R[row(c, d, t) + (i >> 6)] >> (i & 63)) & 1ull; }
  __device__ bool s(int64_t c, int d, int t, int i) const { return (S[row(c, d, t) + (i >> 6)] >> (i & 63)) & 1ull; }
  __device__ bool z(int64_t c, int d, int t, int i) const { return (Z[row(c, d, t) + (i >> 6)] >> (i & 63)) & 1ull; }
  __device__ bool f(int64_t c, int d, int t, int eo) const { return (F[frow(c, d, t) + (eo >> 6)] >> (eo & 63)) & 1ull; }
};

struct Tabs {  // problem tables (device)
  const int64_t* mass;
  const double* cost;  // [D][T] costs_ms
  const double* w;     // [E][D][D] copy_cost
  const double* q;     // [D][T] energy q (or null)
  double alpha;
  int energy;
  const int32_t *src, *dst, *in_ptr, *in_edge;
  const uint64_t* cons;  // [T][NW]
};

// ---- bits from canonical cubes: Z = R|S, F per complete_assignment
__global__ void bits_from_cubes_kernel(const uint32_t* __restrict__ cubes, int64_t n, Bits b, Tabs tb, int strict) {
  const int D = b.D, T = b.T, E = b.E, W = (T + 31) / 32;
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= n * D * T) return;
  const int64_t c = k / (D * T);
  const int d = static_cast<int>(k / T % D), t = static_cast<int>(k % T);
  const size_t cw = static_cast<size_t>(2) * D * T * W;
  auto cube_row = [&](int which, int dd, int tt, uint64_t* out) {
    const uint32_t* p = cubes + c * cw + ((static_cast<size_t>(which) * D + dd) * T + tt) * W;
    for (int j = 0; j < b.NW; ++j) {
      const uint64_t lo = 2 * j < W ? p[2 * j] : 0u, hi = 2 * j + 1 < W ? p[2 * j + 1] : 0u;
      out[j] = lo | (hi << 32);
    }
  };
  uint64_t r[4], s[4], sn[4], rany[4];
  cube_row(0, d, t, r);
  cube_row(1, d, t, s);
  for (int j = 0; j < b.NW; ++j) sn[j] = 0, rany[j] = 0;
  if (t + 1 < T) cube_row(1, d, t + 1, sn);
  if (strict)
    for (int dd = 0; dd < D; ++dd) {
      uint64_t x[4];
      cube_row(0, dd, t, x);
      for (int j = 0; j < b.NW; ++j) rany[j] |= x[j];
    }
  const size_t o = b.row(c, d, t);
  for (int j = 0; j < b.NW; ++j) {
    b.R[o + j] = r[j];
    b.S[o + j] = s[j];
    b.Z[o + j] = r[j] | s[j];
  }
  auto bit = [](const uint64_t* x, int i) { return (x[i >> 6] >> (i & 63)) & 1ull; };
  // F(u -> v) = R(v) Z(u) !S(t+1,u) and no later consumer of u computed (model.cpp:492-505)
  auto fires = [&](int u, int v) -> bool {
    if (!bit(r, v) || !(bit(r, u) | bit(s, u))) return false;
    if (t + 1 < T && bit(sn, u)) return false;
    const uint64_t* scan = strict ? rany : r;
    for (int j = 0; j < b.NW; ++j) {
      uint64_t above = ~0ull;
      if (64 * j + 63 <= v) above = 0;
      else if (64 * j <= v) above = (v & 63) == 63 ? 0ull : (~0ull << ((v & 63) + 1));
      if (tb.cons[u * b.NW + j] & above & scan[j]) return false;
    }
    return true;
  };
  const size_t fo = b.frow(c, d, t);
  for (int j = 0; j < b.NWF; ++j) b.F[fo + j] = 0;
  for (int e = 0; e < E; ++e)
    if (fires(tb.src[e], tb.dst[e])) b.F[fo + (e >> 6)] |= 1ull << (e & 63);
  for (int v = 0; v < T; ++v)
    if (fires(v, v)) b.F[fo + ((E + v) >> 6)] |= 1ull << ((E + v) & 63);
}

// ---- bits from a dense assignment (VarRef column order), x > 0.5
__global__ void bits_from_dense_kernel(const double* __restrict__ x, Bits b) {
  const int D = b.D, T = b.T, FE = b.E + b.T;
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= static_cast<int64_t>(D) * T) return;
  const int d = static_cast<int>(k / T), t = static_cast<int>(k % T);
  const int64_t DT2 = static_cast<int64_t>(D) * T * T, base = (static_cast<int64_t>(d) * T + t) * T;
  const size_t o = b.row(0, d, t), fo = b.frow(0, d, t);
  for (int j = 0; j < b.NW; ++j) b.R[o + j] = b.S[o + j] = b.Z[o + j] = 0;
  for (int i = 0; i < T; ++i) {
    if (x[base + i] > 0.5) b.R[o + (i >> 6)] |= 1ull << (i & 63);
    if (x[DT2 + base + i] > 0.5) b.S[o + (i >> 6)] |= 1ull << (i & 63);
    if (x[2 * DT2 + base + i] > 0.5) b.Z[o + (i >> 6)] |= 1ull << (i & 63);
  }
  for (int j = 0; j < b.NWF; ++j) b.F[fo + j] = 0;
  const int64_t fbase = 3 * DT2 + (static_cast<int64_t>(d) * T + t) * FE;
  for (int eo = 0; eo < FE; ++eo)
    if (x[fbase + eo] > 0.5) b.F[fo + (eo >> 6)] |= 1ull << (eo & 63);
}

// ---- decode: one thread per (candidate, timestep); WRITE = 0 counts
template <bool WRITE>
__global__ void decode_kernel(Bits b, Tabs tb, int64_t n, const int64_t* __restrict__ off, xe_action* __restrict__ out,
                              int64_t* __restrict__ count, int32_t* __restrict__ err) {
  const int D = b.D, T = b.T, E = b.E;
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= n * T) return;
  if (WRITE) {  // a failed candidate's timesteps were zeroed: nothing to write
    const int64_t c0 = k / T;
    if (off[c0 * T + T] == off[c0 * T]) return;
  }
  const int64_t c = k / T;
  const int t = static_cast<int>(k % T);
  uint64_t freed[8][4];
  for (int d = 0; d < D; ++d)
    for (int j = 0; j < b.NW; ++j) freed[d][j] = 0;
  int slot = 0;
  int64_t pos = WRITE ? off[k] : 0;
  int ecode = 0, ev = -1, eu = -1;
  auto emit = [&](int kind, int dev, int op, int src, int dst, int from, int to) {
    if (WRITE) out[pos++] = xe_action{kind, t, slot, dev, op, src, dst, from, to};
    ++slot;
  };
  for (int v = 0; v <= t && !ecode; ++v)
    for (int d = 0; d < D && !ecode; ++d) {
      if (!b.r(c, d, t, v)) continue;
      for (int q = tb.in_ptr[v]; q < tb.in_ptr[v + 1]; ++q) {
        const int e = tb.in_edge[q], u = tb.src[e];
        if (b.z(c, d, t, u)) continue;
        int sd = -1;
        for (int d2 = 0; d2 < D; ++d2)
          if (b.z(c, d2, t, u)) {
            sd = d2;
            break;
          }
        if (sd < 0 || ((freed[sd][u >> 6] >> (u & 63)) & 1ull)) {
          ecode = sd < 0 ? 1 : 2;
          ev = v;
          eu = u;
          break;
        }
        emit(1, -1, -1, u, v, sd, d);
      }
      if (ecode) break;
      emit(0, d, v, -1, -1, -1, -1);
      for (int q = tb.in_ptr[v]; q < tb.in_ptr[v + 1]; ++q) {
        const int e = tb.in_edge[q], u = tb.src[e];
        if (!b.f(c, d, t, e)) continue;
        emit(2, d, -1, u, v, -1, -1);
        freed[d][u >> 6] |= 1ull << (u & 63);
      }
      if (b.f(c, d, t, E + v)) {
        emit(2, d, -1, v, v, -1, -1);
        freed[d][v >> 6] |= 1ull << (v & 63);
      }
    }
  if (!ecode)
    for (int d = 0; d < D; ++d)
      for (int i = 0; i < T; ++i) {
        if (!b.z(c, d, t, i) || ((freed[d][i >> 6] >> (i & 63)) & 1ull)) continue;
        if (t + 1 < T && b.s(c, d, t + 1, i)) continue;
        emit(3, d, i, -1, -1, -1, -1);
      }
  if (!WRITE) {
    count[k] = ecode ? 0 : slot;
    err[k * 3 + 0] = ecode;
    err[k * 3 + 1] = ev;
    err[k * 3 + 2] = eu;
  }
}

// ---- validate: one thread per schedule (the reference's simulation is sequential)
template <bool WRITE>
__global__ void validate_kernel(const xe_action* __restrict__ act, const int64_t* __restrict__ aoff, int64_t n,
                                int D, int T, int NW, Tabs tb, const int64_t* __restrict__ bud,
                                const int64_t* __restrict__ voff, xe_violation* __restrict__ vout,
                                int64_t* __restrict__ vcount, uint64_t* __restrict__ scratch) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (c >= n) return;
  // per-schedule scratch: res [D][NW], copyin [D][NW], ever [NW]
  uint64_t* res = scratch + c * (2 * D + 1) * NW;
  uint64_t* cin = res + D * NW;
  uint64_t* ever = cin + D * NW;
  for (int i = 0; i < (2 * D + 1) * NW; ++i) res[i] = 0;
  auto bit = [&](const uint64_t* m, int d, int i) { return (m[d * NW + (i >> 6)] >> (i & 63)) & 1ull; };
  auto set = [&](uint64_t* m, int d, int i, bool on) {
    if (on) m[d * NW + (i >> 6)] |= 1ull << (i & 63);
    else m[d * NW + (i >> 6)] &= ~(1ull << (i & 63));
  };
  int64_t nv = 0, vpos = WRITE ? voff[c] : 0;
  auto viol = [&](int kind, int dev, int t, int slot, int64_t bytes, int a, int bb) {
    if (WRITE) vout[vpos++] = xe_violation{kind, dev, t, slot, bytes, a, bb};
    ++nv;
  };
  int64_t bytes[8];
  int64_t k = aoff[c];
  const int64_t kend = aoff[c + 1];
  for (int t = 0; t < T; ++t) {
    for (int d = 0; d < D; ++d) {
      bytes[d] = 0;
      for (int i = 0; i < T; ++i)
        if (bit(res, d, i)) bytes[d] += tb.mass[i];
    }
    for (int i = 0; i < D * NW; ++i) cin[i] = 0;
    for (; k < kend && act[k].timestep == t; ++k) {
      const xe_action a = act[k];
      if (a.kind == 0) {  // Compute
        for (int q = tb.in_ptr[a.op]; q < tb.in_ptr[a.op + 1]; ++q) {
          const int u = tb.src[tb.in_edge[q]];
          if (bit(res, a.device, u) || bit(cin, a.device, u)) continue;
          viol(0, a.device, t, a.slot, 0, a.op, u);
        }
        set(res, a.device, a.op, true);
        ever[a.op >> 6] |= 1ull << (a.op & 63);
        bytes[a.device] += tb.mass[a.op];
        if (bytes[a.device] > bud[a.device]) viol(2, a.device, t, a.slot, bytes[a.device], -1, -1);
      } else if (a.kind == 1) {  // Copy
        if (!bit(res, a.from, a.src)) viol(1, a.from, t, a.slot, 0, a.src, -1);
        set(cin, a.to, a.src, true);
      } else {  // Free / Drop
        const int tensor = a.kind == 2 ? a.src : a.op;
        if (!bit(res, a.device, tensor)) {
          viol(3, a.device, t, a.slot, 0, tensor, -1);
        } else {
          set(res, a.device, tensor, false);
          if (a.kind == 2) bytes[a.device] -= tb.mass[tensor];
        }
      }
    }
  }
  for (int i = 0; i < T; ++i)
    if (!((ever[i >> 6] >> (i & 63)) & 1ull)) viol(4, -1, -1, -1, 0, i, -1);
  if (!WRITE) vcount[c] = nv;
}

// ---- replay: one thread per schedule; memory [n][D][T*T] optional
__global__ void replay_kernel(const xe_action* __restrict__ act, const int64_t* __restrict__ aoff, int64_t n, int D,
                              int T, int E, int NW, Tabs tb, double* __restrict__ total, double* __restrict__ eq1,
                              int64_t* __restrict__ mem, int64_t* __restrict__ peaks, uint64_t* __restrict__ scratch) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (c >= n) return;
  uint64_t* res = scratch + c * (2 * D) * NW;
  uint64_t* avail = res + D * NW;
  auto bit = [&](const uint64_t* m, int d, int i) { return (m[d * NW + (i >> 6)] >> (i & 63)) & 1ull; };
  auto set = [&](uint64_t* m, int d, int i, bool on) {
    if (on) m[d * NW + (i >> 6)] |= 1ull << (i & 63);
    else m[d * NW + (i >> 6)] &= ~(1ull << (i & 63));
  };
  const int64_t k0 = aoff[c], k1 = aoff[c + 1];
  // total action cost (action_cost, schedule.cpp:242-259), in list order;
  // a copy along no declared edge (a synthesized edge) makes it NaN here and
  // the host computes it from the link model
  double tot = 0.0;
  for (int64_t k = k0; k < k1; ++k) {
    const xe_action a = act[k];
    if (a.kind == 0) {
      tot += tb.cost[a.device * T + a.op];
    } else if (a.kind == 1) {
      int e = -1;
      for (int q = 0; q < E; ++q)
        if (tb.src[q] == a.src && tb.dst[q] == a.dst) {
          e = q;
          break;
        }
      tot += e < 0 ? NAN : (a.from == a.to ? 0.0 : tb.w[(e * D + a.from) * D + a.to]);
    }
  }
  total[c] = tot;
  // Eq. 1 from availability (schedule.cpp:283-323)
  for (int i = 0; i < D * NW; ++i) res[i] = 0;
  double obj = 0.0;
  int64_t k = k0;
  for (int t = 0; t < T; ++t) {
    const int64_t begin = k;
    while (k < k1 && act[k].timestep == t) ++k;
    for (int i = 0; i < D * NW; ++i) avail[i] = res[i];
    for (int64_t j = begin; j < k; ++j)
      if (act[j].kind == 0) set(avail, act[j].device, act[j].op, true);
    for (int64_t j = begin; j < k; ++j) {
      const xe_action a = act[j];
      if (a.kind != 0) continue;
      obj += tb.cost[a.device * T + a.op];
      if (tb.energy) obj += tb.alpha * tb.q[a.device * T + a.op];
      for (int q = tb.in_ptr[a.op]; q < tb.in_ptr[a.op + 1]; ++q) {
        const int e = tb.in_edge[q], u = tb.src[e];
        for (int ds = 0; ds < D; ++ds) {
          if (ds == a.device || !bit(avail, ds, u)) continue;
          obj += tb.w[(e * D + ds) * D + a.device];
        }
      }
    }
    for (int64_t j = begin; j < k; ++j) {
      const xe_action a = act[j];
      if (a.kind == 0) set(res, a.device, a.op, true);
      else if (a.kind == 2) set(res, a.device, a.src, false);
      else if (a.kind == 3) set(res, a.device, a.op, false);
    }
  }
  eq1[c] = obj;
  // memory series (schedule.cpp:325-367)
  for (int i = 0; i < D * NW; ++i) res[i] = 0;
  int64_t pk[8];
  for (int d = 0; d < D; ++d) pk[d] = 0;
  k = k0;
  for (int t = 0; t < T; ++t) {
    int64_t bytes[8];
    for (int d = 0; d < D; ++d) {
      bytes[d] = 0;
      for (int i = 0; i < T; ++i)
        if (bit(res, d, i)) bytes[d] += tb.mass[i];
    }
    const int64_t begin = k;
    while (k < k1 && act[k].timestep == t) ++k;
    for (int v = 0; v < T; ++v) {
      for (int64_t j = begin; j < k; ++j)
        if (act[j].kind == 0 && act[j].op == v) {
          set(res, act[j].device, v, true);
          bytes[act[j].device] += tb.mass[v];
        }
      for (int d = 0; d < D; ++d) {
        if (mem) mem[((c * D + d) * T + t) * T + v] = bytes[d];
        pk[d] = max(pk[d], bytes[d]);
      }
      for (int64_t j = begin; j < k; ++j)
        if (act[j].kind == 2 && act[j].dst == v) {
          set(res, act[j].device, act[j].src, false);
          bytes[act[j].device] -= tb.mass[act[j].src];
        }
    }
    for (int64_t j = begin; j < k; ++j)
      if (act[j].kind == 3) set(res, act[j].device, act[j].op, false);
  }
  for (int d = 0; d < D; ++d) peaks[c * D + d] = pk[d];
}

// a candidate whose decode raised has no schedule: zero all its counts
__global__ void zero_failed_kernel(int64_t* count, const int32_t* err, int64_t n, int T) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (c >= n) return;
  bool bad = false;
  for (int t = 0; t < T; ++t) bad |= err[(c * T + t) * 3] != 0;
  if (bad)
    for (int t = 0; t < T; ++t) count[c * T + t] = 0;
}

Tabs tabs_of(const xe_problem* pr, bool energy) {
  Tabs t{};
  t.mass = pr->d_mass.p;
  t.cost = pr->d_cost.p;
  t.w = pr->d_w.p;
  t.q = pr->d_q.p;
  t.alpha = pr->h.alpha;
  t.energy = energy && pr->h.has_energy ? 1 : 0;
  t.src = pr->d_src.p;
  t.dst = pr->d_dst.p;
  t.in_ptr = pr->d_in_ptr.p;
  t.in_edge = pr->d_in_edge.p;
  t.cons = pr->d_cons.p;
  return t;
}

struct BitsBuf {
  DevBuf<uint64_t> R, S, Z, F;
  Bits b{};
  void alloc(const HostProblem& h, int64_t n) {
    b.D = h.D;
    b.T = h.T;
    b.E = h.E;
    b.NW = (h.T + 63) / 64;
    b.NWF = (h.E + h.T + 63) / 64;
    const size_t rows = static_cast<size_t>(std::max<int64_t>(n, 1)) * h.D * h.T;
    R.alloc(rows * b.NW);
    S.alloc(rows * b.NW);
    Z.alloc(rows * b.NW);
    F.alloc(rows * b.NWF);
    b.R = R.p;
    b.S = S.p;
    b.Z = Z.p;
    b.F = F.p;
  }
};

inline unsigned blocks_for(int64_t n, int b = 128) { return static_cast<unsigned>(std::max<int64_t>(1, (n + b - 1) / b)); }

// Decodes n candidates whose bits are in bb; offsets [n+1] host, actions host or null
void decode_bits(const xe_problem* pr, BitsBuf& bb, int64_t n, int64_t* offsets, xe_action* actions,
                 xe_decode_error* errors, cudaStream_t s) {
  const HostProblem& h = pr->h;
  const Tabs tb = tabs_of(pr, false);
  const int64_t nk = n * h.T;
  DevBuf<int64_t> cnt, off;
  DevBuf<int32_t> err;
  cnt.alloc(static_cast<size_t>(std::max<int64_t>(1, nk)));
  off.alloc(static_cast<size_t>(nk + 1));
  err.alloc(static_cast<size_t>(std::max<int64_t>(1, nk)) * 3);
  if (nk > 0) {
    decode_kernel<false><<<blocks_for(nk), 128, 0, s>>>(bb.b, tb, n, nullptr, nullptr, cnt.p, err.p);
    zero_failed_kernel<<<blocks_for(n), 128, 0, s>>>(cnt.p, err.p, n, h.T);
  }
  XE_CUDA(cudaGetLastError());
  XE_CUDA(cudaMemsetAsync(off.p, 0, 8, s));
  if (nk > 0) thrust::inclusive_scan(thrust::cuda::par.on(s), cnt.p, cnt.p + nk, off.p + 1);
  std::vector<int64_t> hoff(static_cast<size_t>(nk + 1));
  std::vector<int32_t> herr(static_cast<size_t>(nk) * 3);
  XE_CUDA(cudaMemcpyAsync(hoff.data(), off.p, (nk + 1) * 8, cudaMemcpyDeviceToHost, s));
  if (nk) XE_CUDA(cudaMemcpyAsync(herr.data(), err.p, nk * 12, cudaMemcpyDeviceToHost, s));
  XE_CUDA(cudaStreamSynchronize(s));
  for (int64_t c = 0; c <= n; ++c) offsets[c] = hoff[static_cast<size_t>(c * h.T)];
  // the first error in the reference's order: lowest t (within t, the kernel stopped at the first)
  for (int64_t c = 0; c < n; ++c) {
    xe_decode_error e{0, -1, -1, -1};
    for (int t = 0; t < h.T; ++t) {
      const int32_t* q = &herr[static_cast<size_t>((c * h.T + t) * 3)];
      if (q[0]) {
        e = {q[0], t, q[1], q[2]};
        break;
      }
    }
    if (errors) errors[c] = e;
  }
  if (!actions || offsets[n] == 0) return;
  DevBuf<xe_action> out;
  out.alloc(static_cast<size_t>(offsets[n]));
  decode_kernel<true><<<blocks_for(nk), 128, 0, s>>>(bb.b, tb, n, off.p, out.p, nullptr, nullptr);
  XE_CUDA(cudaGetLastError());
  XE_CUDA(cudaMemcpyAsync(actions, out.p, offsets[n] * sizeof(xe_action), cudaMemcpyDeviceToHost, s));
  XE_CUDA(cudaStreamSynchronize(s));
}

}  // namespace sch
}  // namespace xe

using namespace xe;

extern "C" int xe_decode_cubes(const xe_problem* p, const xe_model_opts* opts, const uint32_t* cubes, int64_t n,
                               int64_t* offsets, xe_action* actions, xe_decode_error* errors) {
  return guard([&] {
    if (!p || !offsets || (!cubes && n > 0) || n < 0) fail(XE_ERR_ARG, "null argument");
    require_uploaded(p);
    if (p->h.D > 8 || p->h.T > 256) fail(XE_ERR_TOO_LARGE, "decode: D <= 8 and T <= 256");
    const HostProblem& h = p->h;
    cudaStream_t s = p->stream;
    const size_t cw = xe_cube_bytes(h.D, h.T) / 4;
    DevBuf<uint32_t> dc;
    dc.alloc(static_cast<size_t>(std::max<int64_t>(1, n)) * cw);
    if (n) XE_CUDA(cudaMemcpyAsync(dc.p, cubes, n * cw * 4, cudaMemcpyHostToDevice, s));
    sch::BitsBuf bb;
    bb.alloc(h, n);
    const int strict = opts && opts->strict_free ? 1 : 0;
    if (n) sch::bits_from_cubes_kernel<<<sch::blocks_for(n * h.D * h.T), 128, 0, s>>>(dc.p, n, bb.b,
                                                                                    sch::tabs_of(p, false), strict);
    XE_CUDA(cudaGetLastError());
    sch::decode_bits(p, bb, n, offsets, actions, errors, s);
  });
}

extern "C" int xe_decode_dense(const xe_problem* p, const double* x, int64_t* n_actions, xe_action* actions,
                               xe_decode_error* error) {
  return guard([&] {
    if (!p || !x || !n_actions) fail(XE_ERR_ARG, "null argument");
    require_uploaded(p);
    if (p->h.D > 8 || p->h.T > 256) fail(XE_ERR_TOO_LARGE, "decode: D <= 8 and T <= 256");
    const HostProblem& h = p->h;
    cudaStream_t s = p->stream;
    const int64_t ncols = xe_model_cols(h.D, h.T, h.E);
    DevBuf<double> dx;
    dx.alloc(static_cast<size_t>(ncols));
    XE_CUDA(cudaMemcpyAsync(dx.p, x, ncols * 8, cudaMemcpyHostToDevice, s));
    sch::BitsBuf bb;
    bb.alloc(h, 1);
    sch::bits_from_dense_kernel<<<sch::blocks_for(static_cast<int64_t>(h.D) * h.T), 128, 0, s>>>(dx.p, bb.b);
    XE_CUDA(cudaGetLastError());
    int64_t off[2];
    sch::decode_bits(p, bb, 1, off, actions, error, s);
    *n_actions = off[1];
  });
}

extern "C" int xe_validate_schedules(const xe_problem* p, const xe_action* actions, const int64_t* offsets, int64_t n,
                                     const int64_t* budgets, int64_t* v_offsets, xe_violation* violations) {
  return guard([&] {
    if (!p || !offsets || !v_offsets || n < 0) fail(XE_ERR_ARG, "null argument");
    require_uploaded(p);
    const HostProblem& h = p->h;
    if (h.D > 8) fail(XE_ERR_TOO_LARGE, "validate: D <= 8");
    cudaStream_t s = p->stream;
    const int NW = (h.T + 63) / 64;
    const int64_t na = offsets[n] - offsets[0];
    DevBuf<xe_action> da;
    DevBuf<int64_t> doff, dcnt, dvoff, dbud;
    da.alloc(static_cast<size_t>(std::max<int64_t>(1, na)));
    if (na) XE_CUDA(cudaMemcpyAsync(da.p, actions + offsets[0], na * sizeof(xe_action), cudaMemcpyHostToDevice, s));
    std::vector<int64_t> rel(static_cast<size_t>(n + 1));
    for (int64_t c = 0; c <= n; ++c) rel[static_cast<size_t>(c)] = offsets[c] - offsets[0];
    doff.upload(rel, s);
    std::vector<int64_t> bud(h.budget);
    if (budgets) bud.assign(budgets, budgets + h.D);
    dbud.upload(bud, s);
    DevBuf<uint64_t> scratch;
    scratch.alloc(static_cast<size_t>(std::max<int64_t>(1, n)) * (2 * h.D + 1) * NW);
    dcnt.alloc(static_cast<size_t>(std::max<int64_t>(1, n)));
    const sch::Tabs tb = sch::tabs_of(p, false);
    if (n) sch::validate_kernel<false><<<sch::blocks_for(n, 64), 64, 0, s>>>(da.p, doff.p, n, h.D, h.T, NW, tb, dbud.p,
                                                                            nullptr, nullptr, dcnt.p, scratch.p);
    XE_CUDA(cudaGetLastError());
    std::vector<int64_t> cnt(static_cast<size_t>(std::max<int64_t>(1, n)));
    if (n) XE_CUDA(cudaMemcpyAsync(cnt.data(), dcnt.p, n * 8, cudaMemcpyDeviceToHost, s));
    XE_CUDA(cudaStreamSynchronize(s));
    v_offsets[0] = 0;
    for (int64_t c = 0; c < n; ++c) v_offsets[c + 1] = v_offsets[c] + cnt[static_cast<size_t>(c)];
    if (!violations || v_offsets[n] == 0) return;
    dvoff.upload(std::vector<int64_t>(v_offsets, v_offsets + n + 1), s);
    DevBuf<xe_violation> dv;
    dv.alloc(static_cast<size_t>(v_offsets[n]));
    sch::validate_kernel<true><<<sch::blocks_for(n, 64), 64, 0, s>>>(da.p, doff.p, n, h.D, h.T, NW, tb, dbud.p,
                                                                    dvoff.p, dv.p, nullptr, scratch.p);
    XE_CUDA(cudaGetLastError());
    XE_CUDA(cudaMemcpyAsync(violations, dv.p, v_offsets[n] * sizeof(xe_violation), cudaMemcpyDeviceToHost, s));
    XE_CUDA(cudaStreamSynchronize(s));
  });
}

extern "C" int xe_replay_schedules(const xe_problem* p, const xe_model_opts* opts, const xe_action* actions,
                                   const int64_t* offsets, int64_t n, double* total_ms, double* eq1, int64_t* memory,
                                   int64_t* peaks) {
  return guard([&] {
    if (!p || !offsets || !total_ms || !eq1 || !peaks || n < 0) fail(XE_ERR_ARG, "null argument");
    require_uploaded(p);
    const HostProblem& h = p->h;
    if (h.D > 8) fail(XE_ERR_TOO_LARGE, "replay: D <= 8");
    if (!h.missing_link.empty() && h.D > 1) fail(XE_ERR_MISSING_LINK, h.missing_link);
    cudaStream_t s = p->stream;
    const int NW = (h.T + 63) / 64;
    const int64_t na = offsets[n] - offsets[0];
    DevBuf<xe_action> da;
    DevBuf<int64_t> doff, dmem, dpk;
    DevBuf<double> dtot, deq;
    da.alloc(static_cast<size_t>(std::max<int64_t>(1, na)));
    if (na) XE_CUDA(cudaMemcpyAsync(da.p, actions + offsets[0], na * sizeof(xe_action), cudaMemcpyHostToDevice, s));
    std::vector<int64_t> rel(static_cast<size_t>(n + 1));
    for (int64_t c = 0; c <= n; ++c) rel[static_cast<size_t>(c)] = offsets[c] - offsets[0];
    doff.upload(rel, s);
    const size_t nn = static_cast<size_t>(std::max<int64_t>(1, n));
    dtot.alloc(nn);
    deq.alloc(nn);
    dpk.alloc(nn * h.D);
    if (memory) dmem.alloc(nn * h.D * h.T * h.T);
    DevBuf<uint64_t> scratch;
    scratch.alloc(nn * 2 * h.D * NW);
    const sch::Tabs tb = sch::tabs_of(p, opts && opts->use_energy);
    if (n) sch::replay_kernel<<<sch::blocks_for(n, 64), 64, 0, s>>>(da.p, doff.p, n, h.D, h.T, h.E, NW, tb, dtot.p,
                                                                   deq.p, memory ? dmem.p : nullptr, dpk.p, scratch.p);
    XE_CUDA(cudaGetLastError());
    if (n) {
      XE_CUDA(cudaMemcpyAsync(total_ms, dtot.p, n * 8, cudaMemcpyDeviceToHost, s));
      XE_CUDA(cudaMemcpyAsync(eq1, deq.p, n * 8, cudaMemcpyDeviceToHost, s));
      XE_CUDA(cudaMemcpyAsync(peaks, dpk.p, n * h.D * 8, cudaMemcpyDeviceToHost, s));
      if (memory)
        XE_CUDA(cudaMemcpyAsync(memory, dmem.p, static_cast<size_t>(n) * h.D * h.T * h.T * 8, cudaMemcpyDeviceToHost, s));
    }
    XE_CUDA(cudaStreamSynchronize(s));
  });
}
