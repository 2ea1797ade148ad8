// SPDX-License-Identifier: Apache-2.0
//
// Single-assignment kernels behind the map-based C++ API (include/xengine/
// model.hpp), over the dense closed-form column vector x[n_cols]
// (column order = VarRef order, csr.cu):
//
//   complete_kernel   complete_assignment (proj/src/model.cpp:471-549): from
//                     one canonical (R,S) cube, Z = R|S, the F hazards, the
//                     U recurrence and the P products; one thread per (d,t)
//                     row for R/S/Z/F/U, one per (t,e,ds,dc) for P.
//   objective_kernel  objective_value (model.cpp:369-428) of an arbitrary
//                     (possibly fractional) x: the reference's sum is one
//                     sequential fp64 chain, so one lane walks it in the
//                     reference's loop order (built with -fmad=false).
//   rows_kernel       the row part of check_assignment (model.cpp:449-467):
//                     one thread per row, terms in emission order, scaled
//                     tolerance; writes the violation amount of failing rows.
//
// The batched evaluators (eval_il.cu, eval_cube*.cu) are the throughput
// path; these serve the one-assignment-at-a-time reference API.

#include <cmath>
#include <cstring>

#include "csr.hpp"

namespace xe {
namespace cmp {

struct Cols {  // closed-form column offsets (model.hpp:14-31)
  int64_t D, T, E, FE;
  __host__ __device__ int64_t r(int64_t d, int64_t t, int64_t i) const { return (d * T + t) * T + i; }
  __host__ __device__ int64_t s(int64_t d, int64_t t, int64_t i) const { return D * T * T + r(d, t, i); }
  __host__ __device__ int64_t z(int64_t d, int64_t t, int64_t i) const { return 2 * D * T * T + r(d, t, i); }
  __host__ __device__ int64_t f(int64_t d, int64_t t, int64_t eo) const { return 3 * D * T * T + (d * T + t) * FE + eo; }
  __host__ __device__ int64_t u(int64_t d, int64_t t, int64_t i) const { return 3 * D * T * T + D * T * FE + r(d, t, i); }
  __host__ __device__ int64_t p(int64_t t, int64_t e, int64_t ds, int64_t dc) const {
    return 4 * D * T * T + D * T * FE + ((t * E + e) * D + ds) * (D - 1) + (dc - (dc > ds ? 1 : 0));
  }
  __host__ __device__ int64_t n() const { return 4 * D * T * T + D * T * FE + T * E * D * (D - 1); }
};

struct CubeView {  // one canonical cube: [which][d][t][W32] u32
  const uint32_t* w;
  int D, T, W32;
  __device__ bool bit(int which, int d, int t, int i) const {
    return (w[((static_cast<int64_t>(which) * D + d) * T + t) * W32 + (i >> 5)] >> (i & 31)) & 1u;
  }
};

__global__ void complete_rows_kernel(CubeView c, Cols C, const int32_t* src, const int32_t* dst,
                                     const int32_t* in_ptr, const int32_t* in_edge, const int32_t* out_ptr,
                                     const int32_t* out_edge, const int64_t* mass, int strict, double* x) {
  const int64_t row = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int D = c.D, T = c.T, E = static_cast<int>(C.E);
  if (row >= static_cast<int64_t>(D) * T) return;
  const int d = static_cast<int>(row / T), t = static_cast<int>(row % T);
  auto R = [&](int dd, int i) { return c.bit(0, dd, t, i); };
  auto S = [&](int i) { return c.bit(1, d, t, i); };
  auto Sn = [&](int i) { return t + 1 < T && c.bit(1, d, t + 1, i); };
  auto Z = [&](int i) { return R(d, i) || S(i); };
  for (int i = 0; i < T; ++i) {
    const bool r = R(d, i), s = S(i);
    x[C.r(d, t, i)] = r;
    x[C.s(d, t, i)] = s;
    x[C.z(d, t, i)] = r || s;
  }
  // F(u->v): computed v, resident u, not kept for t+1, no later consumer of u
  // computed this timestep (on d; on any device under strict_free)
  auto later_blocked = [&](int u, int v) {
    for (int k = out_ptr[u]; k < out_ptr[u + 1]; ++k) {
      const int w = dst[out_edge[k]];
      if (w <= v) continue;
      if (strict) {
        for (int dd = 0; dd < D; ++dd)
          if (R(dd, w)) return true;
      } else if (R(d, w)) {
        return true;
      }
    }
    return false;
  };
  auto fval = [&](int u, int v) { return R(d, v) && Z(u) && !Sn(u) && !later_blocked(u, v); };
  for (int e = 0; e < E; ++e) x[C.f(d, t, e)] = fval(src[e], dst[e]);
  for (int v = 0; v < T; ++v) x[C.f(d, t, E + v)] = fval(v, v);
  // U recurrence (integer-valued, exact in int64 and in double < 2^53)
  int64_t cur = 0;
  for (int i = 0; i < T; ++i)
    if (S(i)) cur += mass[i];
  if (R(d, 0)) cur += mass[0];
  x[C.u(d, t, 0)] = static_cast<double>(cur);
  for (int v = 0; v + 1 < T; ++v) {
    int64_t freed = 0;
    for (int k = in_ptr[v]; k < in_ptr[v + 1]; ++k) {
      const int e = in_edge[k];
      if (x[C.f(d, t, e)] != 0.0) freed += mass[src[e]];
    }
    if (x[C.f(d, t, E + v)] != 0.0) freed += mass[v];
    cur = cur - freed + (R(d, v + 1) ? mass[v + 1] : 0);
    x[C.u(d, t, v + 1)] = static_cast<double>(cur);
  }
}

__global__ void complete_p_kernel(CubeView c, Cols C, const int32_t* src, const int32_t* dst, double* x) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int D = c.D;
  const int64_t n = C.T * C.E * D * D;
  if (k >= n) return;
  const int dc = static_cast<int>(k % D), ds = static_cast<int>(k / D % D);
  const int64_t te = k / (static_cast<int64_t>(D) * D);
  const int e = static_cast<int>(te % C.E), t = static_cast<int>(te / C.E);
  if (ds == dc) return;
  const bool z = c.bit(0, ds, t, src[e]) || c.bit(1, ds, t, src[e]);
  x[C.p(t, e, ds, dc)] = (c.bit(0, dc, t, dst[e]) && z) ? 1.0 : 0.0;
}

// objective_value's three loops, one lane, reference order (model.cpp:392-427)
__global__ void objective_kernel(const double* x, Cols C, const double* cost, const double* w,
                                 const int32_t* src, const int32_t* dst, int energy, double alpha,
                                 const double* q, double* out) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const int64_t D = C.D, T = C.T, E = C.E;
  double total = 0.0;
  for (int64_t d = 0; d < D; ++d)
    for (int64_t t = 0; t < T; ++t)
      for (int64_t i = 0; i < T; ++i) {
        const double r = x[C.r(d, t, i)];
        if (r != 0.0) total = __dadd_rn(total, __dmul_rn(cost[d * T + i], r));
      }
  for (int64_t t = 0; t < T; ++t)
    for (int64_t e = 0; e < E; ++e)
      for (int64_t dc = 0; dc < D; ++dc) {
        const double r = x[C.r(dc, t, dst[e])];
        if (r == 0.0) continue;
        for (int64_t ds = 0; ds < D; ++ds) {
          if (ds == dc) continue;
          const double z = x[C.z(ds, t, src[e])];
          if (z != 0.0) total = __dadd_rn(total, __dmul_rn(__dmul_rn(w[(e * D + ds) * D + dc], r), z));
        }
      }
  if (energy)
    for (int64_t d = 0; d < D; ++d)
      for (int64_t t = 0; t < T; ++t)
        for (int64_t i = 0; i < T; ++i) {
          const double r = x[C.r(d, t, i)];
          if (r != 0.0) total = __dadd_rn(total, __dmul_rn(__dmul_rn(alpha, q[d * T + i]), r));
        }
  *out = total;
}

__global__ void rows_kernel(const int64_t* rp, const int32_t* col, const double* val, const double* rhs,
                            const int8_t* sense, int64_t m, const double* x, double tol, double* viol,
                            unsigned long long* count) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= m) return;
  double lhs = 0.0, scale = fmax(1.0, fabs(rhs[r]));
  for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
    const double term = __dmul_rn(val[k], x[col[k]]);
    lhs = __dadd_rn(lhs, term);
    scale = fmax(scale, fabs(term));
  }
  double v = 0.0;
  switch (sense[r]) {
    case 'L': v = __dsub_rn(lhs, rhs[r]); break;
    case 'G': v = __dsub_rn(rhs[r], lhs); break;
    default: v = fabs(__dsub_rn(lhs, rhs[r])); break;
  }
  const bool bad = v > __dmul_rn(tol, scale);
  viol[r] = bad ? v : 0.0;
  if (bad) atomicAdd(count, 1ull);
}

inline unsigned blocks(int64_t n, int b = 256) { return static_cast<unsigned>((n + b - 1) / b); }

}  // namespace cmp

using namespace cmp;

namespace {
Cols cols_of(const HostProblem& h) { return Cols{h.D, h.T, h.E, h.E + h.T}; }
}  // namespace

int64_t model_cols(int D, int T, int E) { return Cols{D, T, E, E + T}.n(); }

void complete_cube_host(const xe_problem* pr, const xe_model_opts& o, const uint32_t* cube_host, double* x_host) {
  const HostProblem& h = pr->h;
  const Cols C = cols_of(h);
  const int W32 = (h.T + 31) / 32;
  const size_t cw = static_cast<size_t>(2) * h.D * h.T * W32;
  cudaStream_t s = pr->stream;
  // out-edges of each op in edge order (later-consumer scan)
  std::vector<int32_t> optr(static_cast<size_t>(h.T) + 1, 0), oedge(static_cast<size_t>(h.E));
  for (int e = 0; e < h.E; ++e) optr[static_cast<size_t>(h.src[static_cast<size_t>(e)]) + 1]++;
  for (int v = 0; v < h.T; ++v) optr[static_cast<size_t>(v) + 1] += optr[static_cast<size_t>(v)];
  {
    std::vector<int32_t> fill(optr.begin(), optr.end() - 1);
    for (int e = 0; e < h.E; ++e) oedge[static_cast<size_t>(fill[static_cast<size_t>(h.src[static_cast<size_t>(e)])]++)] = e;
  }
  DevBuf<uint32_t> dcube;
  DevBuf<double> dx;
  DevBuf<int32_t> dop, doe;
  dcube.alloc(cw);
  dx.alloc(static_cast<size_t>(C.n()));
  dop.upload(optr, s);
  doe.upload(oedge, s);
  XE_CUDA(cudaMemcpyAsync(dcube.p, cube_host, cw * 4, cudaMemcpyHostToDevice, s));
  XE_CUDA(cudaMemsetAsync(dx.p, 0, static_cast<size_t>(C.n()) * 8, s));
  CubeView cv{dcube.p, h.D, h.T, W32};
  const DevProblem& P = pr->dev;
  complete_rows_kernel<<<blocks(static_cast<int64_t>(h.D) * h.T, 128), 128, 0, s>>>(
      cv, C, P.src, P.dst, P.in_ptr, P.in_edge, dop.p, doe.p, P.mass, o.strict_free ? 1 : 0, dx.p);
  XE_CUDA(cudaGetLastError());
  if (h.E > 0 && h.D > 1) {
    complete_p_kernel<<<blocks(static_cast<int64_t>(h.T) * h.E * h.D * h.D), 256, 0, s>>>(cv, C, P.src, P.dst, dx.p);
    XE_CUDA(cudaGetLastError());
  }
  XE_CUDA(cudaMemcpyAsync(x_host, dx.p, static_cast<size_t>(C.n()) * 8, cudaMemcpyDeviceToHost, s));
  XE_CUDA(cudaStreamSynchronize(s));
}

double objective_dense_host(const xe_problem* pr, const xe_model_opts& o, const double* x_host) {
  const HostProblem& h = pr->h;
  const Cols C = cols_of(h);
  // objective_value prices a copy only when it is charged, R(dc,t,dst) != 0
  // and Z(ds,t,src) != 0, and copy_cost raises MissingLink there
  // (model.cpp:399-411, problem.cpp:374-376): the same lazy check, in the
  // reference's loop order so the first charged uncovered pair is named
  if (!h.missing_link.empty() && h.D > 1 && !h.w_missing.empty()) {
    for (int64_t t = 0; t < h.T; ++t)
      for (int64_t e = 0; e < h.E; ++e)
        for (int64_t dc = 0; dc < h.D; ++dc) {
          if (x_host[C.r(dc, t, h.dst[static_cast<size_t>(e)])] == 0.0) continue;
          for (int64_t ds = 0; ds < h.D; ++ds) {
            if (ds == dc || x_host[C.z(ds, t, h.src[static_cast<size_t>(e)])] == 0.0) continue;
            if (h.w_missing[static_cast<size_t>((e * h.D + ds) * h.D + dc)])
              fail(XE_ERR_MISSING_LINK, "no link covers " + h.device_ids[static_cast<size_t>(ds)] + "->" +
                                            h.device_ids[static_cast<size_t>(dc)]);
          }
        }
  }
  cudaStream_t s = pr->stream;
  DevBuf<double> dx, dout;
  dx.alloc(static_cast<size_t>(C.n()));
  dout.alloc(1);
  XE_CUDA(cudaMemcpyAsync(dx.p, x_host, static_cast<size_t>(C.n()) * 8, cudaMemcpyHostToDevice, s));
  const bool energy = o.use_energy && h.has_energy;
  objective_kernel<<<1, 32, 0, s>>>(dx.p, C, pr->d_cost.p, pr->d_w.p, pr->dev.src, pr->dev.dst, energy ? 1 : 0,
                                    h.alpha, pr->d_q.p, dout.p);
  XE_CUDA(cudaGetLastError());
  double v = 0.0;
  XE_CUDA(cudaMemcpyAsync(&v, dout.p, 8, cudaMemcpyDeviceToHost, s));
  XE_CUDA(cudaStreamSynchronize(s));
  return v;
}

int64_t check_rows_host(xe_csr* m, const double* x_host, double tol, double* viol_host) {
  const xe_csr_info& in = m->info;
  cudaStream_t s = m->stream;
  DevBuf<double> dx, dv;
  DevBuf<unsigned long long> dc;
  dx.alloc(static_cast<size_t>(in.n_cols));
  dv.alloc(static_cast<size_t>(std::max<int64_t>(1, in.n_rows)));
  dc.alloc(1);
  XE_CUDA(cudaMemcpyAsync(dx.p, x_host, static_cast<size_t>(in.n_cols) * 8, cudaMemcpyHostToDevice, s));
  XE_CUDA(cudaMemsetAsync(dc.p, 0, 8, s));
  if (in.n_rows > 0) {
    rows_kernel<<<blocks(in.n_rows), 256, 0, s>>>(m->row_ptr.p, m->col.p, m->val.p, m->rhs.p, m->sense.p, in.n_rows,
                                                  dx.p, tol, dv.p, dc.p);
    XE_CUDA(cudaGetLastError());
  }
  unsigned long long cnt = 0;
  XE_CUDA(cudaMemcpyAsync(&cnt, dc.p, 8, cudaMemcpyDeviceToHost, s));
  if (viol_host && in.n_rows > 0)
    XE_CUDA(cudaMemcpyAsync(viol_host, dv.p, static_cast<size_t>(in.n_rows) * 8, cudaMemcpyDeviceToHost, s));
  XE_CUDA(cudaStreamSynchronize(s));
  return static_cast<int64_t>(cnt);
}

}  // namespace xe
