// SPDX-License-Identifier: Apache-2.0
//
// K3 — first-order LP relaxation (PDHG, PDLP-style) of the K1 model.
//
// The reference has no LP solver: its relaxation is reachable only through
// MPS -> an external MILP solver (proj/src/solver.cpp:501-561,
// proj/tools/mps_solve.py).  This solves the same model with every binary
// relaxed to [0,1] (BV -> [0,1], FX -> 0, U in [0,b_d], P in [0,1]) and is
// judged against HiGHS on the reference's MPS (tests/golden/lp_values.json).
//
//   min c'x  s.t.  K x in [l, u] (L: (-inf,b], G: [b,inf), E: [b,b]),  0 <= x <= ub
//
// Saddle point  c'x - y'(Kx - b)  with y >= 0 on G rows, y <= 0 on L rows.
// Iteration (tau = eta/omega, sigma = eta*omega):
//   x+ = clip(x - tau (c - K'y), lb, ub)           one thread per column, CSC
//   y+ = proj(y + sigma (b - K (2x+ - x)))          one thread per row, CSR
// Preconditioning: rows normalised to unit inf-norm, then 10 Ruiz passes
// (inf-norm) + Pock-Chambolle (alpha = 1); columns with the prohibitive cost
// (>= 1e9) fixed at 0 and certified afterwards by their reduced costs; step
// 0.95/||K||_2 (power iteration); adaptive restarts to the current or average
// iterate on the normalised KKT error, primal-weight updates at restarts
// (PDLP's rules); blocks of `check_every` iterations replayed from a captured
// CUDA graph (a cooperative single-kernel variant with two grid barriers per
// iteration measured 2x slower on B200: 37.5 vs 17.9 us/iter at VGG-16).
// FP64 throughout.

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "csr.hpp"

namespace xe {
namespace pd {

constexpr int kB = 256;

inline int grid(int64_t n) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + kB - 1) / kB, 148LL * 32)));
}

#define GRID_LOOP(i, n) \
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < (n); i += static_cast<int64_t>(gridDim.x) * blockDim.x)

__global__ void col_of_kernel(const int64_t* col_ptr, int64_t n, int32_t* col_of) {
  GRID_LOOP(j, n)
  for (int64_t q = col_ptr[j]; q < col_ptr[j + 1]; ++q) col_of[q] = static_cast<int32_t>(j);
}

// norm of each row of Dr*K*Dc: inf-norm (p=0) or l1 (p=1)
__global__ void row_norm_kernel(const int64_t* rp, const int32_t* col, const double* val, const double* Dr,
                                const double* Dc, int64_t m, int p, double* out) {
  GRID_LOOP(i, m) {
    double s = 0.0;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
      const double a = fabs(val[k] * Dc[col[k]]);
      s = p ? s + a : fmax(s, a);
    }
    out[i] = s * Dr[i];
  }
}

__global__ void col_norm_kernel(const int64_t* cp, const int32_t* row, const double* val, const double* Dr,
                                const double* Dc, int64_t n, int p, double* out) {
  GRID_LOOP(j, n) {
    double s = 0.0;
    for (int64_t q = cp[j]; q < cp[j + 1]; ++q) {
      const double a = fabs(val[q] * Dr[row[q]]);
      s = p ? s + a : fmax(s, a);
    }
    out[j] = s * Dc[j];
  }
}

// 1 / inf-norm of each row of K (1 for empty rows): the rows are normalised
// before Ruiz, so the equilibration starts from unit-scale rows whatever the
// units (bytes in EQ13/EQ14, h_max in EQ16, q in the energy rows)
__global__ void row_inf_kernel(const int64_t* rp, const double* val, int64_t m, double* out) {
  GRID_LOOP(i, m) {
    double s = 0.0;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) s = fmax(s, fabs(val[k]));
    out[i] = s > 0.0 ? 1.0 / s : 1.0;
  }
}

// Presolve of the prohibitive-cost columns (cost >= 1e9, lower bound 0):
// fixed at 0 with zero cost in the solved problem.
__global__ void sentinel_kernel(const double* c, const double* lb, const double* ub, int64_t n, double* c_out,
                                double* ub_out, unsigned long long* count) {
  GRID_LOOP(j, n) {
    const bool fix = c[j] >= 1.0e9 && lb[j] <= 0.0;
    c_out[j] = fix ? 0.0 : c[j];
    ub_out[j] = fix ? 0.0 : ub[j];
    if (fix) atomicAdd(count, 1ull);
  }
}

// Certificate for the presolve: reduced cost of every fixed column under the
// final duals, c_j - (K'y)_j with (K'y)_j = (K~'y~)_j / Dc_j, must be >= 0.
__global__ void certify_kernel(const double* c, const double* lb, const double* Kty_s, const double* Dc, int64_t n,
                               unsigned long long* bad) {
  GRID_LOOP(j, n) {
    if (c[j] >= 1.0e9 && lb[j] <= 0.0 && c[j] - Kty_s[j] / Dc[j] < 0.0) atomicAdd(bad, 1ull);
  }
}

__global__ void rescale_kernel(double* D, const double* nrm, int64_t n) {
  GRID_LOOP(i, n) {
    const double v = nrm[i];
    if (v > 0.0) D[i] /= sqrt(v);
  }
}

__global__ void scale_csr_kernel(const int64_t* rp, const int32_t* col, const double* val, const double* Dr,
                                 const double* Dc, int64_t m, double* out) {
  GRID_LOOP(i, m)
  for (int64_t k = rp[i]; k < rp[i + 1]; ++k) out[k] = val[k] * Dr[i] * Dc[col[k]];
}

__global__ void scale_csc_kernel(const int64_t* cp, const int32_t* row, const double* val, const double* Dr,
                                 const double* Dc, int64_t n, double* out) {
  GRID_LOOP(j, n)
  for (int64_t q = cp[j]; q < cp[j + 1]; ++q) out[q] = val[q] * Dr[row[q]] * Dc[j];
}

// scaled problem vectors
__global__ void scale_vec_kernel(const double* c, const double* lb, const double* ub, const double* Dc, int64_t n,
                                 double* cs, double* lbs, double* ubs) {
  GRID_LOOP(j, n) {
    cs[j] = c[j] * Dc[j];
    lbs[j] = lb[j] / Dc[j];
    ubs[j] = ub[j] / Dc[j];
  }
}
__global__ void scale_b_kernel(const double* b, const double* Dr, int64_t m, double* bs) {
  GRID_LOOP(i, m) bs[i] = b[i] * Dr[i];
}

// y = K x  (CSR, thread per row)
__global__ void spmv_kernel(const int64_t* rp, const int32_t* col, const double* val, const double* x, int64_t m,
                            double* y) {
  GRID_LOOP(i, m) {
    double s = 0.0;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) s += val[k] * x[col[k]];
    y[i] = s;
  }
}
// x = K' y  (CSC, thread per column)
__global__ void spmtv_kernel(const int64_t* cp, const int32_t* row, const double* val, const double* y, int64_t n,
                             double* x) {
  GRID_LOOP(j, n) {
    double s = 0.0;
    for (int64_t q = cp[j]; q < cp[j + 1]; ++q) s += val[q] * y[row[q]];
    x[j] = s;
  }
}

struct Iter {
  const int64_t *rp, *cp;
  const int32_t *col, *row;
  const double *val, *cval;
  const double *c, *lb, *ub, *b;
  const int8_t* sense;
  double *x, *xbar, *xsum, *y, *ysum;
  const double* step;  // device [tau, sigma]
  int64_t m, n;
};

// primal step: x+ = clip(x - tau (c - K'y)); xbar = 2x+ - x; running sum
// dual step:   y+ = proj(y + sigma (b - K xbar)); running sum
// Both half-steps run with G lanes per column / row (G a power of two
// <= 32): each lane takes every G-th nonzero, a G-wide shuffle reduction
// combines them, and lane 0 of the group applies the update.  Thread per row
// walks ~5 nonzeros as a chain of dependent loads (offsets -> index ->
// vector), which leaves the small relaxations latency-bound; G lanes cut the
// chain to one nonzero each and coalesce the index/value loads.
template <int G>
__device__ __forceinline__ double group_sum(double v, unsigned mask) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o, G);
  return v;
}

template <int G>
__global__ void primal_group_kernel(Iter it) {
  const double tau = it.step[0];
  const int gl = threadIdx.x & (G - 1);
  const unsigned mask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << ((threadIdx.x & 31) & ~(G - 1));
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x / G;
  for (int64_t j = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / G; j < it.n; j += stride) {
    double acc = 0.0;
    for (int64_t q = it.cp[j] + gl; q < it.cp[j + 1]; q += G) acc += it.cval[q] * it.y[it.row[q]];
    acc = group_sum<G>(acc, mask);
    if (gl == 0) {
      const double g = it.c[j] - acc;
      const double x0 = it.x[j];
      const double xn = fmin(fmax(x0 - tau * g, it.lb[j]), it.ub[j]);
      it.xbar[j] = 2.0 * xn - x0;
      it.x[j] = xn;
      it.xsum[j] += xn;
    }
  }
}

template <int G>
__global__ void dual_group_kernel(Iter it) {
  const double sigma = it.step[1];
  const int gl = threadIdx.x & (G - 1);
  const unsigned mask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << ((threadIdx.x & 31) & ~(G - 1));
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x / G;
  for (int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / G; i < it.m; i += stride) {
    double acc = 0.0;
    for (int64_t q = it.rp[i] + gl; q < it.rp[i + 1]; q += G) acc += it.val[q] * it.xbar[it.col[q]];
    acc = group_sum<G>(acc, mask);
    if (gl == 0) {
      double yn = it.y[i] + sigma * (it.b[i] - acc);
      const int8_t sn = it.sense[i];
      if (sn == 'G') yn = fmax(yn, 0.0);
      else if (sn == 'L') yn = fmin(yn, 0.0);
      it.y[i] = yn;
      it.ysum[i] += yn;
    }
  }
}

// group width for an average of `avg` nonzeros per vector
inline int group_width(double avg) {
  int g = 1;
  while (g < 32 && g < avg) g <<= 1;
  return std::max(2, g);
}

template <int G>
void launch_half_steps(const Iter& it, int64_t m, int64_t n, cudaStream_t s, bool primal) {
  const int64_t len = primal ? n : m;
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((len * G + kB - 1) / kB, 148LL * 16)));
  if (primal) primal_group_kernel<G><<<blocks, kB, 0, s>>>(it);
  else dual_group_kernel<G><<<blocks, kB, 0, s>>>(it);
}

void launch_half_step(const Iter& it, int64_t m, int64_t n, int g, cudaStream_t s, bool primal) {
  switch (g) {
    case 2: return launch_half_steps<2>(it, m, n, s, primal);
    case 4: return launch_half_steps<4>(it, m, n, s, primal);
    case 8: return launch_half_steps<8>(it, m, n, s, primal);
    case 16: return launch_half_steps<16>(it, m, n, s, primal);
    default: return launch_half_steps<32>(it, m, n, s, primal);
  }
}

// partial sums for the KKT measures, 8 doubles per block:
// [primal obj, primal viol^2 (unscaled), dual row obj, dual bound obj, |b|^2, |c|^2, -, -]
__global__ void kkt_rows_kernel(const double* Kx, const double* b, const int8_t* sense, const double* y,
                                const double* Dr, const double* Dr0, int64_t m, double* part) {
  __shared__ double sh[2][kB];
  double v2 = 0.0, dobj = 0.0;
  GRID_LOOP(i, m) {
    const double r = Kx[i] - b[i];
    double viol = 0.0;
    const int8_t sn = sense[i];
    if (sn == 'E') viol = r;
    else if (sn == 'G') viol = fmin(r, 0.0);
    else viol = fmax(r, 0.0);
    viol = viol / Dr[i] * Dr0[i];  // residual of the row-normalised problem
    v2 += viol * viol;
    dobj += b[i] * y[i];
  }
  sh[0][threadIdx.x] = v2;
  sh[1][threadIdx.x] = dobj;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      sh[0][threadIdx.x] += sh[0][threadIdx.x + s];
      sh[1][threadIdx.x] += sh[1][threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[blockIdx.x * 4 + 0] = sh[0][0];
    part[blockIdx.x * 4 + 1] = sh[1][0];
  }
}

__global__ void kkt_cols_kernel(const double* x, const double* c, const double* lb, const double* ub,
                                const double* Kty, int64_t n, double* part) {
  __shared__ double sh[2][kB];
  double pobj = 0.0, dbound = 0.0;
  GRID_LOOP(j, n) {
    pobj += c[j] * x[j];
    const double r = c[j] - Kty[j];  // reduced cost (scaled)
    dbound += (r > 0.0 ? lb[j] * r : ub[j] * r);
  }
  sh[0][threadIdx.x] = pobj;
  sh[1][threadIdx.x] = dbound;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      sh[0][threadIdx.x] += sh[0][threadIdx.x + s];
      sh[1][threadIdx.x] += sh[1][threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[blockIdx.x * 4 + 2] = sh[0][0];
    part[blockIdx.x * 4 + 3] = sh[1][0];
  }
}

__global__ void avg_kernel(const double* sum, double inv, int64_t n, double* out) {
  GRID_LOOP(i, n) out[i] = sum[i] * inv;
}
__global__ void unscale_kernel(const double* xs, const double* D, int64_t n, double* x, int mul) {
  GRID_LOOP(i, n) x[i] = mul ? xs[i] * D[i] : xs[i] / D[i];
}
__global__ void sq_diff_kernel(const double* a, const double* b, int64_t n, double* part) {
  __shared__ double sh[kB];
  double s = 0.0;
  GRID_LOOP(i, n) {
    const double d = a[i] - b[i];
    s += d * d;
  }
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int k = blockDim.x / 2; k > 0; k >>= 1) {
    if (threadIdx.x < k) sh[threadIdx.x] += sh[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}
__global__ void normalize_kernel(double* v, const double* part, int nb, int64_t n) {
  __shared__ double s;
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < nb; ++i) t += part[i];
    s = t > 0 ? 1.0 / sqrt(t) : 1.0;
  }
  __syncthreads();
  GRID_LOOP(i, n) v[i] *= s;
}

}  // namespace pd

using namespace pd;

struct PdhgState {
  DevBuf<double> Dr, Dr0, Dc, c_fix, ub_fix, val_s, cval_s, c_s, lb_s, ub_s, b_s, x, xbar, xsum, y, ysum, xr, yr, Kx, Kty, xa, ya, part,
      step, tmpn, tmpm;
  DevBuf<int32_t> col_of;
};

// One xe_pdhg_solve call.  Returns the result; x/y unscaled on the host if asked.
void pdhg_solve(xe_csr* M, const xe_pdhg_opts& o, xe_pdhg_result* res, double* x_out, double* y_out) {
  cudaStream_t s = M->stream;
  build_csc(M, s);
  const int64_t m = M->info.n_rows, n = M->info.n_cols, nnz = M->info.nnz;
  PdhgState S;
  S.Dr.alloc(m);
  S.Dr0.alloc(m);
  S.Dc.alloc(n);
  S.c_fix.alloc(n);
  S.ub_fix.alloc(n);
  S.val_s.alloc(nnz);
  S.cval_s.alloc(nnz);
  S.c_s.alloc(n);
  S.lb_s.alloc(n);
  S.ub_s.alloc(n);
  S.b_s.alloc(m);
  for (auto* v : {&S.x, &S.xbar, &S.xsum, &S.xr, &S.Kty, &S.xa, &S.tmpn}) v->alloc(n);
  for (auto* v : {&S.y, &S.ysum, &S.yr, &S.Kx, &S.ya, &S.tmpm}) v->alloc(m);
  const int gb = grid(std::max(m, n));
  S.part.alloc(static_cast<size_t>(gb) * 4 + 8);
  S.step.alloc(2);

  // bounds (node overrides for branch-and-bound)
  DevBuf<double> lb_o, ub_o;
  const double* lb = M->lb.p;
  const double* ub = M->ub.p;
  if (o.lb_override) {
    lb_o.upload(std::vector<double>(o.lb_override, o.lb_override + n), s);
    lb = lb_o.p;
  }
  if (o.ub_override) {
    ub_o.upload(std::vector<double>(o.ub_override, o.ub_override + n), s);
    ub = ub_o.p;
  }

  DevBuf<unsigned long long> fixcnt;
  fixcnt.alloc(2);
  XE_CUDA(cudaMemsetAsync(fixcnt.p, 0, 16, s));
  cudaEvent_t e0, e1;
  XE_CUDA(cudaEventCreate(&e0));
  XE_CUDA(cudaEventCreate(&e1));
  XE_CUDA(cudaEventRecord(e0, s));

  // ---- preconditioning: Ruiz (inf-norm) x10, then Pock-Chambolle (l1)
  {
    std::vector<double> ones_n(static_cast<size_t>(n), 1.0);
    row_inf_kernel<<<grid(m), kB, 0, s>>>(M->row_ptr.p, M->val.p, m, S.Dr0.p);
    XE_CUDA(cudaMemcpyAsync(S.Dr.p, S.Dr0.p, m * 8, cudaMemcpyDeviceToDevice, s));
    XE_CUDA(cudaMemcpyAsync(S.Dc.p, ones_n.data(), n * 8, cudaMemcpyHostToDevice, s));
    for (int it = 0; it < 11; ++it) {
      const int p = it == 10 ? 1 : 0;
      row_norm_kernel<<<grid(m), kB, 0, s>>>(M->row_ptr.p, M->col.p, M->val.p, S.Dr.p, S.Dc.p, m, p, S.tmpm.p);
      col_norm_kernel<<<grid(n), kB, 0, s>>>(M->col_ptr.p, M->crow.p, M->cval.p, S.Dr.p, S.Dc.p, n, p, S.tmpn.p);
      rescale_kernel<<<grid(m), kB, 0, s>>>(S.Dr.p, S.tmpm.p, m);
      rescale_kernel<<<grid(n), kB, 0, s>>>(S.Dc.p, S.tmpn.p, n);
    }
    scale_csr_kernel<<<grid(m), kB, 0, s>>>(M->row_ptr.p, M->col.p, M->val.p, S.Dr.p, S.Dc.p, m, S.val_s.p);
    scale_csc_kernel<<<grid(n), kB, 0, s>>>(M->col_ptr.p, M->crow.p, M->cval.p, S.Dr.p, S.Dc.p, n, S.cval_s.p);
    sentinel_kernel<<<grid(n), kB, 0, s>>>(M->obj.p, lb, ub, n, S.c_fix.p, S.ub_fix.p, fixcnt.p);
    scale_vec_kernel<<<grid(n), kB, 0, s>>>(S.c_fix.p, lb, S.ub_fix.p, S.Dc.p, n, S.c_s.p, S.lb_s.p, S.ub_s.p);
    scale_b_kernel<<<grid(m), kB, 0, s>>>(M->rhs.p, S.Dr.p, m, S.b_s.p);
    XE_CUDA(cudaGetLastError());
  }
  auto sqdist = [&](const double* a, const double* b, int64_t len) {
    const int g = grid(len);
    sq_diff_kernel<<<g, kB, 0, s>>>(a, b, len, S.part.p);
    std::vector<double> h(static_cast<size_t>(g));
    XE_CUDA(cudaMemcpyAsync(h.data(), S.part.p, h.size() * 8, cudaMemcpyDeviceToHost, s));
    XE_CUDA(cudaStreamSynchronize(s));
    double t = 0.0;
    for (double v : h) t += v;
    return t;
  };
  // ---- ||K~||_2 by power iteration on K~'K~
  double knorm = 1.0;
  {
    std::vector<double> v0(static_cast<size_t>(n));
    for (int64_t j = 0; j < n; ++j) v0[static_cast<size_t>(j)] = 1.0 + 0.01 * static_cast<double>((j * 7919) % 97);
    XE_CUDA(cudaMemcpyAsync(S.xr.p, v0.data(), n * 8, cudaMemcpyHostToDevice, s));
    XE_CUDA(cudaMemsetAsync(S.xa.p, 0, n * 8, s));
    normalize_kernel<<<1, kB, 0, s>>>(S.xr.p, S.part.p, 0, n);
    double lam = 0.0;
    for (int it = 0; it < 40; ++it) {
      spmv_kernel<<<grid(m), kB, 0, s>>>(M->row_ptr.p, M->col.p, S.val_s.p, S.xr.p, m, S.Kx.p);
      spmtv_kernel<<<grid(n), kB, 0, s>>>(M->col_ptr.p, M->crow.p, S.cval_s.p, S.Kx.p, n, S.xr.p);
      lam = sqdist(S.xr.p, S.xa.p, n);  // ||K'K v||^2 with |v| = 1
      const int g = grid(n);
      sq_diff_kernel<<<g, kB, 0, s>>>(S.xr.p, S.xa.p, n, S.part.p);
      normalize_kernel<<<1, kB, 0, s>>>(S.xr.p, S.part.p, g, n);
    }
    knorm = std::sqrt(std::sqrt(lam));
    if (!(knorm > 0)) knorm = 1.0;
  }
  const double eta = 0.95 / knorm;
  // initial primal weight ||c~|| / ||b~||
  const double cn = std::sqrt(sqdist(S.c_s.p, S.xa.p, n));
  XE_CUDA(cudaMemsetAsync(S.ya.p, 0, m * 8, s));
  const double bn = std::sqrt(sqdist(S.b_s.p, S.ya.p, m));
  double omega = (cn > 0 && bn > 0) ? cn / bn : 1.0;

  // ---- state
  XE_CUDA(cudaMemsetAsync(S.x.p, 0, n * 8, s));
  XE_CUDA(cudaMemsetAsync(S.y.p, 0, m * 8, s));
  XE_CUDA(cudaMemsetAsync(S.xsum.p, 0, n * 8, s));
  XE_CUDA(cudaMemsetAsync(S.ysum.p, 0, m * 8, s));
  XE_CUDA(cudaMemsetAsync(S.xr.p, 0, n * 8, s));  // last restart point
  XE_CUDA(cudaMemsetAsync(S.yr.p, 0, m * 8, s));
  auto set_step = [&] {
    const double st[2] = {eta / omega, eta * omega};
    XE_CUDA(cudaMemcpyAsync(S.step.p, st, sizeof st, cudaMemcpyHostToDevice, s));
  };
  set_step();

  Iter it{};
  it.rp = M->row_ptr.p;
  it.cp = M->col_ptr.p;
  it.col = M->col.p;
  it.row = M->crow.p;
  it.val = S.val_s.p;
  it.cval = S.cval_s.p;
  it.c = S.c_s.p;
  it.lb = S.lb_s.p;
  it.ub = S.ub_s.p;
  it.b = S.b_s.p;
  it.sense = M->sense.p;
  it.x = S.x.p;
  it.xbar = S.xbar.p;
  it.xsum = S.xsum.p;
  it.y = S.y.p;
  it.ysum = S.ysum.p;
  it.step = S.step.p;
  it.m = m;
  it.n = n;

  const int block = o.check_every > 0 ? o.check_every : 64;
  // lanes per column (SpM'V) and per row (SpMV) from the average lengths
  const int g_col = group_width(n ? static_cast<double>(nnz) / static_cast<double>(n) : 1.0);
  const int g_row = group_width(m ? static_cast<double>(nnz) / static_cast<double>(m) : 1.0);
  // captured graph of `block` iterations
  cudaGraph_t graph;
  cudaGraphExec_t gexec;
  XE_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  for (int k = 0; k < block; ++k) {
    launch_half_step(it, m, n, g_col, s, true);
    launch_half_step(it, m, n, g_row, s, false);
  }
  XE_CUDA(cudaStreamEndCapture(s, &graph));
  XE_CUDA(cudaGraphInstantiate(&gexec, graph, 0));

  // KKT of (xs, ys) (scaled): returns rel gap, rel primal res, pobj, dobj
  struct Kkt {
    double gap, pres, pobj, dobj, err;
  };
  std::vector<double> hb(static_cast<size_t>(m)), hd0(static_cast<size_t>(m));
  XE_CUDA(cudaMemcpyAsync(hb.data(), M->rhs.p, m * 8, cudaMemcpyDeviceToHost, s));
  XE_CUDA(cudaMemcpyAsync(hd0.data(), S.Dr0.p, m * 8, cudaMemcpyDeviceToHost, s));
  XE_CUDA(cudaStreamSynchronize(s));
  double b_l2 = 0.0;
  for (size_t i = 0; i < hb.size(); ++i) b_l2 += (hb[i] * hd0[i]) * (hb[i] * hd0[i]);
  b_l2 = std::sqrt(b_l2);

  auto kkt = [&](const double* xs, const double* ys) {
    spmv_kernel<<<grid(m), kB, 0, s>>>(M->row_ptr.p, M->col.p, S.val_s.p, xs, m, S.Kx.p);
    spmtv_kernel<<<grid(n), kB, 0, s>>>(M->col_ptr.p, M->crow.p, S.cval_s.p, ys, n, S.Kty.p);
    const int gm = grid(m), gn = grid(n), g = std::max(gm, gn);
    XE_CUDA(cudaMemsetAsync(S.part.p, 0, static_cast<size_t>(g) * 4 * 8, s));
    kkt_rows_kernel<<<gm, kB, 0, s>>>(S.Kx.p, S.b_s.p, M->sense.p, ys, S.Dr.p, S.Dr0.p, m, S.part.p);
    kkt_cols_kernel<<<gn, kB, 0, s>>>(xs, S.c_s.p, S.lb_s.p, S.ub_s.p, S.Kty.p, n, S.part.p);
    std::vector<double> h(static_cast<size_t>(g) * 4);
    XE_CUDA(cudaMemcpyAsync(h.data(), S.part.p, h.size() * 8, cudaMemcpyDeviceToHost, s));
    XE_CUDA(cudaStreamSynchronize(s));
    double v2 = 0, drow = 0, pobj = 0, dbound = 0;
    for (int i = 0; i < g; ++i) {
      v2 += h[static_cast<size_t>(i) * 4 + 0];
      drow += h[static_cast<size_t>(i) * 4 + 1];
      pobj += h[static_cast<size_t>(i) * 4 + 2];
      dbound += h[static_cast<size_t>(i) * 4 + 3];
    }
    Kkt k{};
    k.pobj = pobj;
    k.dobj = drow + dbound;
    k.gap = std::fabs(k.pobj - k.dobj) / (1.0 + std::fabs(k.pobj) + std::fabs(k.dobj));
    k.pres = std::sqrt(v2) / (1.0 + b_l2);
    k.err = std::sqrt(k.gap * k.gap + k.pres * k.pres);
    return k;
  };

  const int max_iters = o.max_iters > 0 ? o.max_iters : 200000;
  const double tol = o.tol_rel > 0 ? o.tol_rel : 1e-6;
  int iters = 0, restarts = 0, since = 0;
  Kkt last_restart = kkt(S.x.p, S.y.p), prev_cand = last_restart, cur{};
  int status = 1;
  float loop_ms = 0.f;
  cudaEvent_t l0, l1;
  XE_CUDA(cudaEventCreate(&l0));
  XE_CUDA(cudaEventCreate(&l1));
  while (iters < max_iters) {
    XE_CUDA(cudaEventRecord(l0, s));
    XE_CUDA(cudaGraphLaunch(gexec, s));
    XE_CUDA(cudaEventRecord(l1, s));
    XE_CUDA(cudaEventSynchronize(l1));
    float ms = 0.f;
    XE_CUDA(cudaEventElapsedTime(&ms, l0, l1));
    loop_ms += ms;
    iters += block;
    since += block;
    // current and average iterates
    avg_kernel<<<grid(n), kB, 0, s>>>(S.xsum.p, 1.0 / since, n, S.xa.p);
    avg_kernel<<<grid(m), kB, 0, s>>>(S.ysum.p, 1.0 / since, m, S.ya.p);
    cur = kkt(S.x.p, S.y.p);
    Kkt avg = kkt(S.xa.p, S.ya.p);
    const bool use_avg = avg.err < cur.err;
    const Kkt cand = use_avg ? avg : cur;
    if (o.verbose)
      std::fprintf(stderr, "pdhg it=%d pobj=%.12g dobj=%.12g gap=%.2e pres=%.2e (avg %.2e) w=%.3g\n", iters,
                   cur.pobj, cur.dobj, cur.gap, cur.pres, avg.err, omega);
    if (cand.gap <= tol && cand.pres <= tol) {
      if (use_avg) {
        XE_CUDA(cudaMemcpyAsync(S.x.p, S.xa.p, n * 8, cudaMemcpyDeviceToDevice, s));
        XE_CUDA(cudaMemcpyAsync(S.y.p, S.ya.p, m * 8, cudaMemcpyDeviceToDevice, s));
      }
      cur = cand;
      status = 0;
      break;
    }
    // PDLP adaptive restart criteria
    const bool restart = cand.err <= 0.2 * last_restart.err ||
                         (cand.err <= 0.8 * last_restart.err && cand.err > prev_cand.err) ||
                         since >= 0.36 * iters;
    prev_cand = cand;
    if (restart) {
      if (use_avg) {
        XE_CUDA(cudaMemcpyAsync(S.x.p, S.xa.p, n * 8, cudaMemcpyDeviceToDevice, s));
        XE_CUDA(cudaMemcpyAsync(S.y.p, S.ya.p, m * 8, cudaMemcpyDeviceToDevice, s));
      }
      // primal weight update (theta = 0.5) from the movement since the last restart
      const double dx = std::sqrt(sqdist(S.x.p, S.xr.p, n)), dy = std::sqrt(sqdist(S.y.p, S.yr.p, m));
      if (dx > 1e-10 && dy > 1e-10) omega = std::exp(0.5 * std::log(dy / dx) + 0.5 * std::log(omega));
      set_step();
      XE_CUDA(cudaMemcpyAsync(S.xr.p, S.x.p, n * 8, cudaMemcpyDeviceToDevice, s));
      XE_CUDA(cudaMemcpyAsync(S.yr.p, S.y.p, m * 8, cudaMemcpyDeviceToDevice, s));
      XE_CUDA(cudaMemsetAsync(S.xsum.p, 0, n * 8, s));
      XE_CUDA(cudaMemsetAsync(S.ysum.p, 0, m * 8, s));
      last_restart = cand;
      since = 0;
      ++restarts;
    }
  }
  XE_CUDA(cudaEventRecord(e1, s));
  XE_CUDA(cudaEventSynchronize(e1));
  float total_ms = 0.f;
  XE_CUDA(cudaEventElapsedTime(&total_ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(l0);
  cudaEventDestroy(l1);
  cudaGraphExecDestroy(gexec);
  cudaGraphDestroy(graph);

  // certify the prohibitive-cost presolve with the final duals
  spmtv_kernel<<<grid(n), kB, 0, s>>>(M->col_ptr.p, M->crow.p, S.cval_s.p, S.y.p, n, S.Kty.p);
  certify_kernel<<<grid(n), kB, 0, s>>>(M->obj.p, lb, S.Kty.p, S.Dc.p, n, fixcnt.p + 1);
  unsigned long long fc[2] = {0, 0};
  XE_CUDA(cudaMemcpyAsync(fc, fixcnt.p, 16, cudaMemcpyDeviceToHost, s));
  XE_CUDA(cudaStreamSynchronize(s));
  res->presolve_fixed = static_cast<int32_t>(fc[0]);
  res->certified = fc[1] == 0 ? 1 : 0;
  res->primal_obj = cur.pobj;
  res->dual_obj = cur.dobj;
  res->rel_gap = cur.gap;
  res->rel_primal_res = cur.pres;
  res->rel_dual_res = 0.0;  // every column is boxed: reduced costs are absorbed by bound multipliers
  res->iters = iters;
  res->restarts = restarts;
  res->status = status;
  res->solve_ms = total_ms;
  res->spmv_ms_per_iter = iters ? loop_ms / iters : 0.0;
  if (x_out) {
    unscale_kernel<<<grid(n), kB, 0, s>>>(S.x.p, S.Dc.p, n, S.tmpn.p, 1);
    XE_CUDA(cudaMemcpyAsync(x_out, S.tmpn.p, n * 8, cudaMemcpyDeviceToHost, s));
  }
  if (y_out) {
    unscale_kernel<<<grid(m), kB, 0, s>>>(S.y.p, S.Dr.p, m, S.tmpm.p, 1);
    XE_CUDA(cudaMemcpyAsync(y_out, S.tmpm.p, m * 8, cudaMemcpyDeviceToHost, s));
  }
  XE_CUDA(cudaStreamSynchronize(s));
}

}  // namespace xe

extern "C" int xe_pdhg_solve(xe_csr* m, const xe_pdhg_opts* opts, xe_pdhg_result* res, double* x_out,
                             double* y_out) {
  return xe::guard([&] {
    if (!m || !res) xe::fail(XE_ERR_ARG, "null argument");
    xe::require_uploaded(m->prob);
    xe_pdhg_opts o{};
    if (opts) o = *opts;
    std::memset(res, 0, sizeof *res);
    xe::pdhg_solve(m, o, res, x_out, y_out);
  });
}
