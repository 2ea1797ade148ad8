// SPDX-License-Identifier: Apache-2.0
//
// K1 — assembly of the scheduling MILP as CSR on the GPU.
//
// Reproduces build_model (proj/src/model.cpp:86-256) + add_energy_extension
// (model.cpp:258-312) row for row: rows in emission order, terms of each row
// in the reference's push order, per-tag ordinals, rhs and sense; the
// objective map (model.cpp:107-124, 273-284), the fixed-zero triangles
// (model.cpp:127-132) and the write_mps bounds (mps_io.cpp:172-186) as dense
// per-column arrays.  Columns use the closed-form VarRef index (model.hpp:
// 14-31; VarFamily order R<S<Z<F<U<P, lexicographic indices), so column order
// equals write_mps's std::map order and the MPS text is reproduced byte for
// byte from the column-major (stable) copy (xe_write_mps, mps_writer.cpp).
//
// Kernels: (1) one thread per row computes the row's length, sense, rhs, tag
// and ordinal in closed form; (2) exclusive scan of lengths -> row_ptr;
// (3) one thread per row writes its terms; (4) one thread per column writes
// objective / bounds.  All HBM-write bound: 12 B per nonzero + 26 B per row
// + 26 B per column.

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstring>
#include <memory>

#include "csr.hpp"

namespace xe {
namespace k1 {

// ConstraintTag values (model.hpp:36-39)
enum : uint8_t { EQ7, EQ8, EQ9, EQ10, EQ11, EQ12, EQ13, EQ14, EQ16_LO, EQ16_HI, Z_LINK, P_LINK,
                 ENERGY_DEV, ENERGY_TOTAL };
// row families in emission order
enum Fam { F_EQ8, F_EQ9, F_EQ11, F_EQ12, F_EQ13, F_EQ14, F_EQ16, F_ZLINK, F_PLINK, F_EDEV, F_ETOT, F_END };

struct Args {
  int D, T, E, FE, strict;
  int64_t fam_off[F_END + 1];  // first row of each family
  const int32_t* src;
  const int32_t* dst;
  const int32_t* in_ptr;   // [T+1] in-edges of v (edge order)
  const int32_t* in_edge;
  const int32_t* out_ptr;  // [T+1] out-edges of u (edge order)
  const int32_t* out_edge;
  const int64_t* mass;
  const double* q;         // [D][T]
  const int32_t* edev;     // devices with an energy limit, ascending
  const double* elim;
  int n_edev;
  int etot_nnz;            // terms per ENERGY_TOTAL row (q != 0)
  double etot_rhs;
  // outputs
  int64_t* row_ptr;
  int32_t* col;
  double* val;
  double* rhs;
  int8_t* sense;
  uint8_t* tag;
  int32_t* ordinal;
};

struct Cols {
  int64_t R, S, Z, F, U, P, n;
  int D, T, E, FE;
  __host__ __device__ int64_t r(int d, int t, int i) const { return R + (static_cast<int64_t>(d) * T + t) * T + i; }
  __host__ __device__ int64_t s(int d, int t, int i) const { return S + (static_cast<int64_t>(d) * T + t) * T + i; }
  __host__ __device__ int64_t z(int d, int t, int i) const { return Z + (static_cast<int64_t>(d) * T + t) * T + i; }
  __host__ __device__ int64_t f(int d, int t, int eo) const { return F + (static_cast<int64_t>(d) * T + t) * FE + eo; }
  __host__ __device__ int64_t u(int d, int t, int i) const { return U + (static_cast<int64_t>(d) * T + t) * T + i; }
  __host__ __device__ int64_t p(int t, int e, int ds, int dc) const {
    return P + ((static_cast<int64_t>(t) * E + e) * D + ds) * (D - 1) + (dc - (dc > ds ? 1 : 0));
  }
};

__host__ __device__ inline Cols make_cols(int D, int T, int E) {
  Cols c;
  c.D = D;
  c.T = T;
  c.E = E;
  c.FE = E + T;
  const int64_t DT2 = static_cast<int64_t>(D) * T * T;
  c.R = 0;
  c.S = DT2;
  c.Z = 2 * DT2;
  c.F = 3 * DT2;
  c.U = 3 * DT2 + static_cast<int64_t>(D) * T * c.FE;
  c.P = c.U + DT2;
  c.n = c.P + static_cast<int64_t>(T) * E * D * (D - 1);
  return c;
}

__device__ __forceinline__ int family(const Args& a, int64_t r) {
  int f = 0;
#pragma unroll
  for (int k = 1; k < F_END; ++k)
    if (r >= a.fam_off[k]) f = k;
  return f;
}

// number of consumers w > v of u (EQ16 "later"), from u's out-edges
__device__ __forceinline__ int later_count(const Args& a, int u, int v) {
  int c = 0;
  for (int k = a.out_ptr[u]; k < a.out_ptr[u + 1]; ++k) c += a.dst[a.out_edge[k]] > v;
  return c;
}

// One row's metadata (and terms when `emit`), in the reference's order.
template <bool EMIT>
__device__ __forceinline__ int row_gen(const Args& a, const Cols& C, int64_t r, int64_t pos,
                                       double* rhs_o, int8_t* sense_o, uint8_t* tag_o, int32_t* ord_o) {
  const int D = a.D, T = a.T, E = a.E;
  const int fam = family(a, r);
  const int64_t k = r - a.fam_off[fam];
  int n = 0;
  auto put = [&](int64_t col, double v) {
    if (EMIT) {
      a.col[pos + n] = static_cast<int32_t>(col);
      a.val[pos + n] = v;
    }
    ++n;
  };
  double rhs = 0.0;
  int8_t sense = 'L';
  uint8_t tag = EQ8;
  int32_t ord = static_cast<int32_t>(k);
  switch (fam) {
    case F_EQ8: {  // model.cpp:138-146, GE then LE per t
      const int t = static_cast<int>(k >> 1);
      for (int d = 0; d < D; ++d) put(C.r(d, t, t), 1.0);
      sense = (k & 1) ? 'L' : 'G';
      rhs = 1.0;
      tag = EQ8;
      break;
    }
    case F_EQ9: {  // model.cpp:147-152
      for (int t = 0; t < T; ++t)
        for (int d = 0; d < D; ++d) put(C.r(d, t, t), 1.0);
      sense = 'E';
      rhs = static_cast<double>(T);
      tag = EQ9;
      break;
    }
    case F_EQ11: {  // model.cpp:155-160
      const int i = static_cast<int>(k % T);
      const int t = static_cast<int>((k / T) % (T - 1));
      const int d = static_cast<int>(k / (static_cast<int64_t>(T) * (T - 1)));
      put(C.s(d, t + 1, i), 1.0);
      put(C.s(d, t, i), -1.0);
      put(C.r(d, t, i), -1.0);
      tag = EQ11;
      break;
    }
    case F_EQ12: {  // model.cpp:163-173
      const int e = static_cast<int>(k % E);
      const int t = static_cast<int>((k / E) % T);
      const int d = static_cast<int>(k / (static_cast<int64_t>(E) * T));
      put(C.r(d, t, a.dst[e]), 1.0);
      for (int ds = 0; ds < D; ++ds) {
        put(C.r(ds, t, a.src[e]), -1.0);
        put(C.s(ds, t, a.src[e]), -1.0);
      }
      tag = EQ12;
      break;
    }
    case F_EQ13: {  // model.cpp:176-182
      const int t = static_cast<int>(k % T), d = static_cast<int>(k / T);
      put(C.u(d, t, 0), 1.0);
      for (int i = 0; i < T; ++i) put(C.s(d, t, i), -static_cast<double>(a.mass[i]));
      put(C.r(d, t, 0), -static_cast<double>(a.mass[0]));
      sense = 'E';
      tag = EQ13;
      break;
    }
    case F_EQ14: {  // model.cpp:185-195
      const int v = static_cast<int>(k % (T - 1));
      const int t = static_cast<int>((k / (T - 1)) % T);
      const int d = static_cast<int>(k / (static_cast<int64_t>(T - 1) * T));
      put(C.u(d, t, v + 1), 1.0);
      put(C.u(d, t, v), -1.0);
      for (int j = a.in_ptr[v]; j < a.in_ptr[v + 1]; ++j) {
        const int e = a.in_edge[j];
        put(C.f(d, t, e), static_cast<double>(a.mass[a.src[e]]));
      }
      put(C.f(d, t, E + v), static_cast<double>(a.mass[v]));
      put(C.r(d, t, v + 1), -static_cast<double>(a.mass[v + 1]));
      sense = 'E';
      tag = EQ14;
      break;
    }
    case F_EQ16: {  // model.cpp:200-224, LO then HI per (d,t,eo)
      const bool hi = k & 1;
      const int64_t kk = k >> 1;
      const int eo = static_cast<int>(kk % a.FE);
      const int t = static_cast<int>((kk / a.FE) % T);
      const int d = static_cast<int>(kk / (static_cast<int64_t>(a.FE) * T));
      const int u = eo < E ? a.src[eo] : eo - E;
      const int v = eo < E ? a.dst[eo] : eo - E;
      const int nl = later_count(a, u, v);
      const double h_max = 2.0 + static_cast<double>(nl) * (a.strict ? static_cast<double>(D) : 1.0);
      put(C.r(d, t, v), -1.0);
      put(C.z(d, t, u), -1.0);
      if (t + 1 < T) put(C.s(d, t + 1, u), 1.0);
      for (int j = a.out_ptr[u]; j < a.out_ptr[u + 1]; ++j) {
        const int w = a.dst[a.out_edge[j]];
        if (w <= v) continue;
        if (a.strict)
          for (int dd = 0; dd < D; ++dd) put(C.r(dd, t, w), 1.0);
        else
          put(C.r(d, t, w), 1.0);
      }
      put(C.f(d, t, eo), hi ? h_max : 1.0);
      sense = hi ? 'L' : 'G';
      rhs = hi ? h_max - 2.0 : -1.0;
      tag = hi ? EQ16_HI : EQ16_LO;
      ord = static_cast<int32_t>(kk);
      break;
    }
    case F_ZLINK: {  // model.cpp:227-237, three rows per (d,t,i)
      const int which = static_cast<int>(k % 3);
      const int64_t kk = k / 3;
      const int i = static_cast<int>(kk % T), t = static_cast<int>((kk / T) % T);
      const int d = static_cast<int>(kk / (static_cast<int64_t>(T) * T));
      put(C.z(d, t, i), 1.0);
      if (which != 2) put(C.r(d, t, i), -1.0);
      if (which != 1) put(C.s(d, t, i), -1.0);
      sense = which == 0 ? 'L' : 'G';
      tag = Z_LINK;
      break;
    }
    case F_PLINK: {  // model.cpp:240-252
      const int dm1 = D - 1;
      const int x = static_cast<int>(k % dm1);
      const int ds = static_cast<int>((k / dm1) % D);
      const int e = static_cast<int>((k / (static_cast<int64_t>(dm1) * D)) % E);
      const int t = static_cast<int>(k / (static_cast<int64_t>(dm1) * D * E));
      const int dc = x >= ds ? x + 1 : x;
      put(C.p(t, e, ds, dc), 1.0);
      put(C.r(dc, t, a.dst[e]), -1.0);
      put(C.z(ds, t, a.src[e]), -1.0);
      sense = 'G';
      rhs = -1.0;
      tag = P_LINK;
      break;
    }
    case F_EDEV: {  // model.cpp:292-297 (zero q kept)
      const int i = static_cast<int>(k % T), t = static_cast<int>((k / T) % T);
      const int kd = static_cast<int>(k / (static_cast<int64_t>(T) * T));
      const int d = a.edev[kd];
      put(C.r(d, t, i), a.q[static_cast<int64_t>(d) * T + i]);
      rhs = a.elim[kd];
      tag = ENERGY_DEV;
      break;
    }
    default: {  // F_ETOT, model.cpp:299-310 (zero q dropped)
      const int t = static_cast<int>(k);
      if (EMIT) {
        for (int d = 0; d < D; ++d)
          for (int i = 0; i < T; ++i) {
            const double qv = a.q[static_cast<int64_t>(d) * T + i];
            if (qv != 0.0) put(C.r(d, t, i), qv);
          }
      } else {
        n = a.etot_nnz;
      }
      rhs = a.etot_rhs;
      tag = ENERGY_TOTAL;
      break;
    }
  }
  if (!EMIT) {
    *rhs_o = rhs;
    *sense_o = sense;
    *tag_o = tag;
    *ord_o = ord;
  }
  return n;
}

__global__ void row_meta_kernel(const Args a, Cols C, int64_t m) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < m;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double rhs;
    int8_t sense;
    uint8_t tag;
    int32_t ord;
    const int n = row_gen<false>(a, C, r, 0, &rhs, &sense, &tag, &ord);
    a.row_ptr[r] = n;  // lengths; scanned in place afterwards
    a.rhs[r] = rhs;
    a.sense[r] = sense;
    a.tag[r] = tag;
    a.ordinal[r] = ord;
  }
}

__global__ void row_fill_kernel(const Args a, Cols C, int64_t m) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < m;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double rhs;
    int8_t sense;
    uint8_t tag;
    int32_t ord;
    row_gen<true>(a, C, r, a.row_ptr[r], &rhs, &sense, &tag, &ord);
  }
}

struct ColArgs {
  int D, T, E;
  const double* cost;  // [D][T]
  const double* w;     // [E][D][D]
  const double* aq;    // alpha*q [D][T] or null
  const int64_t* budget;
  double* obj;
  uint8_t* present;
  double* lb;
  double* ub;
  uint8_t* kind;
};

// objective (model.cpp:107-124 + energy 273-284), bounds (mps_io.cpp:172-186)
__global__ void col_kernel(const ColArgs a, Cols C) {
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < C.n;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double o = 0.0;
    uint8_t pres = 0, kind;
    double ub;
    if (j < C.F) {  // R, S, Z: binaries; fixed triangles
      const int64_t x = j % C.S;
      const int fam = static_cast<int>(j / C.S);
      const int i = static_cast<int>(x % a.T), t = static_cast<int>((x / a.T) % a.T);
      const int d = static_cast<int>(x / (static_cast<int64_t>(a.T) * a.T));
      const bool fixed = (fam == 0 && i > t) || (fam == 1 && i >= t);
      kind = fixed ? 0 : 1;
      ub = fixed ? 0.0 : 1.0;
      if (fam == 0) {
        const double c = a.cost[static_cast<int64_t>(d) * a.T + i];
        if (c != 0.0) {
          o = c;
          pres = 1;
        }
        if (a.aq) {
          const double add = a.aq[static_cast<int64_t>(d) * a.T + i];
          if (add != 0.0) {
            const double next = pres ? o + add : add;
            o = next == 0.0 ? 0.0 : next;
            pres = next != 0.0;
          }
        }
      }
    } else if (j < C.U) {  // F
      kind = 1;
      ub = 1.0;
    } else if (j < C.P) {  // U
      const int d = static_cast<int>((j - C.U) / (static_cast<int64_t>(a.T) * a.T));
      kind = 2;
      ub = static_cast<double>(a.budget[d]);
    } else {  // P
      const int64_t x = j - C.P;
      const int dm1 = a.D - 1;
      const int xx = static_cast<int>(x % dm1);
      const int ds = static_cast<int>((x / dm1) % a.D);
      const int e = static_cast<int>((x / (static_cast<int64_t>(dm1) * a.D)) % a.E);
      const int dc = xx >= ds ? xx + 1 : xx;
      const double w = a.w[(static_cast<int64_t>(e) * a.D + ds) * a.D + dc];
      if (w != 0.0) {
        o = w;
        pres = 1;
      }
      kind = 3;
      ub = 1.0;
    }
    a.obj[j] = o;
    a.present[j] = pres;
    a.lb[j] = 0.0;
    a.ub[j] = ub;
    a.kind[j] = kind;
  }
}

__global__ void iota_kernel(int64_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = i;
}

__global__ void csc_gather_kernel(const int64_t* perm, const double* val, const int64_t* row_of_entry_unused,
                                  double* cval, int64_t nnz) {
  (void)row_of_entry_unused;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nnz;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    cval[i] = val[perm[i]];
}

// row index of every entry (entries of row r are [row_ptr[r], row_ptr[r+1]))
__global__ void entry_row_kernel(const int64_t* row_ptr, int64_t m, int32_t* row_of) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < m;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x)
    for (int64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) row_of[k] = static_cast<int32_t>(r);
}

__global__ void csc_rows_kernel(const int64_t* perm, const int32_t* row_of, int32_t* crow, int64_t nnz) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nnz;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    crow[i] = row_of[perm[i]];
}

// column pointers from sorted column keys: col_ptr[c] = first i with key >= c
__global__ void col_ptr_kernel(const int32_t* keys, int64_t nnz, int64_t ncol, int64_t* col_ptr) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i <= nnz;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t lo = i == 0 ? 0 : static_cast<int64_t>(keys[i - 1]) + 1;
    const int64_t hi = i == nnz ? ncol : static_cast<int64_t>(keys[i]);
    for (int64_t c = lo; c <= hi && c <= ncol; ++c) col_ptr[c] = i;
  }
}

}  // namespace k1
}  // namespace xe

namespace xe {

static int64_t h_in_deg(const HostProblem& h, int v) {
  int64_t c = 0;
  for (int e = 0; e < h.E; ++e) c += h.dst[static_cast<size_t>(e)] == v;
  return c;
}

static int grid_for(int64_t n, int block = 256) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + block - 1) / block, 148LL * 64)));
}

xe_csr* build_csr(const xe_problem* pr, const xe_model_opts& opts, cudaStream_t s) {
  const HostProblem& h = pr->h;
  if (!h.missing_link.empty() && h.D > 1) fail(XE_ERR_MISSING_LINK, h.missing_link);
  const int D = h.D, T = h.T, E = h.E, FE = E + T;
  if (T > 32767 || FE > 32767) fail(XE_ERR_TOO_LARGE, "VarRef indices are int16 (model.hpp:20-24)");
  const bool energy = opts.use_energy && h.has_energy;
  auto m = std::make_unique<xe_csr>();
  m->prob = pr;
  m->opts = opts;
  m->stream = s;
  const k1::Cols C = k1::make_cols(D, T, E);
  if (C.n > INT32_MAX) fail(XE_ERR_TOO_LARGE, "more than 2^31 columns");

  // family sizes in emission order
  std::vector<int32_t> edev;
  std::vector<double> elim;
  if (energy)
    for (int d = 0; d < D; ++d)
      if (h.has_lim[static_cast<size_t>(d)]) {
        edev.push_back(d);
        elim.push_back(h.lim[static_cast<size_t>(d)]);
      }
  int etot_nnz = 0;
  if (energy)
    for (double q : h.q) etot_nnz += q != 0.0;
  const int64_t T64 = T, D64 = D, E64 = E;
  int64_t sizes[k1::F_END] = {
      2 * T64,                                   // EQ8
      1,                                         // EQ9
      D64 * (T64 - 1) * T64,                     // EQ11
      D64 * T64 * E64,                           // EQ12
      D64 * T64,                                 // EQ13
      D64 * T64 * (T64 - 1),                     // EQ14
      2 * D64 * T64 * FE,                        // EQ16 LO/HI
      3 * D64 * T64 * T64,                       // Z_LINK
      T64 * E64 * D64 * (D64 - 1),               // P_LINK
      static_cast<int64_t>(edev.size()) * T64 * T64,           // ENERGY_DEV
      (energy && h.has_total) ? T64 : 0,         // ENERGY_TOTAL
  };
  k1::Args a{};
  a.D = D;
  a.T = T;
  a.E = E;
  a.FE = FE;
  a.strict = opts.strict_free ? 1 : 0;
  a.fam_off[0] = 0;
  for (int f = 0; f < k1::F_END; ++f) a.fam_off[f + 1] = a.fam_off[f] + sizes[f];
  const int64_t nrows = a.fam_off[k1::F_END];

  // out-edge lists (edge order) for the EQ16 "later consumers"
  std::vector<int32_t> out_ptr(static_cast<size_t>(T) + 1, 0), out_edge(static_cast<size_t>(E));
  for (int e = 0; e < E; ++e) out_ptr[static_cast<size_t>(h.src[static_cast<size_t>(e)]) + 1]++;
  for (int v = 0; v < T; ++v) out_ptr[static_cast<size_t>(v) + 1] += out_ptr[static_cast<size_t>(v)];
  {
    std::vector<int32_t> fill(out_ptr.begin(), out_ptr.end() - 1);
    for (int e = 0; e < E; ++e) out_edge[static_cast<size_t>(fill[static_cast<size_t>(h.src[static_cast<size_t>(e)])]++)] = e;
  }
  DevBuf<int32_t> d_out_ptr, d_out_edge, d_edev;
  DevBuf<double> d_elim, d_aq;
  d_out_ptr.upload(out_ptr, s);
  d_out_edge.upload(out_edge.empty() ? std::vector<int32_t>(1, 0) : out_edge, s);
  d_edev.upload(edev.empty() ? std::vector<int32_t>(1, 0) : edev, s);
  d_elim.upload(elim.empty() ? std::vector<double>(1, 0.0) : elim, s);

  a.src = pr->d_src.p;
  a.dst = pr->d_dst.p;
  a.in_ptr = pr->d_in_ptr.p;
  a.in_edge = pr->d_in_edge.p;
  a.out_ptr = d_out_ptr.p;
  a.out_edge = d_out_edge.p;
  a.mass = pr->d_mass.p;
  a.q = pr->d_q.p;
  a.edev = d_edev.p;
  a.elim = d_elim.p;
  a.n_edev = static_cast<int>(edev.size());
  a.etot_nnz = etot_nnz;
  a.etot_rhs = h.total_limit - h.board;

  // nnz in closed form (the row lengths row_gen emits, summed per family):
  // every buffer is allocated before the timed kernels, no mid-build sync
  int64_t nnz_closed = 0;
  {
    int64_t sum_indeg = 0;  // EQ14: v = 0 .. T-2
    for (int v = 0; v + 1 < T; ++v) sum_indeg += h_in_deg(h, v);
    int64_t sum_later = 0;  // EQ16: later consumers of (u, v) over free-edges
    auto later = [&](int u, int v) {
      int64_t c = 0;
      for (int k = out_ptr[static_cast<size_t>(u)]; k < out_ptr[static_cast<size_t>(u) + 1]; ++k)
        c += h.dst[static_cast<size_t>(out_edge[static_cast<size_t>(k)])] > v;
      return c;
    };
    for (int e = 0; e < E; ++e) sum_later += later(h.src[static_cast<size_t>(e)], h.dst[static_cast<size_t>(e)]);
    for (int v = 0; v < T; ++v) sum_later += later(v, v);
    const int64_t kq = opts.strict_free ? D64 : 1;
    nnz_closed = 2 * T64 * D64                                          // EQ8
                 + T64 * D64                                            // EQ9
                 + 3 * D64 * (T64 - 1) * T64                            // EQ11
                 + D64 * T64 * E64 * (1 + 2 * D64)                      // EQ12
                 + D64 * T64 * (T64 + 2)                                // EQ13
                 + D64 * T64 * (4 * (T64 - 1) + sum_indeg)              // EQ14
                 + 2 * D64 * (T64 * (3 * FE + kq * sum_later) + (T64 - 1) * FE)  // EQ16 LO+HI
                 + 7 * D64 * T64 * T64                                  // Z_LINK
                 + 3 * T64 * E64 * D64 * (D64 - 1)                      // P_LINK
                 + sizes[k1::F_EDEV]                                    // ENERGY_DEV
                 + sizes[k1::F_ETOT] * etot_nnz;                        // ENERGY_TOTAL
  }
  m->row_ptr.alloc(static_cast<size_t>(nrows) + 1);
  m->col.alloc(static_cast<size_t>(std::max<int64_t>(1, nnz_closed)));
  m->val.alloc(static_cast<size_t>(std::max<int64_t>(1, nnz_closed)));
  m->rhs.alloc(static_cast<size_t>(nrows));
  m->sense.alloc(static_cast<size_t>(nrows));
  m->tag.alloc(static_cast<size_t>(nrows));
  m->ordinal.alloc(static_cast<size_t>(nrows));
  a.row_ptr = m->row_ptr.p;
  a.rhs = m->rhs.p;
  a.sense = m->sense.p;
  a.tag = m->tag.p;
  a.ordinal = m->ordinal.p;

  a.col = m->col.p;
  a.val = m->val.p;
  // columns: objective (+ alpha*q), bounds, kind
  k1::ColArgs ca{};
  ca.D = D;
  ca.T = T;
  ca.E = E;
  ca.cost = pr->d_cost.p;
  ca.w = pr->d_w.p;
  if (energy && h.alpha != 0.0) {
    std::vector<double> aq(static_cast<size_t>(D) * T);
    for (size_t i = 0; i < aq.size(); ++i) aq[i] = h.alpha * h.q[i];
    d_aq.upload(aq, s);
    ca.aq = d_aq.p;
  }
  ca.budget = pr->d_budget.p;
  m->obj.alloc(static_cast<size_t>(C.n));
  m->present.alloc(static_cast<size_t>(C.n));
  m->lb.alloc(static_cast<size_t>(C.n));
  m->ub.alloc(static_cast<size_t>(C.n));
  m->kind.alloc(static_cast<size_t>(C.n));
  ca.obj = m->obj.p;
  ca.present = m->present.p;
  ca.lb = m->lb.p;
  ca.ub = m->ub.p;
  ca.kind = m->kind.p;
  size_t tmp_bytes = 0;
  XE_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, m->row_ptr.p, m->row_ptr.p, nrows + 1, s));
  DevBuf<unsigned char> tmp;
  tmp.alloc(std::max<size_t>(1, tmp_bytes));

  // the timed build: kernels only (row metadata and lengths, exclusive scan
  // of the lengths in place, row terms, columns)
  cudaEvent_t e0, e1;
  XE_CUDA(cudaEventCreate(&e0));
  XE_CUDA(cudaEventCreate(&e1));
  XE_CUDA(cudaEventRecord(e0, s));
  k1::row_meta_kernel<<<grid_for(nrows), 256, 0, s>>>(a, C, nrows);
  XE_CUDA(cudaGetLastError());
  XE_CUDA(cudaMemsetAsync(m->row_ptr.p + nrows, 0, sizeof(int64_t), s));
  XE_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, m->row_ptr.p, m->row_ptr.p, nrows + 1, s));
  k1::row_fill_kernel<<<grid_for(nrows), 256, 0, s>>>(a, C, nrows);
  XE_CUDA(cudaGetLastError());
  k1::col_kernel<<<grid_for(C.n), 256, 0, s>>>(ca, C);
  XE_CUDA(cudaGetLastError());
  XE_CUDA(cudaEventRecord(e1, s));
  int64_t nnz = 0;
  XE_CUDA(cudaMemcpyAsync(&nnz, m->row_ptr.p + nrows, sizeof nnz, cudaMemcpyDeviceToHost, s));
  XE_CUDA(cudaEventSynchronize(e1));
  XE_CUDA(cudaStreamSynchronize(s));
  XE_CUDA(cudaEventElapsedTime(&m->build_ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (nnz != nnz_closed) fail(XE_ERR_ARG, "K1: closed-form nnz " + std::to_string(nnz_closed) + " != scanned " + std::to_string(nnz));

  xe_csr_info& in = m->info;
  in.n_cols = C.n;
  in.n_rows = nrows;
  in.nnz = nnz;
  in.D = D;
  in.T = T;
  in.E = E;
  in.n_tags = 14;
  std::memset(in.tag_rows, 0, sizeof in.tag_rows);
  in.tag_rows[k1::EQ8] = sizes[k1::F_EQ8];
  in.tag_rows[k1::EQ9] = sizes[k1::F_EQ9];
  in.tag_rows[k1::EQ11] = sizes[k1::F_EQ11];
  in.tag_rows[k1::EQ12] = sizes[k1::F_EQ12];
  in.tag_rows[k1::EQ13] = sizes[k1::F_EQ13];
  in.tag_rows[k1::EQ14] = sizes[k1::F_EQ14];
  in.tag_rows[k1::EQ16_LO] = sizes[k1::F_EQ16] / 2;
  in.tag_rows[k1::EQ16_HI] = sizes[k1::F_EQ16] / 2;
  in.tag_rows[k1::Z_LINK] = sizes[k1::F_ZLINK];
  in.tag_rows[k1::P_LINK] = sizes[k1::F_PLINK];
  in.tag_rows[k1::ENERGY_DEV] = sizes[k1::F_EDEV];
  in.tag_rows[k1::ENERGY_TOTAL] = sizes[k1::F_ETOT];
  in.n_rows_mps = nrows - (opts.quadratic_objective ? sizes[k1::F_PLINK] : 0);
  return m.release();
}

// Column-major copy, stable in row order: LSD radix sort of the column keys
// carrying the entry index (CUB), then gathers.
void build_csc(xe_csr* m, cudaStream_t s) {
  if (m->has_csc) return;
  const int64_t nnz = m->info.nnz, nrows = m->info.n_rows, ncol = m->info.n_cols;
  DevBuf<int32_t> keys_out, row_of;
  DevBuf<int64_t> idx_in, idx_out;
  keys_out.alloc(static_cast<size_t>(std::max<int64_t>(1, nnz)));
  idx_in.alloc(static_cast<size_t>(std::max<int64_t>(1, nnz)));
  idx_out.alloc(static_cast<size_t>(std::max<int64_t>(1, nnz)));
  row_of.alloc(static_cast<size_t>(std::max<int64_t>(1, nnz)));
  k1::iota_kernel<<<grid_for(nnz), 256, 0, s>>>(idx_in.p, nnz);
  int end_bit = 1;
  while ((1ll << end_bit) <= ncol) ++end_bit;
  size_t tmp_bytes = 0;
  XE_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, m->col.p, keys_out.p, idx_in.p, idx_out.p, nnz, 0,
                                          end_bit, s));
  DevBuf<unsigned char> tmp;
  tmp.alloc(std::max<size_t>(1, tmp_bytes));
  XE_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, m->col.p, keys_out.p, idx_in.p, idx_out.p, nnz, 0,
                                          end_bit, s));
  m->col_ptr.alloc(static_cast<size_t>(ncol) + 1);
  m->crow.alloc(static_cast<size_t>(std::max<int64_t>(1, nnz)));
  m->cval.alloc(static_cast<size_t>(std::max<int64_t>(1, nnz)));
  k1::entry_row_kernel<<<grid_for(nrows), 256, 0, s>>>(m->row_ptr.p, nrows, row_of.p);
  k1::csc_rows_kernel<<<grid_for(nnz), 256, 0, s>>>(idx_out.p, row_of.p, m->crow.p, nnz);
  k1::csc_gather_kernel<<<grid_for(nnz), 256, 0, s>>>(idx_out.p, m->val.p, nullptr, m->cval.p, nnz);
  k1::col_ptr_kernel<<<grid_for(nnz + 1), 256, 0, s>>>(keys_out.p, nnz, ncol, m->col_ptr.p);
  XE_CUDA(cudaGetLastError());
  XE_CUDA(cudaStreamSynchronize(s));
  m->has_csc = true;
}

}  // namespace xe
