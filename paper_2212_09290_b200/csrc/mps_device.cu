// SPDX-License-Identifier: Apache-2.0
//
// write_mps (proj/src/mps_io.cpp:109-199) emitted on the GPU from the
// device model.  Each section is a sequence of items of at most a few lines
// (a row, a column head = marker + OBJ entry, one CSC entry, a right-hand
// side, a bound); one pass counts each item's bytes, a scan places them, a
// second pass formats a block's items into shared memory and stores the
// block's contiguous byte range with coalesced stores.  The text stays in HBM
// until the caller's copy call downloads it into the caller's buffer.  Numbers follow format_number (mps_io.cpp:14-27): integral
// |v| < 1e15 print as integers on the device; the few non-integral values a
// model can hold (costs, copy costs, energy terms and limits) are formatted
// once on the host with the shortest round-trip rule and looked up by their
// bits.  A value missing from that table (it cannot happen for models K1
// builds) makes the caller fall back to the host writer.  QUADOBJ models
// drop the P columns and P_LINK rows and add the QUADOBJ section, one item
// per (t, e, ds, dc) with a nonzero copy cost.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include <thrust/execution_policy.h>
#include <thrust/scan.h>

#include "csr.hpp"

namespace xe {
std::string format_number(double v);  // mps_writer.cpp
namespace mpsd {

__constant__ char kTagC[14][13] = {"EQ7",     "EQ8",     "EQ9",    "EQ10",   "EQ11",       "EQ12",        "EQ13",
                                   "EQ14",    "EQ16_LO", "EQ16_HI", "Z_LINK", "P_LINK", "ENERGY_DEV", "ENERGY_TOTAL"};

struct Args {
  int64_t D, T, E, n_rows, n_cols, firstU;
  int64_t ncol_out;  // columns written: all, or up to the first P column (QUADOBJ models)
  int quad;          // QUADOBJ model: P columns and P_LINK rows dropped, a QUADOBJ section added
  const int32_t *src, *dst;
  const double* w;   // [E][D][D] copy costs
  const int8_t* sense;
  const uint8_t *tag, *present, *kind;
  const int32_t *ordinal, *crow;
  const int64_t* col_ptr;
  const double *cval, *rhs, *obj, *ub;
  // non-integral numbers: sorted keys (double bits) and their strings
  const uint64_t* nkeys;
  const int32_t* noff;  // [n + 1] into npool
  const char* npool;
  int nnum;
  int* missing;
};

// byte writer: counts when p is null
struct W {
  char* p;
  int64_t n;
  __device__ void c(char ch) {
    if (p) p[n] = ch;
    ++n;
  }
  __device__ void s(const char* z) {
    for (; *z; ++z) c(*z);
  }
  __device__ void u(uint64_t v) {
    char b[24];
    int k = 0;
    do {
      b[k++] = static_cast<char>('0' + v % 10);
      v /= 10;
    } while (v);
    while (k) c(b[--k]);
  }
  __device__ void i(int64_t v) {
    if (v < 0) {
      c('-');
      u(static_cast<uint64_t>(-v));
    } else {
      u(static_cast<uint64_t>(v));
    }
  }
};

__device__ void num(W& w, const Args& a, double v) {
  if (v == 0.0) {
    w.c('0');
    return;
  }
  if (isfinite(v) && v == floor(v) && fabs(v) < 1e15) {  // "%.0f"
    w.i(static_cast<int64_t>(v));
    return;
  }
  const uint64_t key = static_cast<uint64_t>(__double_as_longlong(v));
  int lo = 0, hi = a.nnum;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a.nkeys[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  if (lo < a.nnum && a.nkeys[lo] == key) {
    for (int k = a.noff[lo]; k < a.noff[lo + 1]; ++k) w.c(a.npool[k]);
  } else {
    atomicExch(a.missing, 1);
    w.c('?');
  }
}

// var_name of a closed-form column (mps_io.cpp:29-43)
__device__ void col_name(W& w, const Args& a, int64_t j) {
  const int64_t T = a.T, D = a.D, E = a.E, FE = a.E + a.T;
  const int64_t DT2 = D * T * T, DTF = D * T * FE;
  auto tri = [&](char f, int64_t x, int64_t y, int64_t z) {
    w.c(f);
    w.c('_');
    w.u(static_cast<uint64_t>(x));
    w.c('_');
    w.u(static_cast<uint64_t>(y));
    w.c('_');
    w.u(static_cast<uint64_t>(z));
  };
  if (j < 3 * DT2) {
    const char f = j < DT2 ? 'R' : j < 2 * DT2 ? 'S' : 'Z';
    const int64_t r = j % DT2;
    tri(f, r / (T * T), r / T % T, r % T);
    return;
  }
  j -= 3 * DT2;
  if (j < DTF) {
    tri('F', j / (T * FE), j / FE % T, j % FE);
    return;
  }
  j -= DTF;
  if (j < DT2) {
    tri('U', j / (T * T), j / T % T, j % T);
    return;
  }
  j -= DT2;
  const int64_t dm1 = D - 1, t = j / (E * D * dm1);
  int64_t rem = j % (E * D * dm1);
  const int64_t e = rem / (D * dm1);
  rem %= D * dm1;
  const int64_t ds = rem / dm1;
  int64_t dc = rem % dm1;
  if (dc >= ds) ++dc;
  tri('P', t, e, ds);
  w.c('_');
  w.u(static_cast<uint64_t>(dc));
}

__device__ void row_name(W& w, const Args& a, int64_t r) {
  w.s(kTagC[a.tag[r]]);
  w.c('_');
  w.i(a.ordinal[r]);
}

constexpr uint8_t kPLink = 11;

// section items: 0 ROWS (row r), 1 COLUMNS (column heads and entries), 2 RHS
// (row r), 3 BOUNDS (column j), 4 QUADOBJ ((t, e, ds, dc) in loop order)
template <int SEC>
__device__ void item(W& w, const Args& a, int64_t k) {
  if (SEC == 0) {
    if (a.quad && a.tag[k] == kPLink) return;
    w.c(' ');
    w.c(static_cast<char>(a.sense[k]));
    w.c(' ');
    row_name(w, a, k);
    w.c('\n');
  } else if (SEC == 1) {
    // column j's head sits at col_ptr[j] + j, its entries follow
    int64_t lo = 0, hi = a.ncol_out - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (a.col_ptr[mid] + mid <= k) lo = mid;
      else hi = mid - 1;
    }
    const int64_t j = lo, head = a.col_ptr[j] + j;
    if (k == head) {
      if (j == 0 && a.firstU > 0) w.s("    MARK  'MARKER'  'INTORG'\n");
      if (j == a.firstU && j > 0) w.s("    MARK  'MARKER'  'INTEND'\n");
      if (a.present[j]) {
        w.s("    ");
        col_name(w, a, j);
        w.s("  OBJ  ");
        num(w, a, a.obj[j]);
        w.c('\n');
      }
    } else {
      const int64_t q = a.col_ptr[j] + (k - head - 1);
      if (a.quad && a.tag[a.crow[q]] == kPLink) return;
      w.s("    ");
      col_name(w, a, j);
      w.s("  ");
      row_name(w, a, a.crow[q]);
      w.s("  ");
      num(w, a, a.cval[q]);
      w.c('\n');
    }
  } else if (SEC == 2) {
    const double v = a.rhs[k];
    if (v == 0.0 || (a.quad && a.tag[k] == kPLink)) return;
    w.s("    RHS  ");
    row_name(w, a, k);
    w.s("  ");
    num(w, a, v);
    w.c('\n');
  } else if (SEC == 4) {
    const int64_t D = a.D, T = a.T, E = a.E;
    const int64_t dc = k % D, ds = k / D % D, e = k / (D * D) % E, t = k / (D * D * E);
    if (ds == dc) return;
    const double wv = a.w[(e * D + ds) * D + dc];
    if (wv == 0.0) return;
    w.s("    ");
    col_name(w, a, (dc * T + t) * T + a.dst[e]);
    w.s("  ");
    col_name(w, a, 2 * D * T * T + (ds * T + t) * T + a.src[e]);
    w.s("  ");
    num(w, a, wv);
    w.c('\n');
  } else {
    const uint8_t kd = a.kind[k];
    if (kd == 0) {
      w.s(" FX BND ");
      col_name(w, a, k);
      w.s(" 0\n");
    } else if (kd == 1) {
      w.s(" BV BND ");
      col_name(w, a, k);
      w.c('\n');
    } else {
      w.s(" UP BND ");
      col_name(w, a, k);
      w.c(' ');
      if (kd == 2) num(w, a, a.ub[k]);
      else w.c('1');
      w.c('\n');
    }
  }
}

template <int SEC>
__global__ void size_kernel(Args a, int64_t n, int64_t* len) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    W w{nullptr, 0};
    item<SEC>(w, a, k);
    len[k] = w.n;
  }
}

constexpr int kBlock = 256, kStage = kBlock * 128;  // bytes staged per block

// one block per kBlock consecutive items: format into shared memory, then
// store the block's byte range [off[k0], off[k1]) with consecutive threads on
// consecutive bytes; a block whose range exceeds the stage writes directly
template <int SEC>
__global__ void __launch_bounds__(kBlock) write_kernel(Args a, int64_t n, const int64_t* off, char* out) {
  __shared__ char stage[kStage];
  for (int64_t k0 = blockIdx.x * static_cast<int64_t>(kBlock); k0 < n; k0 += static_cast<int64_t>(gridDim.x) * kBlock) {
    const int64_t k1 = k0 + kBlock < n ? k0 + kBlock : n;
    const int64_t base = off[k0], bytes = off[k1] - base;
    const int64_t k = k0 + threadIdx.x;
    if (bytes <= kStage) {
      if (k < k1) {
        W w{stage + (off[k] - base), 0};
        item<SEC>(w, a, k);
      }
      __syncthreads();
      for (int64_t b = threadIdx.x; b < bytes; b += kBlock) out[base + b] = stage[b];
      __syncthreads();
    } else if (k < k1) {
      W w{out + off[k], 0};
      item<SEC>(w, a, k);
    }
  }
}

inline unsigned grid_for(int64_t n) {
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((n + kBlock - 1) / kBlock, 148 * 16)));
}

}  // namespace mpsd

// Leaves the text in m->mps_dev.  Returns false when the device writer
// cannot serve the model (a non-integral number outside the host-formatted
// table): the caller then uses the host writer.
bool mps_text_device(xe_csr* m) {
  using namespace mpsd;
  const bool quad = m->opts.quadratic_objective != 0;
  const xe_csr_info& in = m->info;
  const HostProblem& h = m->prob->h;
  cudaStream_t s = m->stream;
  build_csc(m, s);
  // the non-integral values a K1 model can hold: costs (+ alpha q), copy
  // costs, energy q, limits and the total-limit right-hand side
  std::vector<double> vals;
  auto add = [&](double v) {
    if (!(std::isfinite(v) && v == std::floor(v) && std::fabs(v) < 1e15)) vals.push_back(v);
  };
  for (double v : h.cost) add(v);
  for (double v : h.w) add(v);
  if (h.has_energy) {
    for (size_t i = 0; i < h.q.size(); ++i) {
      add(h.q[i]);
      const double aq = h.alpha * h.q[i];  // K1 adds the precomputed product
      add(aq);
      add(h.cost[i] + aq);
    }
    for (double v : h.lim) add(v);
    add(h.total_limit - h.board);
  }
  std::vector<uint64_t> keys;
  for (double v : vals) {
    uint64_t k;
    std::memcpy(&k, &v, 8);
    keys.push_back(k);
  }
  std::sort(keys.begin(), keys.end());
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  std::vector<int32_t> noff(1, 0);
  std::string pool;
  for (uint64_t k : keys) {
    double v;
    std::memcpy(&v, &k, 8);
    pool += format_number(v);
    noff.push_back(static_cast<int32_t>(pool.size()));
  }
  if (keys.empty()) keys.push_back(0);  // never matched: nnum stays the real count
  std::vector<char> pool_v(pool.begin(), pool.end());
  pool_v.push_back(0);
  DevBuf<uint64_t> dkeys;
  DevBuf<int32_t> doff;
  DevBuf<char> dpool;
  DevBuf<int> missing;
  dkeys.upload(keys, s);
  doff.upload(noff, s);
  dpool.upload(pool_v, s);
  missing.alloc(1);
  XE_CUDA(cudaMemsetAsync(missing.p, 0, sizeof(int), s));
  Args a{};
  a.D = in.D;
  a.T = in.T;
  a.E = in.E;
  a.n_rows = in.n_rows;
  a.n_cols = in.n_cols;
  a.firstU = 3ll * in.D * in.T * in.T + static_cast<int64_t>(in.D) * in.T * (in.E + in.T);
  const int64_t firstP = a.firstU + static_cast<int64_t>(in.D) * in.T * in.T;
  a.quad = quad ? 1 : 0;
  a.ncol_out = quad ? std::min<int64_t>(firstP, in.n_cols) : in.n_cols;
  a.src = m->prob->dev.src;
  a.dst = m->prob->dev.dst;
  a.w = m->prob->d_w.p;
  a.sense = m->sense.p;
  a.tag = m->tag.p;
  a.present = m->present.p;
  a.kind = m->kind.p;
  a.ordinal = m->ordinal.p;
  a.crow = m->crow.p;
  a.col_ptr = m->col_ptr.p;
  a.cval = m->cval.p;
  a.rhs = m->rhs.p;
  a.obj = m->obj.p;
  a.ub = m->ub.p;
  a.nkeys = dkeys.p;
  a.noff = doff.p;
  a.npool = dpool.p;
  a.nnum = static_cast<int>(noff.size()) - 1;
  a.missing = missing.p;
  // column items: heads and entries of the columns written
  int64_t col_items = in.n_cols + in.nnz;
  if (a.ncol_out < in.n_cols) {
    int64_t e_out = 0;
    XE_CUDA(cudaMemcpyAsync(&e_out, m->col_ptr.p + a.ncol_out, 8, cudaMemcpyDeviceToHost, s));
    XE_CUDA(cudaStreamSynchronize(s));
    col_items = a.ncol_out + e_out;
  }
  bool any_quad = false;  // QUADOBJ lines exist (a nonzero cross-device copy cost)
  if (quad)
    for (int e = 0; e < h.E && !any_quad; ++e)
      for (int x = 0; x < h.D && !any_quad; ++x)
        for (int y = 0; y < h.D; ++y)
          if (x != y && h.w[(static_cast<size_t>(e) * h.D + x) * h.D + y] != 0.0) {
            any_quad = true;
            break;
          }
  constexpr int kSec = 5;
  const int64_t ns[kSec] = {in.n_rows, col_items, in.n_rows, a.ncol_out,
                            any_quad ? static_cast<int64_t>(in.T) * in.E * in.D * in.D : 0};
  // the INTEND that closes a model without continuous columns follows the
  // last column item
  const std::string sec_tail[kSec] = {
      "", a.firstU == a.ncol_out && a.firstU > 0 ? "    MARK  'MARKER'  'INTEND'\n" : "", "", "", ""};
  const char* const head[kSec] = {"NAME XENGINE\nROWS\n N OBJ\n", "COLUMNS\n", "RHS\n", "BOUNDS\n",
                                  any_quad ? "QUADOBJ\n" : ""};
  // per section: lengths -> in-place inclusive scan -> offsets
  std::vector<DevBuf<int64_t>> off(kSec);
  std::vector<int64_t> bytes(kSec, 0);
  for (int sec = 0; sec < kSec; ++sec) {
    const int64_t n = ns[sec];
    off[static_cast<size_t>(sec)].alloc(static_cast<size_t>(n) + 1);
    int64_t* o = off[static_cast<size_t>(sec)].p;
    XE_CUDA(cudaMemsetAsync(o, 0, 8, s));
    if (n == 0) continue;
    switch (sec) {
      case 0: size_kernel<0><<<grid_for(n), kBlock, 0, s>>>(a, n, o + 1); break;
      case 1: size_kernel<1><<<grid_for(n), kBlock, 0, s>>>(a, n, o + 1); break;
      case 2: size_kernel<2><<<grid_for(n), kBlock, 0, s>>>(a, n, o + 1); break;
      case 3: size_kernel<3><<<grid_for(n), kBlock, 0, s>>>(a, n, o + 1); break;
      default: size_kernel<4><<<grid_for(n), kBlock, 0, s>>>(a, n, o + 1); break;
    }
    XE_CUDA(cudaGetLastError());
    thrust::inclusive_scan(thrust::cuda::par.on(s), o + 1, o + 1 + n, o + 1);
    XE_CUDA(cudaMemcpyAsync(&bytes[static_cast<size_t>(sec)], o + n, 8, cudaMemcpyDeviceToHost, s));
  }
  int miss = 0;
  XE_CUDA(cudaMemcpyAsync(&miss, missing.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  XE_CUDA(cudaStreamSynchronize(s));
  if (miss) return false;
  const std::string tail = "ENDATA\n";
  size_t total = tail.size();
  for (int sec = 0; sec < kSec; ++sec)
    total += std::strlen(head[sec]) + static_cast<size_t>(bytes[static_cast<size_t>(sec)]) + sec_tail[sec].size();
  DevBuf<char>& text = m->mps_dev;
  text.alloc(std::max<size_t>(1, total));
  m->mps_dev_len = total;
  size_t at = 0;
  for (int sec = 0; sec < kSec; ++sec) {
    const size_t hl = std::strlen(head[sec]);
    if (hl) XE_CUDA(cudaMemcpyAsync(text.p + at, head[sec], hl, cudaMemcpyHostToDevice, s));
    at += hl;
    char* base = text.p + at;
    const int64_t n = ns[sec];
    const int64_t* o = off[static_cast<size_t>(sec)].p;
    if (n > 0) {
      switch (sec) {
        case 0: write_kernel<0><<<grid_for(n), kBlock, 0, s>>>(a, n, o, base); break;
        case 1: write_kernel<1><<<grid_for(n), kBlock, 0, s>>>(a, n, o, base); break;
        case 2: write_kernel<2><<<grid_for(n), kBlock, 0, s>>>(a, n, o, base); break;
        case 3: write_kernel<3><<<grid_for(n), kBlock, 0, s>>>(a, n, o, base); break;
        default: write_kernel<4><<<grid_for(n), kBlock, 0, s>>>(a, n, o, base); break;
      }
      XE_CUDA(cudaGetLastError());
    }
    at += static_cast<size_t>(bytes[static_cast<size_t>(sec)]);
    if (!sec_tail[sec].empty()) {
      XE_CUDA(cudaMemcpyAsync(text.p + at, sec_tail[sec].data(), sec_tail[sec].size(), cudaMemcpyHostToDevice, s));
      at += sec_tail[sec].size();
    }
  }
  XE_CUDA(cudaMemcpyAsync(text.p + at, tail.data(), tail.size(), cudaMemcpyHostToDevice, s));
  XE_CUDA(cudaStreamSynchronize(s));
  return true;
}

}  // namespace xe
