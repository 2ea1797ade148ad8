// SPDX-License-Identifier: Apache-2.0
//
// K2a v5 host side: shared-memory plan and launch of the streaming evaluator
// (eval_stream.cuh), the generalised interleaved layout (NW u64 words per
// bit row), and the exact re-score of the best-of-batch:
//
//   refine_best: the streaming kernel sums each candidate's objective per
//   timestep (a reassociation of objective_value's sequential loop,
//   model.cpp:392-427).  Every valid candidate whose reassociated objective
//   lies within 1e-12 relative of the batch minimum (the two orders differ by
//   at most ~#terms * 2^-53 relative, so the reference's argmin is among
//   them) is gathered, re-evaluated by the reference-order kernel
//   (eval_il.cu for T <= 64, eval_cube_v3.cuh above) and the first minimum of
//   the exact objective bits by global index wins — solver.cpp:57-61.  Skipped
//   when every objective term is dyadic (exact_fix_k >= 0): then both orders
//   give the same bits.

#include <cstdlib>
#include <algorithm>
#include <cstring>

#include "eval_stream.cuh"

namespace xe {

size_t eval_scratch_bytes(int device);
void reduce_best_launch(const uint64_t* key, const int64_t* idx, const int64_t* valid, int n, uint64_t* out,
                        cudaStream_t s);
void eval_cubes_device(const xe_problem* pr, const xe_model_opts& opts, const uint32_t* cubes, int64_t n,
                       double* obj, int64_t* peak, uint32_t* flags, uint32_t valid_mask, uint64_t* best3,
                       unsigned char* scratch, cudaStream_t stream);

namespace st {
namespace {

int align16(int x) { return (x + 15) & ~15; }

// canonical [n][2*D*T*W32] u32 -> interleaved [ceil(n/32)][2*D*T*NW][32] u64.
// One CTA per 32-candidate group, a 32x32 tile of u64 words in shared
// memory: coalesced reads along each cube, coalesced writes along the
// candidates.
__global__ void __launch_bounds__(256) to_il_kernel(const uint32_t* __restrict__ in, int64_t n, int rows, int W32,
                                                    int NW, uint64_t* __restrict__ out) {
  __shared__ uint64_t tile[32][33];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t g = blockIdx.x;
  const int K = rows * NW;
  for (int k0 = 0; k0 < K; k0 += 32) {
    for (int j = wid; j < 32; j += 8) {
      const int64_t c = g * 32 + j;
      const int k = k0 + lane;
      uint64_t v = 0;
      if (c < n && k < K) {
        const int r = k / NW, w = k - r * NW;
        const uint32_t* p = in + static_cast<size_t>(c) * rows * W32 + static_cast<size_t>(r) * W32 + 2 * w;
        v = p[0];
        if (2 * w + 1 < W32) v |= static_cast<uint64_t>(p[1]) << 32;
      }
      tile[j][lane] = v;
    }
    __syncthreads();
    for (int r = wid; r < 32; r += 8) {
      const int k = k0 + r;
      if (k < K) out[(static_cast<size_t>(g) * K + k) * 32 + lane] = tile[lane][r];
    }
    __syncthreads();
  }
}

// ---- refine: near-best collection, gather, exact minimum ------------------

__global__ void collect_near_kernel(const double* __restrict__ obj, const uint32_t* __restrict__ flags, int64_t n,
                                    uint32_t mask, const uint64_t* best3, int64_t* list, int* cnt, int cap) {
  const int64_t bi = static_cast<int64_t>(best3[1]);
  if (bi < 0) return;
  const double b = __longlong_as_double(static_cast<long long>(best3[0]));
  const uint64_t thr = static_cast<uint64_t>(__double_as_longlong(b + fabs(b) * 1e-12 + 1e-300));
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < n;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if ((flags[c] & mask) == 0 && static_cast<uint64_t>(__double_as_longlong(obj[c])) <= thr) {
      const int k = atomicAdd(cnt, 1);
      if (k < cap) list[k] = c;
    }
  }
}

// listed candidates -> compact canonical cubes [cap][rows*W32] u32 (unused slots zero)
__global__ void gather_il_kernel(const uint64_t* __restrict__ il, int rows, int NW, int W32, const int64_t* list,
                                 const int* cnt, int cap, uint32_t* out) {
  const int k = blockIdx.x;
  const int m = min(*cnt, cap);
  uint32_t* o = out + static_cast<size_t>(k) * rows * W32;
  if (k >= m) {
    for (int i = threadIdx.x; i < rows * W32; i += blockDim.x) o[i] = 0;
    return;
  }
  const int64_t c = list[k];
  const uint64_t* src = il + static_cast<size_t>(c / 32) * rows * NW * 32 + (c % 32);
  for (int i = threadIdx.x; i < rows * W32; i += blockDim.x) {
    const int r = i / W32, w32 = i - r * W32;
    const uint64_t v = src[(static_cast<size_t>(r) * NW + (w32 >> 1)) * 32];
    o[i] = static_cast<uint32_t>((w32 & 1) ? (v >> 32) : v);
  }
}

__global__ void gather_canon_kernel(const uint32_t* __restrict__ canon, int words, const int64_t* list, const int* cnt,
                                    int cap, uint32_t* out) {
  const int k = blockIdx.x;
  const int m = min(*cnt, cap);
  uint32_t* o = out + static_cast<size_t>(k) * words;
  const uint32_t* src = k < m ? canon + static_cast<size_t>(list[k]) * words : nullptr;
  for (int i = threadIdx.x; i < words; i += blockDim.x) o[i] = src ? src[i] : 0u;
}

__global__ void il_to_canon_kernel(const uint64_t* __restrict__ il, int rows, int NW, int W32, int64_t first,
                                   uint32_t* out) {
  const int64_t c = first + blockIdx.x;
  uint32_t* o = out + static_cast<size_t>(blockIdx.x) * rows * W32;
  const uint64_t* src = il + static_cast<size_t>(c / 32) * rows * NW * 32 + (c % 32);
  for (int i = threadIdx.x; i < rows * W32; i += blockDim.x) {
    const int r = i / W32, w32 = i - r * W32;
    const uint64_t v = src[(static_cast<size_t>(r) * NW + (w32 >> 1)) * 32];
    o[i] = static_cast<uint32_t>((w32 & 1) ? (v >> 32) : v);
  }
}

// exact minimum over the gathered candidates: (exact objective bits, global index)
__global__ void final_best_kernel(const int64_t* list, const int* cnt, int cap, const double* xobj,
                                  const uint32_t* xflags, uint32_t mask, uint64_t* best3) {
  __shared__ uint64_t sk[256];
  __shared__ int64_t si[256];
  const int total = *cnt;
  if (static_cast<int64_t>(best3[1]) < 0) return;  // nothing valid
  if (total > cap) {                                // too many near-ties: the caller re-runs exactly
    if (threadIdx.x == 0) best3[1] = static_cast<uint64_t>(-2ll);
    return;
  }
  uint64_t bk = ~0ull;
  int64_t bi = -1;
  for (int k = threadIdx.x; k < total; k += blockDim.x) {
    if (xflags[k] & mask) continue;
    const uint64_t key = static_cast<uint64_t>(__double_as_longlong(xobj[k]));
    if (key < bk || (key == bk && list[k] < bi)) {
      bk = key;
      bi = list[k];
    }
  }
  sk[threadIdx.x] = bk;
  si[threadIdx.x] = bi;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < blockDim.x; ++i)
      if (si[i] >= 0 && (sk[i] < bk || (sk[i] == bk && (bi < 0 || si[i] < bi)))) {
        bk = sk[i];
        bi = si[i];
      }
    if (bi >= 0) {
      best3[0] = bk;
      best3[1] = static_cast<uint64_t>(bi);
    }
  }
}

}  // namespace
}  // namespace st

using namespace st;

int il_words(int T) { return (T + 63) / 64; }

bool il_layout_ok(const xe_problem* pr) { return pr->h.T <= 256 && pr->h.D <= 8; }

size_t il_bytes(int D, int T, int64_t n) {
  return static_cast<size_t>((n + 31) / 32) * 32 * 2 * D * T * il_words(T) * 8;
}

void cubes_to_il_device(const xe_problem* pr, const uint32_t* cubes, int64_t n, uint64_t* il, cudaStream_t s) {
  const HostProblem& h = pr->h;
  if (!il_layout_ok(pr)) fail(XE_ERR_TOO_LARGE, "interleaved cubes need T <= 256 and D <= 8");
  const int64_t ngroups = (n + 31) / 32;
  if (ngroups == 0) return;
  to_il_kernel<<<static_cast<unsigned>(ngroups), 256, 0, s>>>(cubes, n, 2 * h.D * h.T, (h.T + 31) / 32,
                                                             il_words(h.T), il);
  XE_CUDA(cudaGetLastError());
}

void il_to_canon_device(const xe_problem* pr, const uint64_t* il, int64_t first, int64_t n, uint32_t* canon,
                        cudaStream_t s) {
  const HostProblem& h = pr->h;
  if (n <= 0) return;
  il_to_canon_kernel<<<static_cast<unsigned>(n), 128, 0, s>>>(il, 2 * h.D * h.T, il_words(h.T), (h.T + 31) / 32,
                                                              first, canon);
  XE_CUDA(cudaGetLastError());
}

// XE_STREAM_WIDE=0 keeps the 8-warp plan everywhere (A/B switch)
static bool wide_disabled() {
  const char* e = std::getenv("XE_STREAM_WIDE");
  return e && e[0] == '0';
}

bool stream_supported(const xe_problem* pr, const xe_model_opts& opts) {
  const HostProblem& h = pr->h;
  if (opts.use_energy && h.has_energy) return false;  // energy terms/rows: the exact kernels
  if (pr->exact_objective) return false;               // reference order requested
  if (!il_layout_ok(pr) || h.E >= 65536) return false;
  return static_cast<size_t>(h.E) * h.D * h.D * 8 <= 64 * 1024;  // copy table in shared memory
}

// True when the reassociated objective equals the reference's bits.
bool stream_objective_exact(const xe_problem* pr) { return pr->fix_k_plain >= 0; }

int eval_stream_device(const xe_problem* pr, const xe_model_opts& opts, const uint64_t* il, int64_t n, double* obj,
                       int64_t* peak, uint32_t* flags, uint32_t valid_mask, uint64_t* best3, unsigned char* scratch,
                       cudaStream_t stream) {
  const HostProblem& h = pr->h;
  if (!h.missing_link.empty() && h.D > 1) fail(XE_ERR_MISSING_LINK, h.missing_link);
  if (!stream_supported(pr, opts)) fail(XE_ERR_TOO_LARGE, "streaming evaluator: unsupported problem");
  StArgs a{};
  a.P = pr->view(false);
  a.il = il;
  a.n = n;
  a.obj = obj;
  a.peak = peak;
  a.flags = flags;
  a.strict = opts.strict_free ? 1 : 0;
  a.valid_mask = valid_mask;
  int64_t total_mass = 0;
  for (int64_t m : h.mass) total_mass += m;
  const bool m32 = total_mass < (int64_t{1} << 30);  // every U is at most twice the save-all total
  const int msz = m32 ? 4 : 8;
  const int NW = il_words(h.T);
  const int maxd = h.D <= 4 ? h.D : 8;
  int nsm = 0, smem_limit = 0;
  XE_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, pr->device));
  XE_CUDA(cudaDeviceGetAttribute(&smem_limit, cudaDevAttrMaxSharedMemoryPerBlockOptin, pr->device));
  // the wide plan (one 24-warp CTA per SM, 11-bit mass tables): one-word
  // rows of 34..64 operators with int32 masses and D in 2..4, when its
  // shared-memory plan fits; else the 8-warp plan
  const int nch = (h.T + 10) / 11;
  auto plan = [&](bool wide) {
    int off = 0;
    auto take = [&](int bytes) {
      int o = off;
      off = align16(off + bytes);
      return o;
    };
    const int nbl_bytes = (h.T - 64 * (NW - 1) + 7) / 8;  // row bytes of the last word
    take(wide ? nch * 2048 * msz : (8 * (NW - 1) + (nbl_bytes <= 4 ? 4 : nbl_bytes <= 6 ? 6 : 8)) * 256 * msz);
    a.off_mass = take(msz * h.T);
    a.off_pmask = take(8 * h.T * NW);
    a.off_cons = take(8 * h.T * NW);
    a.off_c = take(8 * h.D * h.T);
    a.off_w = take(8 * std::max(1, h.E * h.D * h.D));
    a.off_inl = take(4 * std::max(1, h.E));
    a.off_inptr = take(4 * (h.T + 1));
    a.off_inedge = take(4 * std::max(1, h.E));
    a.off_src = take(4 * std::max(1, h.E));
    a.off_dst = take(4 * std::max(1, h.E));
    a.off_warp = off;
    // per warp: queue | fl[32] | cnt[32] | pk[32][maxd] | slow[32] | park[32]
    const int pf_words = maxd * NW <= 4 ? maxd * NW : 1;  // Park::Rn / Sn
    const int park_bytes = 8 + 16 + 8 * maxd * NW + 2 * 8 * pf_words + msz * maxd + 4;
    const int park_sz = (park_bytes + 7) & ~7;
    a.warp_bytes = align16(static_cast<int>(sizeof(Job)) * qcap(NW) + 4 * 32 + 4 * 32 + msz * 32 * maxd +
                           8 * 32 + 32 * park_sz + 64);
    a.smem_bytes = off + (wide ? kWideWarps : kWarps) * a.warp_bytes;
  };
  bool wide = NW == 1 && m32 && h.D >= 2 && h.D <= 4 && nch >= 4 && !wide_disabled();
  if (wide) {
    plan(true);
    if (a.smem_bytes > smem_limit) wide = false;
  }
  if (!wide) plan(false);
  const int warps = wide ? kWideWarps : kWarps;
  if (a.smem_bytes > smem_limit) fail(XE_ERR_TOO_LARGE, "streaming evaluator: shared-memory plan too large");
  const size_t nw_max = static_cast<size_t>(nsm) * 8 * cube::kWarps;  // eval_scratch_bytes layout
  a.wbest_key = reinterpret_cast<uint64_t*>(scratch);
  a.wbest_idx = reinterpret_cast<int64_t*>(scratch + nw_max * 8);
  a.wvalid = reinterpret_cast<int64_t*>(scratch + nw_max * 16);
  int grid = 0;
  if (n > 0) {
    const int tl = h.T - 64 * (NW - 1);
    const int nbl = (tl + 7) / 8;
    switch (NW) {
      case 1: grid = launch_stream<1>(a, m32, wide ? nch : nbl, stream, nsm, wide); break;
      case 2: grid = launch_stream<2>(a, m32, wide ? nch : nbl, stream, nsm, wide); break;
      case 3: grid = launch_stream<3>(a, m32, wide ? nch : nbl, stream, nsm, wide); break;
      default: grid = launch_stream<4>(a, m32, nbl, stream, nsm, false); break;
    }
    if (static_cast<size_t>(grid) * warps > nw_max) fail(XE_ERR_ARG, "evaluator scratch too small");
  }
  if (best3) {
    if (n > 0) {
      reduce_best_launch(a.wbest_key, a.wbest_idx, a.wvalid, grid * warps, best3, stream);
    } else {
      const uint64_t none[3] = {~0ull, ~0ull, 0ull};
      XE_CUDA(cudaMemcpyAsync(best3, none, sizeof none, cudaMemcpyHostToDevice, stream));
    }
  }
  return grid;
}

void eval_il_device(const xe_problem* pr, const xe_model_opts& opts, const uint64_t* il, int64_t n, double* obj,
                    int64_t* peak, uint32_t* flags, uint32_t valid_mask, uint64_t* best3, unsigned char* scratch,
                    cudaStream_t stream);
bool il_supported(const xe_problem* pr);

// Re-scores the near-best candidates of one evaluated batch in the
// reference's summation order and overwrites best3 with the exact first
// minimum (index -2: more near-ties than kRefineCap, the caller falls back to
// the exact evaluator).  src_il / src_canon: the batch (one of them).
void refine_best_device(const xe_problem* pr, const xe_model_opts& opts, const uint64_t* src_il,
                        const uint32_t* src_canon, int64_t n, const double* obj, const uint32_t* flags,
                        uint32_t valid_mask, uint64_t* best3, RefineBuf& rb, unsigned char* scratch,
                        cudaStream_t s) {
  if (stream_objective_exact(pr) || n == 0) return;
  const HostProblem& h = pr->h;
  const int cap = kRefineCap;
  const int W32 = (h.T + 31) / 32, rows = 2 * h.D * h.T, words = rows * W32;
  rb.list.reserve(cap);
  rb.cnt.reserve(1);
  rb.canon.reserve(static_cast<size_t>(cap) * words);
  rb.obj.reserve(cap);
  rb.flags.reserve(cap);
  XE_CUDA(cudaMemsetAsync(rb.cnt.p, 0, sizeof(int), s));
  const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 8));
  collect_near_kernel<<<blocks, 256, 0, s>>>(obj, flags, n, valid_mask, best3, rb.list.p, rb.cnt.p, cap);
  XE_CUDA(cudaGetLastError());
  if (src_il)
    gather_il_kernel<<<cap, 128, 0, s>>>(src_il, rows, il_words(h.T), W32, rb.list.p, rb.cnt.p, cap, rb.canon.p);
  else
    gather_canon_kernel<<<cap, 128, 0, s>>>(src_canon, words, rb.list.p, rb.cnt.p, cap, rb.canon.p);
  XE_CUDA(cudaGetLastError());
  // the reference-order evaluation of the gathered cubes
  if (il_supported(pr)) {
    rb.il.reserve(il_bytes(h.D, h.T, cap) / 8);
    cubes_to_il_device(pr, rb.canon.p, cap, rb.il.p, s);
    eval_il_device(pr, opts, rb.il.p, cap, rb.obj.p, nullptr, rb.flags.p, valid_mask, nullptr, scratch, s);
  } else {
    eval_cubes_device(pr, opts, rb.canon.p, cap, rb.obj.p, nullptr, rb.flags.p, valid_mask, nullptr, scratch, s);
  }
  final_best_kernel<<<1, 256, 0, s>>>(rb.list.p, rb.cnt.p, cap, rb.obj.p, rb.flags.p, valid_mask, best3);
  XE_CUDA(cudaGetLastError());
}

}  // namespace xe
