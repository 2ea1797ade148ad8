// SPDX-License-Identifier: Apache-2.0
//
// K2a host launcher: shared-memory plan, grid sizing, best-of-batch
// reduction.  The kernel is in eval_cube_kernel.cuh.
#include <cstring>

#include "eval_cube_v3.cuh"

namespace xe {
namespace cube {
int launch_nw1(const EvalArgs& a, int grid, int smem, cudaStream_t s, int nsm);
int launch_nw2(const EvalArgs& a, int grid, int smem, cudaStream_t s, int nsm);
int launch_nw3(const EvalArgs& a, int grid, int smem, cudaStream_t s, int nsm);
int launch_nw4(const EvalArgs& a, int grid, int smem, cudaStream_t s, int nsm);
namespace {
__global__ void reduce_best_kernel(const uint64_t* key, const int64_t* idx, const int64_t* valid,
                                   int n, uint64_t* out_key, int64_t* out_idx, int64_t* out_valid) {
  uint64_t bk = ~0ull;
  int64_t bi = -1, nv = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    nv += valid[i];
    if (idx[i] >= 0 && (key[i] < bk || (key[i] == bk && (bi < 0 || idx[i] < bi)))) {
      bk = key[i];
      bi = idx[i];
    }
  }
  __shared__ uint64_t sk[256];
  __shared__ int64_t si[256], sv[256];
  sk[threadIdx.x] = bk;
  si[threadIdx.x] = bi;
  sv[threadIdx.x] = nv;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < blockDim.x; ++i) {
      nv += sv[i];
      if (si[i] >= 0 && (sk[i] < bk || (sk[i] == bk && (bi < 0 || si[i] < bi)))) {
        bk = sk[i];
        bi = si[i];
      }
    }
    *out_key = bk;
    *out_idx = bi;
    *out_valid = nv;
  }
}

int align16(int x) { return (x + 15) & ~15; }

}  // namespace
}  // namespace cube

using namespace cube;

// Lexicographic (objective bits, index) minimum over per-warp partials.
void reduce_best_launch(const uint64_t* key, const int64_t* idx, const int64_t* valid, int n, uint64_t* out,
                        cudaStream_t s) {
  reduce_best_kernel<<<1, 256, 0, s>>>(key, idx, valid, n, out, reinterpret_cast<int64_t*>(out + 1),
                                       reinterpret_cast<int64_t*>(out + 2));
  XE_CUDA(cudaGetLastError());
}

// Host launcher: plans shared memory, launches the evaluator and the
// best-of-batch reduction into best3 (device: objective bits, index, valid
// count), all on `stream`, without synchronising.
size_t eval_scratch_bytes(int device) {
  int nsm = 0;
  XE_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
  return static_cast<size_t>(nsm) * 8 * kWarps * 24 + 64;
}

void eval_cubes_device(const xe_problem* pr, const xe_model_opts& opts, const uint32_t* cubes,
                       int64_t n, double* obj, int64_t* peak, uint32_t* flags, uint32_t valid_mask,
                       uint64_t* best3, unsigned char* scratch, cudaStream_t stream) {
  const HostProblem& h = pr->h;
  if (!h.missing_link.empty() && h.D > 1) fail(XE_ERR_MISSING_LINK, h.missing_link);
  if (h.T > 256) fail(XE_ERR_TOO_LARGE, "dense cube evaluation supports T <= 256 (use placements)");
  if (h.D > 8) fail(XE_ERR_TOO_LARGE, "dense cube evaluation supports D <= 8");
  EvalArgs a{};
  a.P = pr->view(opts.use_energy != 0);
  const DevProblem& P = a.P;
  if (P.n_table > 65535) fail(XE_ERR_TOO_LARGE, "objective term table exceeds 16-bit indices");
  a.cubes = cubes;
  a.n = n;
  a.obj = obj;
  a.peak = peak;
  a.flags = flags;
  a.strict = opts.strict_free ? 1 : 0;
  a.energy = (opts.use_energy && h.has_energy) ? 1 : 0;
  a.valid_mask = valid_mask;
  a.cube_words = static_cast<uint32_t>(2 * P.D * P.T * P.W32);
  const int cube_bytes = static_cast<int>(a.cube_words * 4);
  a.use_bulk = (cube_bytes % 16 == 0) && (reinterpret_cast<uintptr_t>(cubes) % 16 == 0);
  // double-buffer small cubes; a large cube (configs 3-4: 17-22 KB) single-buffered,
  // so twice as many warps fit the shared memory plan
  a.stages = cube_bytes > 8192 ? 1 : 2;

  // shared-memory plan
  int off = 0;
  auto take = [&](int bytes) {
    int o = off;
    off = align16(off + bytes);
    return o;
  };
  a.off_mass = take(8 * P.T);
  a.off_pmask = take(8 * P.T * P.NW);
  a.off_cons = take(8 * P.T * P.NW);
  a.off_mtab = take(8 * 256 * P.NB);
  a.off_tab = take(8 * P.n_table);
  a.off_inptr = take(4 * (P.T + 1));
  a.off_inedge = take(4 * std::max(1, P.E));
  a.off_src = take(4 * std::max(1, P.E));
  a.off_dst = take(4 * std::max(1, P.E));
  a.off_ebad = take(8 * P.D * P.NW);
  a.off_q = take(a.energy && P.has_total ? 8 * P.D * P.T : 8);
  a.off_warp = off;
  const bool exact = P.fix_k >= 0;
  // serial term-list capacity: covers placements plus a few recomputes and
  // copies; larger candidates take the (slow, exact) one-lane path
  int cap = exact ? 0 : ((std::min(1024, 2 * P.T + 32) + 7) & ~7);
  int cap2 = (exact || !a.energy) ? 0 : cap;
  // per-warp: stages | barriers | term lists (R+copy) | energy terms | slot results
  int w = 0;
  a.off_w_stage = w;
  w = align16(w + a.stages * cube_bytes);
  a.off_w_bar = w;
  w = align16(w + 8 * a.stages);
  a.off_w_terms = w;
  int smem_limit = 0, smem_sm = 0;
  XE_CUDA(cudaDeviceGetAttribute(&smem_limit, cudaDevAttrMaxSharedMemoryPerBlockOptin, pr->device));
  XE_CUDA(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, pr->device));
  auto warp_total = [&](int c, int c2) {
    int x = align16(a.off_w_terms + 2 * kSlots * c);
    x = align16(x + 2 * kSlots * c2);
    x = align16(x + kSlots * (8 + 4 + 4 + 4) + 8 * kSlots * P.D + 2 * 32 * kCopyScratch);
    return x;
  };
  // the most resident warps per SM: two CTAs (tables duplicated) or one
  // bigger CTA, whichever holds more
  const int two = smem_sm / 2 - 1024;
  int w2 = kWarps, w1 = kWarps;
  while (w2 > 1 && a.off_warp + w2 * warp_total(cap, cap2) > two) --w2;
  while (w1 > 1 && a.off_warp + w1 * warp_total(cap, cap2) > smem_limit) --w1;
  if (a.off_warp + w2 * warp_total(cap, cap2) > two) w2 = 0;
  int warps = 2 * w2 >= w1 ? w2 : w1;
  while (!exact && cap > 16 && a.off_warp + warps * warp_total(cap, cap2) > smem_limit) {
    cap /= 2;
    cap2 = cap2 ? cap : 0;
  }
  a.warps = warps;
  a.cap = cap;
  a.cap2 = cap2;
  a.off_w_terms2 = align16(a.off_w_terms + 2 * kSlots * cap);
  a.off_w_slot = align16(a.off_w_terms2 + 2 * kSlots * cap2);
  a.warp_bytes = warp_total(cap, cap2);
  const int smem = a.off_warp + warps * a.warp_bytes;
  if (smem > smem_limit) fail(XE_ERR_TOO_LARGE, "candidate cube too large for the shared-memory plan");

  int nsm = 0;
  XE_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, pr->device));
  const int64_t nblocks = (n + kSlots - 1) / kSlots;
  const int grid_cap = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((nblocks + warps - 1) / warps, static_cast<int64_t>(nsm) * 8)));

  const size_t nw_max = static_cast<size_t>(nsm) * 8 * kWarps;
  unsigned char* sc = scratch;
  a.wbest_key = reinterpret_cast<uint64_t*>(sc);
  a.wbest_idx = reinterpret_cast<int64_t*>(sc + nw_max * 8);
  a.wvalid = reinterpret_cast<int64_t*>(sc + nw_max * 16);

  int grid = 0;
  if (n > 0) {
    switch (P.NW) {
      case 1: grid = launch_nw1(a, grid_cap, smem, stream, nsm); break;
      case 2: grid = launch_nw2(a, grid_cap, smem, stream, nsm); break;
      case 3: grid = launch_nw3(a, grid_cap, smem, stream, nsm); break;
      default: grid = launch_nw4(a, grid_cap, smem, stream, nsm); break;
    }
  }
  const size_t nw = static_cast<size_t>(grid) * warps;
  if (best3) {
    if (n > 0) {
      reduce_best_kernel<<<1, 256, 0, stream>>>(a.wbest_key, a.wbest_idx, a.wvalid, static_cast<int>(nw),
                                                best3, reinterpret_cast<int64_t*>(best3 + 1),
                                                reinterpret_cast<int64_t*>(best3 + 2));
      XE_CUDA(cudaGetLastError());
    } else {
      const uint64_t none[3] = {~0ull, ~0ull, 0ull};
      XE_CUDA(cudaMemcpyAsync(best3, none, sizeof none, cudaMemcpyHostToDevice, stream));
    }
  }
}

}  // namespace xe
