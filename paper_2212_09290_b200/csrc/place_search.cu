// SPDX-License-Identifier: Apache-2.0
//
// Chain control of the placement local search (search_placements): one
// iteration's decision for every chain on the device, so the loop
// (xe_move_placements -> xe_eval_placements -> this) runs without host
// round trips.  Chain c holds a base placement [T] u8, its objective `cur`
// and a stall counter.  Its M neighbours' scores are their objectives when
// (flags & valid_mask) == 0, else +inf; the best one (first index among
// equal scores) is taken when it improves, or after `stall` iterations
// without improvement when it is valid.  The incumbent (best objective and
// its placement) is updated in the same launch sequence.

#include <cmath>

#include "xe_internal.hpp"

namespace xe {
namespace {

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads) chain_step_kernel(const double* obj, const uint32_t* flags,
                                                              uint32_t valid_mask, const uint8_t* nb, int M, int T,
                                                              int stall, uint8_t* bases, double* cur,
                                                              int32_t* stalled) {
  __shared__ double sv[kThreads];
  __shared__ int sj[kThreads];
  __shared__ int take_j;
  const int c = blockIdx.x;
  double bv = INFINITY;
  int bj = -1;
  for (int j = threadIdx.x; j < M; j += kThreads) {
    const int64_t k = static_cast<int64_t>(c) * M + j;
    const double v = (flags[k] & valid_mask) == 0 ? obj[k] : INFINITY;
    if (v < bv) {  // j ascending per thread: the first index wins ties
      bv = v;
      bj = j;
    }
  }
  sv[threadIdx.x] = bv;
  sj[threadIdx.x] = bj;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double ov = sv[threadIdx.x + s];
      const int oj = sj[threadIdx.x + s];
      if (ov < sv[threadIdx.x] || (ov == sv[threadIdx.x] && oj >= 0 && (sj[threadIdx.x] < 0 || oj < sj[threadIdx.x]))) {
        sv[threadIdx.x] = ov;
        sj[threadIdx.x] = oj;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double v = sv[0], cv = cur[c];
    const bool improve = v < cv;
    const bool take = sj[0] >= 0 && (improve || (stalled[c] >= stall && isfinite(v)));
    stalled[c] = (improve || take) ? 0 : stalled[c] + 1;
    if (take) cur[c] = v;
    take_j = take ? sj[0] : -1;
  }
  __syncthreads();
  if (take_j >= 0) {
    const uint8_t* src = nb + (static_cast<int64_t>(c) * M + take_j) * T;
    for (int i = threadIdx.x; i < T; i += kThreads) bases[static_cast<int64_t>(c) * T + i] = src[i];
  }
}

// incumbent: the lowest chain objective (first chain among equals) replaces
// the best when strictly lower; improvements counted on the device
__global__ void __launch_bounds__(kThreads) best_update_kernel(const double* cur, const uint8_t* bases, int P, int T,
                                                               double* best, uint8_t* best_dev, int32_t* improvements) {
  __shared__ double sv[kThreads];
  __shared__ int sc[kThreads];
  __shared__ int win;
  double bv = INFINITY;
  int bc = -1;
  for (int c = threadIdx.x; c < P; c += kThreads)
    if (cur[c] < bv) {
      bv = cur[c];
      bc = c;
    }
  sv[threadIdx.x] = bv;
  sc[threadIdx.x] = bc;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double ov = sv[threadIdx.x + s];
      const int oc = sc[threadIdx.x + s];
      if (ov < sv[threadIdx.x] || (ov == sv[threadIdx.x] && oc >= 0 && (sc[threadIdx.x] < 0 || oc < sc[threadIdx.x]))) {
        sv[threadIdx.x] = ov;
        sc[threadIdx.x] = oc;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    win = (sc[0] >= 0 && sv[0] < *best) ? sc[0] : -1;
    if (win >= 0) {
      *best = sv[0];
      ++*improvements;
    }
  }
  __syncthreads();
  if (win >= 0)
    for (int i = threadIdx.x; i < T; i += kThreads) best_dev[i] = bases[static_cast<int64_t>(win) * T + i];
}

}  // namespace
}  // namespace xe

using namespace xe;

extern "C" int xe_placement_chains_step(const xe_problem* p, const double* obj, const uint32_t* flags,
                                        uint32_t valid_mask, const uint8_t* nb, int32_t chains, int32_t chain_n,
                                        int32_t stall, uint8_t* bases, double* cur, int32_t* stalled, double* best,
                                        uint8_t* best_dev, int32_t* improvements, void* stream) {
  return guard([&] {
    if (!p || !obj || !flags || !nb || !bases || !cur || !stalled || !best || !best_dev || !improvements ||
        chains < 1 || chain_n < 1)
      fail(XE_ERR_ARG, "bad argument");
    require_uploaded(p);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    chain_step_kernel<<<chains, kThreads, 0, s>>>(obj, flags, valid_mask, nb, chain_n, p->h.T, stall, bases, cur,
                                                  stalled);
    XE_CUDA(cudaGetLastError());
    best_update_kernel<<<1, kThreads, 0, s>>>(cur, bases, chains, p->h.T, best, best_dev, improvements);
    XE_CUDA(cudaGetLastError());
  });
}
