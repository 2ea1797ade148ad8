// SPDX-License-Identifier: Apache-2.0
// K2a v5 streaming evaluator, instantiation for 1-word bit rows (T <= 64).
#include "eval_stream.cuh"

namespace xe {
namespace st {

template <int MAXD, class M, int NBL, int WARPS = kWarps, int TB = 8>
static int launch_one(const StArgs& a, cudaStream_t s, int nsm) {
  auto k = stream_kernel<MAXD, 1, M, NBL, WARPS, TB>;
  XE_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, a.smem_bytes));
  int per_sm = 0;
  XE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, WARPS * 32, a.smem_bytes));
  if (per_sm < 1) fail(XE_ERR_TOO_LARGE, "streaming evaluator does not fit on an SM");
  const int64_t need = ((a.n + 31) / 32 + WARPS - 1) / WARPS;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, static_cast<int64_t>(nsm) * per_sm)));
  k<<<grid, WARPS * 32, a.smem_bytes, s>>>(a);
  XE_CUDA(cudaGetLastError());
  return grid;
}

template <int NCH>
static int launch_wide(const StArgs& a, cudaStream_t s, int nsm) {
  switch (a.P.D) {
    case 2: return launch_one<2, int32_t, NCH, kWideWarps, 11>(a, s, nsm);
    case 3: return launch_one<3, int32_t, NCH, kWideWarps, 11>(a, s, nsm);
    default: return launch_one<4, int32_t, NCH, kWideWarps, 11>(a, s, nsm);
  }
}

template <int NBL>
static int launch_nbl(const StArgs& a, bool m32, cudaStream_t s, int nsm) {
  switch (a.P.D) {
    case 1: return m32 ? launch_one<1, int32_t, NBL>(a, s, nsm) : launch_one<1, int64_t, NBL>(a, s, nsm);
    case 2: return m32 ? launch_one<2, int32_t, NBL>(a, s, nsm) : launch_one<2, int64_t, NBL>(a, s, nsm);
    case 3: return m32 ? launch_one<3, int32_t, NBL>(a, s, nsm) : launch_one<3, int64_t, NBL>(a, s, nsm);
    case 4: return m32 ? launch_one<4, int32_t, NBL>(a, s, nsm) : launch_one<4, int64_t, NBL>(a, s, nsm);
    default: return m32 ? launch_one<8, int32_t, NBL>(a, s, nsm) : launch_one<8, int64_t, NBL>(a, s, nsm);
  }
}

template <>
int launch_stream<1>(const StArgs& a, bool m32, int nbl, cudaStream_t s, int nsm, bool wide) {
  if (wide) return nbl <= 4 ? launch_wide<4>(a, s, nsm) : nbl == 5 ? launch_wide<5>(a, s, nsm) : launch_wide<6>(a, s, nsm);
  return nbl <= 4 ? launch_nbl<4>(a, m32, s, nsm) : nbl <= 6 ? launch_nbl<6>(a, m32, s, nsm) : launch_nbl<8>(a, m32, s, nsm);
}

}  // namespace st
}  // namespace xe
