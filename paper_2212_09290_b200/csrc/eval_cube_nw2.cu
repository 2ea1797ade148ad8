// SPDX-License-Identifier: Apache-2.0
// K2a instantiation for 128-bit rows (T <= 128).
#include "eval_cube_v3.cuh"

namespace xe {
namespace cube {
int launch_nw2(const EvalArgs& a, int grid, int smem, cudaStream_t s, int nsm) {
  return launch3_d<2>(a, grid, smem, s, nsm);
}
}  // namespace cube
}  // namespace xe
