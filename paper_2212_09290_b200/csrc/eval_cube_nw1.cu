// SPDX-License-Identifier: Apache-2.0
// K2a instantiation for 64-bit rows (T <= 64).
#include "eval_cube_v3.cuh"

namespace xe {
namespace cube {
int launch_nw1(const EvalArgs& a, int grid, int smem, cudaStream_t s, int nsm) {
  return launch3_d<1>(a, grid, smem, s, nsm);
}
}  // namespace cube
}  // namespace xe
