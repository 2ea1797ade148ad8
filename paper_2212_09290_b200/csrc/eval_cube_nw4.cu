// SPDX-License-Identifier: Apache-2.0
// K2a instantiation for 256-bit rows (T <= 256).
#include "eval_cube_v3.cuh"

namespace xe {
namespace cube {
int launch_nw4(const EvalArgs& a, int grid, int smem, cudaStream_t s, int nsm) {
  return launch3_d<4>(a, grid, smem, s, nsm);
}
}  // namespace cube
}  // namespace xe
