// SPDX-License-Identifier: Apache-2.0
// K2a instantiation for 192-bit rows (T <= 192).
#include "eval_cube_v3.cuh"

namespace xe {
namespace cube {
int launch_nw3(const EvalArgs& a, int grid, int smem, cudaStream_t s, int nsm) {
  return launch3_d<3>(a, grid, smem, s, nsm);
}
}  // namespace cube
}  // namespace xe
