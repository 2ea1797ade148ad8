// SPDX-License-Identifier: Apache-2.0
// Entry points of include/xengine_b200.h whose kernels are not built yet.
// Each returns XE_ERR_ARG with an explicit message (never a CPU fallback).
#include "xe_internal.hpp"

using namespace xe;

#define XE_TODO(name) set_last_error(std::string(name) + ": not implemented in this build"); return XE_ERR_ARG

extern "C" {
int xe_eval_placements(const xe_problem*, const uint8_t*, int64_t, int32_t, xe_eval_out*, uint32_t, xe_best*, void*) { XE_TODO("xe_eval_placements"); }
int xe_assignment_oracle(const xe_problem*, double*, int32_t*, int64_t*) { XE_TODO("xe_assignment_oracle"); }
}
