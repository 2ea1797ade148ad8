// SPDX-License-Identifier: Apache-2.0
//
// MPS serialisation (drop-in for the write side of
// proj/include/xengine/mps_io.hpp:14-29).  write_mps streams the bytes of the
// reference writer from the GPU-assembled, GPU-transposed model (K1).
// parse_solution / format_solution: the solution side of the external-solver
// bridge (mps_io.cpp:201-263), host text.
#pragma once

#include <optional>
#include <string>

#include "xengine/model.hpp"

namespace xengine {

// Shortest round-trip decimal; integral |v| < 1e15 without a decimal point.
std::string format_number(double v);
std::string var_name(const VarRef& v);
std::optional<VarRef> parse_var_name(const std::string& name);
std::string write_mps(const MilpModel& m);
Assignment parse_solution(const std::string& text, const MilpModel& m);
std::string format_solution(const Assignment& a);

}  // namespace xengine
