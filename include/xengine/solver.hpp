// SPDX-License-Identifier: Apache-2.0
//
// Placement solvers (drop-in for proj/include/xengine/solver.hpp:13-40).
//   save_all_assignment  save-all (R, S) cubes of a placement, completed on the GPU
//   assignment_oracle    the full D^T placement sweep as one GPU launch (K2b)
// solve_exact / solve_external (memoised DFS, MPS file bridge) are outside
// the B200 hot path.
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <vector>

#include "xengine/model.hpp"

namespace xengine {

enum class SolveStatus { Optimal, Infeasible, LimitReached };

const char* status_name(SolveStatus s);

struct SearchLimits {
  std::optional<std::int64_t> node_limit;
  std::optional<std::int64_t> time_limit_ms;
};

struct Solution {
  SolveStatus status = SolveStatus::Optimal;
  std::string backend;        // "oracle" here
  double objective_ms = 0.0;  // NaN without a solution
  Assignment assignment;
  std::int64_t nodes_explored = 0;
};

Assignment save_all_assignment(const Problem& p, const std::vector<int>& devices);
Solution assignment_oracle(const Problem& p);

}  // namespace xengine
