// SPDX-License-Identifier: Apache-2.0
//
// Placement solvers (drop-in for proj/include/xengine/solver.hpp:13-40).
//   save_all_assignment  save-all (R, S) cubes of a placement, completed on the GPU
//   assignment_oracle    the full D^T placement sweep as one GPU launch (K2b)
//   solve_exact          the reference's exact search (solver.cpp:101-489) as a
//                        GPU dynamic program over the same states (xe_solve_exact):
//                        same optimum, same tail_less tie-break, same statuses
//   solve_search         the GPU best-schedule search for problems beyond
//                        solve_exact's D*T <= 64 (xe_search)
// solve_external (the MPS file bridge to an external MILP solver) is outside
// the B200 hot path.
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <vector>

#include "xengine/model.hpp"

struct xe_ctx;  // include/xengine_b200.h

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

// Memoized search over (timestep, per-device saved set) states (solver.hpp:42-50):
// per timestep the new operator on one device, optional recomputations of
// earlier operators that feed a computation of this timestep, any saved
// subset with a future consumer; memory trajectory within budget.  Proves
// optimality or infeasibility when it runs to completion; D*T <= 64
// (TooLarge otherwise).  Empty budgets means the problem's device budgets.
// Here: the same state space expanded level by level on the GPU; nodes_explored
// counts the legal (state, computation set) frames.
Solution solve_exact(const Problem& p, const ModelOptions& opts = {}, std::vector<std::int64_t> budgets = {},
                     const SearchLimits& limits = {});

// Parameters of solve_search (xe_search_opts in include/xengine_b200.h).
struct SearchParams {
  std::int64_t candidates_per_round = 1 << 18;
  int rounds = 4;
  int edits = 3;            // drop-and-recompute edits per rounded candidate
  std::uint64_t seed = 1;
  bool use_lp = true;       // LP-guided rounding and the LP lower bound
  int chains = 256;         // local-search population (0: rounding only)
  int chain_neighbours = 1024;
  int chain_iters = 200;
  int max_moves = 4;
  int stall = 15;
  SearchLimits limits;      // time_limit_ms honoured (node_limit: candidates are not nodes)
  bool exact_polish = true; // D*T <= 64: solve_exact bounded by the search's objective (proof + tail_less winner)
  std::int64_t exact_polish_ms = 5000;
};

// Best schedule by the GPU search: K1 model -> K3 LP relaxation -> K4
// rounding with canonical saves -> K2 exact scoring (objective_value of the
// completion, check_assignment, integer budgets, decode legality) -> R-space
// local-search population.  backend "b200"; status Optimal when the
// objective meets the LP lower bound (to the PDHG tolerance, 1e-6 relative), LimitReached
// otherwise (objective NaN and an empty assignment when no valid schedule
// was found: infeasibility is not proven); nodes_explored = candidates
// scored.  The assignment is complete_assignment of the best (R, S).
Solution solve_search(const Problem& p, const ModelOptions& opts = {}, const SearchParams& params = {});

// The same search sharded over the ranks of a native multi-GPU context
// (xe_ctx of include/xengine_b200.h: one per GPU, NCCL underneath): rounding
// blocks interleaved by rank, one local-search population per rank, the
// global first-minimum incumbent; every rank returns the same Solution.
Solution solve_search(const Problem& p, const ModelOptions& opts, const SearchParams& params, xe_ctx* ctx);

}  // namespace xengine
