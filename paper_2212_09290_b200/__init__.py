# SPDX-License-Identifier: Apache-2.0
"""B200-native XEngine hot path (arXiv 2212.09290): MILP assembly (K1),
batched schedule evaluation (K2), PDHG LP relaxation (K3) and randomized
rounding (K4) behind the reference's C++ interfaces, via a C ABI."""
from ._lib import XeError, LIB_PATH  # noqa: F401  (raises ImportError if the .so is missing)
from .api import (ModelOptions, Problem, EvalResult, evaluate_cubes,  # noqa: F401
                  evaluate_cubes_host, evaluate_cubes_il, cubes_to_il, round_cubes,
                  random_placements, evaluate_placements, assignment_oracle, mutate_cubes, move_cubes, move_placements, Model, build_model, pdhg_solve, LpResult,
                  solve_exact, ExactResult)
