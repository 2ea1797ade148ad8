# SPDX-License-Identifier: Apache-2.0
"""ctypes binding of the C ABI (include/xengine_b200.h).

Loads the in-tree ``lib/libxengine_b200.so``.  There is no Python or CPU
fallback: if the library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# XE_LIB overrides the library path (A/B builds of the same sources)
LIB_PATH = os.environ.get("XE_LIB", os.path.join(HERE, "lib", "libxengine_b200.so"))

XE_OK = 0
XE_ERR_NO_DEVICE = 103

# XE_F_* validity bits
F_FIXED_ZERO = 1 << 0
F_EQ8 = 1 << 1
F_EQ9 = 1 << 2
F_EQ11 = 1 << 3
F_EQ12 = 1 << 4
F_EQ16_HI = 1 << 8
F_ENERGY_DEV = 1 << 11
F_ENERGY_TOTAL = 1 << 12
F_U_BOUND = 1 << 13
F_BUDGET = 1 << 15
F_DECODE = 1 << 16
F_DECODE_FREED = 1 << 17
F_CHECK_MASK = 0x7FFF

ERRC = [
    "MalformedDocument", "NonTopologicalEdge", "UnknownDevice", "NonPositiveSize",
    "NegativeCost", "EmptyNetwork", "PercentOutOfRange", "MissingLink", "DimensionMismatch",
    "IncompleteEnergyTable", "UnknownVariable", "NonIntegralBinary", "EmptySolution",
    "InfeasibleMarker", "InfeasibleProblem", "TooLarge", "ExternalSolverUnavailable",
    "SolverFailed", "UnparsableSolution", "ObjectiveMismatch", "IllegalAssignment",
    "IllegalSchedule", "EmptySeries", "NonPositiveTime", "IoError",
]


class XeError(RuntimeError):
    """Mirror of xengine::Error (errors.hpp:46-56): .code is the Errc name."""

    def __init__(self, status: int, msg: str):
        if 1 <= status <= len(ERRC):
            code = ERRC[status - 1]
        else:
            code = {100: "CudaError", 101: "NcclError", 102: "InvalidArgument",
                    103: "NoDevice"}.get(status, f"Status{status}")
        super().__init__(f"{code}: {msg}")
        self.status = status
        self.code = code


class ProblemDesc(C.Structure):
    _fields_ = [
        ("D", C.c_int32), ("T", C.c_int32), ("E", C.c_int32),
        ("output_bytes", C.c_void_p), ("cost_ms", C.c_void_p),
        ("edge_src", C.c_void_p), ("edge_dst", C.c_void_p),
        ("copy_ms", C.c_void_p), ("budget_bytes", C.c_void_p),
        ("has_energy", C.c_int32), ("alpha", C.c_double),
        ("q_joules", C.c_void_p), ("has_dev_limit", C.c_void_p),
        ("dev_limit", C.c_void_p), ("has_total_limit", C.c_int32),
        ("total_limit", C.c_double), ("board_joules", C.c_double),
    ]


class ModelOpts(C.Structure):
    _fields_ = [("strict_free", C.c_int32), ("quadratic_objective", C.c_int32),
                ("use_energy", C.c_int32)]


class EvalOut(C.Structure):
    _fields_ = [("obj", C.c_void_p), ("peak", C.c_void_p), ("flags", C.c_void_p)]


class Best(C.Structure):
    _fields_ = [("obj", C.c_double), ("index", C.c_int64), ("n_valid", C.c_int64)]


class CsrInfo(C.Structure):
    _fields_ = [("n_cols", C.c_int64), ("n_rows", C.c_int64), ("nnz", C.c_int64),
                ("n_rows_mps", C.c_int64), ("D", C.c_int32), ("T", C.c_int32),
                ("E", C.c_int32), ("n_tags", C.c_int32), ("tag_rows", C.c_int64 * 16)]


class CsrView(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "row_ptr", "col", "val", "rhs", "sense", "tag", "ordinal", "obj", "obj_present",
        "lb", "ub", "kind")]


class CsrHost(CsrView):
    """xe_csr_host: the same twelve arrays, host pointers."""


class PdhgOpts(C.Structure):
    _fields_ = [("max_iters", C.c_int32), ("tol_rel", C.c_double),
                ("check_every", C.c_int32), ("verbose", C.c_int32),
                ("lb_override", C.c_void_p), ("ub_override", C.c_void_p)]


class PdhgResult(C.Structure):
    _fields_ = [("primal_obj", C.c_double), ("dual_obj", C.c_double),
                ("rel_gap", C.c_double), ("rel_primal_res", C.c_double),
                ("rel_dual_res", C.c_double), ("iters", C.c_int32),
                ("restarts", C.c_int32), ("status", C.c_int32),
                ("solve_ms", C.c_double), ("spmv_ms_per_iter", C.c_double),
                ("presolve_fixed", C.c_int32), ("certified", C.c_int32), ("coded_entries", C.c_int32)]


class SearchOpts(C.Structure):
    _fields_ = [("n_per_round", C.c_int64), ("rounds", C.c_int32), ("edits", C.c_int32),
                ("seed", C.c_uint64), ("use_lp", C.c_int32), ("lp_tol", C.c_double),
                ("valid_mask", C.c_uint32), ("canonical", C.c_int32), ("chains", C.c_int32),
                ("chain_n", C.c_int32), ("chain_iters", C.c_int32), ("max_moves", C.c_int32),
                ("stall", C.c_int32), ("first", C.c_int64), ("rank", C.c_int32), ("world", C.c_int32),
                ("time_limit_ms", C.c_int64)]


class SearchResult(C.Structure):
    _fields_ = [("objective", C.c_double), ("rounding_objective", C.c_double), ("index", C.c_int64),
                ("lp_bound", C.c_double), ("has_lp", C.c_int32), ("lp_certified", C.c_int32),
                ("n_evaluated", C.c_int64), ("n_valid", C.c_int64), ("improvements", C.c_int32),
                ("time_limited", C.c_int32), ("lp_value", C.c_double), ("lp_converged", C.c_int32),
                ("pad_", C.c_int32)]


class ExactOpts(C.Structure):
    _fields_ = [("node_limit", C.c_int64), ("time_limit_ms", C.c_int64), ("upper_bound", C.c_double),
                ("max_states", C.c_int64)]


class ExactResult(C.Structure):
    _fields_ = [("status", C.c_int32), ("found", C.c_int32), ("objective", C.c_double),
                ("sum_r", C.c_int64), ("sum_s", C.c_int64), ("nodes", C.c_int64), ("states", C.c_int64),
                ("ms", C.c_double)]


class Action(C.Structure):
    _fields_ = [("kind", C.c_int32), ("timestep", C.c_int32), ("slot", C.c_int32), ("device", C.c_int32),
                ("op", C.c_int32), ("src", C.c_int32), ("dst", C.c_int32), ("from_", C.c_int32),
                ("to", C.c_int32)]


class DecodeError(C.Structure):
    _fields_ = [("code", C.c_int32), ("t", C.c_int32), ("v", C.c_int32), ("u", C.c_int32)]


class Violation(C.Structure):
    _fields_ = [("kind", C.c_int32), ("device", C.c_int32), ("timestep", C.c_int32), ("slot", C.c_int32),
                ("bytes", C.c_int64), ("a", C.c_int32), ("b", C.c_int32)]


# symbol -> (restype, argtypes); the set of exports include/xengine_b200.h declares
P = C.c_void_p
SIGNATURES = {
    "xe_last_error": (C.c_char_p, []),
    "xe_version": (C.c_char_p, []),
    "xe_cube_bytes": (C.c_size_t, [C.c_int32, C.c_int32]),
    "xe_problem_load_json": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(P)]),
    "xe_problem_parse_json": (C.c_int, [C.c_char_p, C.POINTER(P)]),
    "xe_problem_create": (C.c_int, [C.POINTER(ProblemDesc), C.c_int, C.POINTER(P)]),
    "xe_problem_destroy": (C.c_int, [P]),
    "xe_problem_describe": (C.c_int, [P, C.POINTER(ProblemDesc)]),
    "xe_problem_with_budgets": (C.c_int, [P, P, C.POINTER(P)]),
    "xe_build_csr": (C.c_int, [P, C.POINTER(ModelOpts), C.POINTER(P)]),
    "xe_csr_destroy": (C.c_int, [P]),
    "xe_csr_get_info": (C.c_int, [P, C.POINTER(CsrInfo)]),
    "xe_csr_get_view": (C.c_int, [P, C.POINTER(CsrView)]),
    "xe_csr_build_csc": (C.c_int, [P]),
    "xe_csr_get_csc": (C.c_int, [P, C.POINTER(P), C.POINTER(P), C.POINTER(P)]),
    "xe_write_mps": (C.c_int, [P, P, C.POINTER(C.c_size_t)]),
    "xe_csr_last_build_ms": (C.c_int, [P, C.POINTER(C.c_float)]),
    "xe_eval_cubes": (C.c_int, [P, C.POINTER(ModelOpts), P, C.c_int64, C.POINTER(EvalOut),
                                C.c_uint32, C.POINTER(Best), P]),
    "xe_eval_cubes_host": (C.c_int, [P, C.POINTER(ModelOpts), P, C.c_int64, C.POINTER(EvalOut),
                                     C.c_uint32, C.POINTER(Best)]),
    "xe_cube_il_bytes": (C.c_size_t, [C.c_int32, C.c_int32, C.c_int64]),
    "xe_objective_order_exact": (C.c_int, [P, C.POINTER(C.c_int32)]),
    "xe_problem_set_exact_objective": (C.c_int, [P, C.c_int32]),
    "xe_problem_device_id": (C.c_char_p, [P, C.c_int32]),
    "xe_problem_op_name": (C.c_char_p, [P, C.c_int32]),
    "xe_cubes_to_il": (C.c_int, [P, P, C.c_int64, P, P]),
    "xe_eval_cubes_il": (C.c_int, [P, C.POINTER(ModelOpts), P, C.c_int64, C.POINTER(EvalOut),
                                   C.c_uint32, C.POINTER(Best), P]),
    "xe_csr_download": (C.c_int, [P, C.POINTER(CsrHost)]),
    "xe_csr_upload": (C.c_int, [P, C.POINTER(ModelOpts), C.c_int64, C.c_int64, C.POINTER(CsrHost), C.POINTER(P)]),
    "xe_check_rows": (C.c_int, [P, P, C.c_double, P, C.POINTER(C.c_int64)]),
    "xe_model_cols": (C.c_int64, [C.c_int32, C.c_int32, C.c_int32]),
    "xe_complete_cube": (C.c_int, [P, C.POINTER(ModelOpts), P, P]),
    "xe_objective_dense": (C.c_int, [P, C.POINTER(ModelOpts), P, C.POINTER(C.c_double)]),
    "xe_eval_placements": (C.c_int, [P, P, C.c_int64, C.c_int32, C.POINTER(EvalOut), C.c_uint32,
                                     C.POINTER(Best), P]),
    "xe_assignment_oracle": (C.c_int, [P, C.POINTER(C.c_double), P, C.POINTER(C.c_int64)]),
    "xe_pdhg_solve": (C.c_int, [P, C.POINTER(PdhgOpts), C.POINTER(PdhgResult), P, P]),
    "xe_search_opts_default": (None, [C.POINTER(SearchOpts)]),
    "xe_search": (C.c_int, [P, P, C.POINTER(SearchOpts), C.POINTER(SearchResult), P, P, P]),
    "xe_mutate_cubes": (C.c_int, [P, P, C.c_uint64, C.c_int64, C.c_int64, C.c_int32, C.c_double, P, P]),
    "xe_move_cubes": (C.c_int, [P, P, C.c_int64, C.c_uint64, C.c_int64, C.c_int64, C.c_int32, P, P]),
    "xe_move_placements": (C.c_int, [P, P, C.c_int64, C.c_uint64, C.c_int64, C.c_int64, C.c_int32, P, P]),
    "xe_placement_chains_step": (C.c_int, [P, P, P, C.c_uint32, P, C.c_int32, C.c_int32, C.c_int32, P, P, P, P, P,
                                            P, P]),
    "xe_random_placements": (C.c_int, [P, C.c_uint64, C.c_int64, C.c_int64, P, P]),
    "xe_round_cubes": (C.c_int, [P, P, C.c_uint64, C.c_int64, C.c_int64, C.c_int32, C.c_double,
                                 P, P]),
    "xe_exact_opts_default": (None, [C.POINTER(ExactOpts)]),
    "xe_decode_cubes": (C.c_int, [P, C.POINTER(ModelOpts), P, C.c_int64, P, P, P]),
    "xe_nccl_unique_id": (C.c_int, [P]),
    "xe_ctx_create": (C.c_int, [C.c_int, C.c_int, C.c_int, P, C.POINTER(P)]),
    "xe_ctx_destroy": (C.c_int, [P]),
    "xe_ctx_info": (C.c_int, [P, P, P, P]),
    "xe_ctx_exchange_best": (C.c_int, [P, C.c_int64, C.POINTER(Best)]),
    "xe_search_dist": (C.c_int, [P, C.POINTER(ModelOpts), C.POINTER(SearchOpts), P, C.POINTER(SearchResult), P, P]),
    "xe_decode_dense": (C.c_int, [P, P, C.POINTER(C.c_int64), P, P]),
    "xe_validate_schedules": (C.c_int, [P, P, P, C.c_int64, P, P, P]),
    "xe_replay_schedules": (C.c_int, [P, C.POINTER(ModelOpts), P, P, C.c_int64, P, P, P, P]),
    "xe_format_schedule": (C.c_int, [P, P, C.c_int64, P, C.POINTER(C.c_size_t)]),
    "xe_format_schedule_named": (C.c_int, [P, P, C.c_int64, P, P, P, C.POINTER(C.c_size_t)]),
    "xe_trace_csv": (C.c_int, [P, P, P, C.POINTER(C.c_size_t)]),
    "xe_trace_csv_named": (C.c_int, [P, P, P, P, C.POINTER(C.c_size_t)]),
    "xe_parse_schedule": (C.c_int, [P, C.c_char_p, P, C.POINTER(C.c_int64)]),
    "xe_parse_schedule_named": (C.c_int, [P, C.c_char_p, P, P, C.c_char_p, P, C.POINTER(C.c_int64)]),
    "xe_solve_exact": (C.c_int, [P, P, C.POINTER(ExactOpts), C.POINTER(ExactResult), P, P]),
}


def load(path: str = LIB_PATH):
    if not os.path.exists(path):
        raise ImportError(
            f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 path has no CPU fallback)")
    lib = C.CDLL(path)
    lenient = os.environ.get("XE_LIB_LENIENT") == "1"  # A/B runs against older builds
    for name, (res, args) in SIGNATURES.items():
        if lenient and not hasattr(lib, name):
            continue
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


LIB = load()


def check(status: int):
    if status != XE_OK:
        raise XeError(status, LIB.xe_last_error().decode(errors="replace"))
