# SPDX-License-Identifier: Apache-2.0
"""Python mirror of the reference's public API for the hot path.

Names follow proj/include/xengine/*.hpp; every call goes through the C ABI
(``_lib``) to the sm_100a kernels.  torch is used only for device memory and
streams.

    reference (C++)                         here
    load_problem / load_problem_file        Problem.from_json / Problem.from_file
    with_budgets                            Problem.with_budgets
    build_model + write_mps                 build_model(...).write_mps()
    complete_assignment + objective_value   evaluate_cubes(...)  (batched)
      + check_assignment (+ replay peaks)
    save_all_assignment + objective_value   evaluate_placements(...)
    assignment_oracle                       assignment_oracle(...)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from ._lib import LIB, check

_new_bytes = C.pythonapi.PyBytes_FromStringAndSize
_new_bytes.restype = C.py_object
_new_bytes.argtypes = [C.c_void_p, C.c_ssize_t]


@dataclass
class ModelOptions:
    """xengine::ModelOptions (model.hpp:58-62); energy=True applies the
    document's energy section (the reference passes an EnergyModel)."""
    strict_free: bool = False
    quadratic_objective: bool = False
    energy: bool = False

    def c(self):
        return _lib.ModelOpts(int(self.strict_free), int(self.quadratic_objective), int(self.energy))


class Problem:
    """Device-resident problem handle (xe_problem)."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        d = _lib.ProblemDesc()
        check(LIB.xe_problem_describe(self._h, C.byref(d)))
        self.D, self.T, self.E = d.D, d.T, d.E
        self._desc = d

    @classmethod
    def from_json(cls, text: str, device: int = 0) -> "Problem":
        h = C.c_void_p()
        check(LIB.xe_problem_load_json(text.encode(), device, C.byref(h)))
        return cls(h)

    @classmethod
    def from_file(cls, path: str, device: int = 0) -> "Problem":
        try:
            with open(path) as f:
                text = f.read()
        except OSError as ex:
            raise _lib.XeError(25, f"cannot open {path}: {ex}")
        return cls.from_json(text, device)

    @classmethod
    def from_arrays(cls, D, T, E, output_bytes, cost_ms, edge_src, edge_dst, copy_ms,
                    budget_bytes, device: int = 0, energy=None) -> "Problem":
        keep = [np.ascontiguousarray(output_bytes, np.int64),
                np.ascontiguousarray(cost_ms, np.float64),
                np.ascontiguousarray(edge_src, np.int32), np.ascontiguousarray(edge_dst, np.int32),
                np.ascontiguousarray(copy_ms, np.float64),
                np.ascontiguousarray(budget_bytes, np.int64)]
        d = _lib.ProblemDesc(D, T, E, *[k.ctypes.data for k in keep])
        if energy is not None:
            q = np.ascontiguousarray(energy["q"], np.float64)
            hl = np.ascontiguousarray(energy.get("has_dev_limit", np.zeros(D)), np.uint8)
            lim = np.ascontiguousarray(energy.get("dev_limit", np.zeros(D)), np.float64)
            keep += [q, hl, lim]
            d.has_energy = 1
            d.alpha = float(energy.get("alpha", 0.0))
            d.q_joules, d.has_dev_limit, d.dev_limit = q.ctypes.data, hl.ctypes.data, lim.ctypes.data
            tl = energy.get("total_limit")
            d.has_total_limit = 0 if tl is None else 1
            d.total_limit = 0.0 if tl is None else float(tl)
            d.board_joules = float(energy.get("board_joules", 0.0))
        h = C.c_void_p()
        check(LIB.xe_problem_create(C.byref(d), device, C.byref(h)))
        return cls(h)

    def __del__(self):
        try:
            if self._h:
                LIB.xe_problem_destroy(self._h)
                self._h = None
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def arrays(self) -> dict:
        """Resolved arrays (after copy_cost) as numpy copies."""
        d = self._desc
        D, T, E = self.D, self.T, self.E

        def arr(ptr, n, dt):
            if n == 0:
                return np.zeros(0, dt)
            return np.ctypeslib.as_array(
                C.cast(ptr, C.POINTER(np.ctypeslib.as_ctypes_type(dt))), shape=(n,)).copy()

        out = {
            "output_bytes": arr(d.output_bytes, T, np.int64),
            "cost_ms": arr(d.cost_ms, D * T, np.float64).reshape(D, T),
            "edge_src": arr(d.edge_src, E, np.int32),
            "edge_dst": arr(d.edge_dst, E, np.int32),
            "copy_ms": arr(d.copy_ms, E * D * D, np.float64).reshape(E, D, D),
            "budget_bytes": arr(d.budget_bytes, D, np.int64),
            "has_energy": bool(d.has_energy),
        }
        if d.has_energy:
            out.update(alpha=d.alpha, q_joules=arr(d.q_joules, D * T, np.float64).reshape(D, T),
                       has_dev_limit=arr(d.has_dev_limit, D, np.uint8),
                       dev_limit=arr(d.dev_limit, D, np.float64),
                       total_limit=d.total_limit if d.has_total_limit else None,
                       board_joules=d.board_joules)
        return out

    def with_budgets(self, budgets) -> "Problem":
        b = np.ascontiguousarray(budgets, np.int64)
        h = C.c_void_p()
        check(LIB.xe_problem_with_budgets(self._h, b.ctypes.data, C.byref(h)))
        return Problem(h)

    @property
    def cube_words(self) -> int:
        return 2 * self.D * self.T * ((self.T + 31) // 32)

    @property
    def objective_order_exact(self) -> bool:
        """True when per-candidate objectives are bit-identical to the
        reference's sequential sum (every term dyadic); otherwise they are a
        per-timestep reassociation within ~#terms * 2^-53 relative.  The
        best-of-batch objective is exact either way."""
        x = C.c_int32()
        check(LIB.xe_objective_order_exact(self._h, C.byref(x)))
        return bool(x.value)

    def names(self) -> dict:
        """Device ids and operator names of the document (problem.hpp:18-60)."""
        return {"devices": [LIB.xe_problem_device_id(self._h, d).decode() for d in range(self.D)],
                "ops": [LIB.xe_problem_op_name(self._h, i).decode() for i in range(self.T)]}

    def set_exact_objective(self, exact: bool = True) -> "Problem":
        """Every batched evaluation on this handle sums each candidate's
        objective in the reference's order (objective_value, model.cpp:
        392-411) when exact, at the reference-order kernels' speed."""
        check(LIB.xe_problem_set_exact_objective(self._h, int(bool(exact))))
        return self


@dataclass
class EvalResult:
    obj: object       # [n] float64 (torch on device, or numpy)
    peak: object      # [n, D] int64
    flags: object     # [n] uint32 (as int32 in torch)
    best_obj: float
    best_index: int
    n_valid: int


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def evaluate_cubes(problem: Problem, cubes, opts: Optional[ModelOptions] = None,
                   valid_mask: int = _lib.F_CHECK_MASK, outputs: bool = True, stream=None,
                   out=None, best: bool = True):
    """Evaluate device-resident cubes (torch uint32/int32 CUDA tensor of
    shape [n, cube_words]).  Returns EvalResult with torch tensors.
    out=(obj, peak, flags) reuses preallocated device tensors; best=False
    skips the best-of-batch reduction and its host read (asynchronous)."""
    import torch
    opts = opts or ModelOptions()
    n = cubes.shape[0] if cubes.dim() > 1 else cubes.numel() // problem.cube_words
    dev = cubes.device
    if out is not None:
        obj, peak, flags = out
    else:
        obj = torch.empty(n, dtype=torch.float64, device=dev) if outputs else None
        peak = torch.empty((n, problem.D), dtype=torch.int64, device=dev) if outputs else None
        flags = torch.empty(n, dtype=torch.int32, device=dev) if outputs else None
    eo = _lib.EvalOut(_ptr(obj), _ptr(peak), _ptr(flags))
    b = _lib.Best()
    s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    check(LIB.xe_eval_cubes(problem.handle, C.byref(opts.c()), C.c_void_p(cubes.data_ptr()), n,
                            C.byref(eo), valid_mask, C.byref(b) if best else None, C.c_void_p(s)))
    if not best:
        return EvalResult(obj, peak, flags, float("nan"), -1, -1)
    return EvalResult(obj, peak, flags, b.obj, b.index, b.n_valid)


def cubes_to_il(problem: Problem, cubes, out=None, stream=None):
    """Canonical device cubes [n, cube_words] -> the interleaved layout
    (xe_cube_il: 32-candidate groups, one u64 bit row per (R|S, d, t))."""
    import torch
    n = cubes.shape[0]
    words = LIB.xe_cube_il_bytes(problem.D, problem.T, n) // 8
    if out is None:
        out = torch.empty(words, dtype=torch.int64, device=cubes.device)
    s = stream if stream is not None else torch.cuda.current_stream(cubes.device).cuda_stream
    check(LIB.xe_cubes_to_il(problem.handle, C.c_void_p(cubes.data_ptr()), n, C.c_void_p(out.data_ptr()),
                             C.c_void_p(s)))
    return out


def evaluate_cubes_il(problem: Problem, il, n: int, opts: Optional[ModelOptions] = None,
                      valid_mask: int = _lib.F_CHECK_MASK, outputs: bool = True, stream=None,
                      out=None, best: bool = True):
    """Evaluate n interleaved device candidates (cubes_to_il / round_cubes(layout="il"));
    same results as evaluate_cubes on the canonical layout."""
    import torch
    opts = opts or ModelOptions()
    dev = il.device
    if out is not None:
        obj, peak, flags = out
    else:
        obj = torch.empty(n, dtype=torch.float64, device=dev) if outputs else None
        peak = torch.empty((n, problem.D), dtype=torch.int64, device=dev) if outputs else None
        flags = torch.empty(n, dtype=torch.int32, device=dev) if outputs else None
    eo = _lib.EvalOut(_ptr(obj), _ptr(peak), _ptr(flags))
    b = _lib.Best()
    s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    check(LIB.xe_eval_cubes_il(problem.handle, C.byref(opts.c()), C.c_void_p(il.data_ptr()), n,
                               C.byref(eo), valid_mask, C.byref(b) if best else None, C.c_void_p(s)))
    if not best:
        return EvalResult(obj, peak, flags, float("nan"), -1, -1)
    return EvalResult(obj, peak, flags, b.obj, b.index, b.n_valid)


def mutate_cubes(problem: Problem, base, n: int, seed: int, first: int = 0, edits: int = 2,
                 perturb: float = 0.0, out=None, stream=None):
    """K4 local search: n neighbours of the canonical device cube `base`
    (int32 CUDA tensor [cube_words])."""
    import torch
    if out is None:
        out = torch.empty((n, problem.cube_words), dtype=torch.int32, device=base.device)
    s = stream if stream is not None else torch.cuda.current_stream(out.device).cuda_stream
    check(LIB.xe_mutate_cubes(problem.handle, C.c_void_p(base.data_ptr()), seed, first, n, edits, perturb,
                              C.c_void_p(out.data_ptr()), C.c_void_p(s)))
    return out


def move_cubes(problem: Problem, base, n: int, seed: int, first: int = 0, max_moves: int = 2, out=None,
               stream=None):
    """K4 local search in R space: n neighbours of `base` (int32 CUDA tensor
    [cube_words], or [n_base, cube_words] for independent chains — n a
    multiple of n_base, neighbour k of base k // (n // n_base); the S part is
    ignored): 1..max_moves random moves on the computations, then the
    canonical saves.  max_moves=0: the base's R with canonical saves."""
    import torch
    nb = 1 if base.dim() == 1 else base.shape[0]
    if out is None:
        out = torch.empty((n, problem.cube_words), dtype=torch.int32, device=base.device)
    s = stream if stream is not None else torch.cuda.current_stream(out.device).cuda_stream
    check(LIB.xe_move_cubes(problem.handle, C.c_void_p(base.contiguous().data_ptr()), nb, seed, first, n,
                            max_moves, C.c_void_p(out.data_ptr()), C.c_void_p(s)))
    return out


def move_placements(problem: Problem, base, n: int, seed: int, first: int = 0, max_moves: int = 4, out=None,
                    stream=None):
    """K4 placement-space neighbours: base uint8 CUDA tensor [n_base, T] (or
    [T]); neighbour k copies base k // (n // n_base) and moves 1..max_moves
    random ops to a random allowed device."""
    import torch
    b = base.unsqueeze(0) if base.dim() == 1 else base
    b = b.contiguous()
    if out is None:
        out = torch.empty((n, problem.T), dtype=torch.uint8, device=b.device)
    s = stream if stream is not None else torch.cuda.current_stream(out.device).cuda_stream
    check(LIB.xe_move_placements(problem.handle, C.c_void_p(b.data_ptr()), b.shape[0], seed, first, n, max_moves,
                                 C.c_void_p(out.data_ptr()), C.c_void_p(s)))
    return out


def random_placements(problem: Problem, n: int, seed: int, first: int = 0, out=None, stream=None):
    """n uniform random placements (uint8 CUDA tensor [n, T]); candidate k is
    a pure function of (seed, first + k)."""
    import torch
    if out is None:
        out = torch.empty((n, problem.T), dtype=torch.uint8, device="cuda")
    s = stream if stream is not None else torch.cuda.current_stream(out.device).cuda_stream
    check(LIB.xe_random_placements(problem.handle, seed, first, n, C.c_void_p(out.data_ptr()), C.c_void_p(s)))
    return out


def evaluate_placements(problem: Problem, dev, policy: int = 0, valid_mask: int = _lib.F_CHECK_MASK,
                        outputs: bool = True, stream=None, out=None, best: bool = True):
    """K2b: device placements (uint8 CUDA tensor [n, T]); policy 0 = save-all
    (save_all_assignment, solver.cpp:30-42), 1 = minimal-save."""
    import torch
    n = dev.shape[0]
    if out is not None:
        obj, peak, flags = out
    else:
        obj = torch.empty(n, dtype=torch.float64, device=dev.device) if outputs else None
        peak = torch.empty((n, problem.D), dtype=torch.int64, device=dev.device) if outputs else None
        flags = torch.empty(n, dtype=torch.int32, device=dev.device) if outputs else None
    eo = _lib.EvalOut(_ptr(obj), _ptr(peak), _ptr(flags))
    b = _lib.Best()
    s = stream if stream is not None else torch.cuda.current_stream(dev.device).cuda_stream
    check(LIB.xe_eval_placements(problem.handle, C.c_void_p(dev.data_ptr()), n, policy, C.byref(eo), valid_mask,
                                 C.byref(b) if best else None, C.c_void_p(s)))
    if not best:
        return EvalResult(obj, peak, flags, float("nan"), -1, -1)
    return EvalResult(obj, peak, flags, b.obj, b.index, b.n_valid)


def assignment_oracle(problem: Problem):
    """assignment_oracle (solver.cpp:44-75): the full D^T save-all sweep on the
    GPU; returns (best objective, device vector, placements evaluated)."""
    obj, n = C.c_double(), C.c_int64()
    dev = np.zeros(problem.T, np.int32)
    check(LIB.xe_assignment_oracle(problem.handle, C.byref(obj), dev.ctypes.data, C.byref(n)))
    return obj.value, dev, n.value


@dataclass
class ExactResult:
    status: str                   # "optimal" | "infeasible" | "limit" (status_name, solver.cpp)
    objective: float              # the search's tail cost (objective_ms); nan without a solution
    cube: Optional[np.ndarray]    # canonical (R, S) cube words of the optimum (uint32), None without one
    sum_r: int                    # tail_less keys of the optimum (solver.cpp:87-92)
    sum_s: int
    nodes: int                    # legal (state, computation set) frames expanded
    states: int                   # distinct (timestep, saved-set) states kept
    ms: float


def solve_exact(problem: Problem, opts: Optional[ModelOptions] = None, node_limit: Optional[int] = None,
                time_limit_ms: Optional[int] = None, upper_bound: float = float("inf")) -> ExactResult:
    """solve_exact (solver.hpp:42-50, solver.cpp:449-489) as the GPU dynamic
    program of csrc/exact.cu: same states, transitions and tail_less optimum
    as the reference's memoised DFS.  Budgets are the problem's (use
    Problem.with_budgets for the reference's budget override)."""
    o = _lib.ExactOpts()
    LIB.xe_exact_opts_default(C.byref(o))
    if node_limit is not None:
        o.node_limit = int(node_limit)
    if time_limit_ms is not None:
        o.time_limit_ms = int(time_limit_ms)
    o.upper_bound = float(upper_bound)
    r = _lib.ExactResult()
    cube = np.zeros(LIB.xe_cube_bytes(problem.D, problem.T) // 4, np.uint32)
    mo = (opts or ModelOptions()).c()
    check(LIB.xe_solve_exact(problem.handle, C.byref(mo), C.byref(o), C.byref(r), cube.ctypes.data, None))
    status = {0: "optimal", 1: "infeasible", 2: "limit"}[r.status]
    return ExactResult(status, r.objective, cube if r.found else None, r.sum_r, r.sum_s, r.nodes, r.states, r.ms)


class _DevArray:
    """__cuda_array_interface__ view of a device pointer owned by the library."""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr,
                                         "data": (int(ptr or 0), False), "version": 3}


def _dev_tensor(ptr, n, typestr):
    import torch
    return torch.as_tensor(_DevArray(ptr, n, typestr), device="cuda")


TAGS = ["EQ7", "EQ8", "EQ9", "EQ10", "EQ11", "EQ12", "EQ13", "EQ14", "EQ16_LO", "EQ16_HI",
        "Z_LINK", "P_LINK", "ENERGY_DEV", "ENERGY_TOTAL"]


class Model:
    """Device-resident MILP (xe_csr): the B200 counterpart of MilpModel
    (model.hpp:81-101) as CSR over closed-form VarRef columns."""

    def __init__(self, problem: "Problem", handle):
        self.problem = problem
        self._h = handle
        info = _lib.CsrInfo()
        check(LIB.xe_csr_get_info(self._h, C.byref(info)))
        self.n_cols, self.n_rows, self.nnz = info.n_cols, info.n_rows, info.nnz
        self.tag_rows = {TAGS[i]: info.tag_rows[i] for i in range(14)}
        v = _lib.CsrView()
        check(LIB.xe_csr_get_view(self._h, C.byref(v)))
        self._v = v

    def __del__(self):
        try:
            if self._h:
                LIB.xe_csr_destroy(self._h)
                self._h = None
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def build_ms(self) -> float:
        ms = C.c_float()
        check(LIB.xe_csr_last_build_ms(self._h, C.byref(ms)))
        return ms.value

    def device_arrays(self) -> dict:
        """Zero-copy torch views of the device model."""
        v, m, n, z = self._v, self.n_rows, self.n_cols, self.nnz
        return {
            "row_ptr": _dev_tensor(v.row_ptr, m + 1, "<i8"), "col": _dev_tensor(v.col, z, "<i4"),
            "val": _dev_tensor(v.val, z, "<f8"), "rhs": _dev_tensor(v.rhs, m, "<f8"),
            "sense": _dev_tensor(v.sense, m, "|i1"), "tag": _dev_tensor(v.tag, m, "|u1"),
            "ordinal": _dev_tensor(v.ordinal, m, "<i4"), "obj": _dev_tensor(v.obj, n, "<f8"),
            "obj_present": _dev_tensor(v.obj_present, n, "|u1"), "lb": _dev_tensor(v.lb, n, "<f8"),
            "ub": _dev_tensor(v.ub, n, "<f8"), "kind": _dev_tensor(v.kind, n, "|u1"),
        }

    def to_host(self) -> dict:
        return {k: t.cpu().numpy() for k, t in self.device_arrays().items()}

    def csc(self) -> dict:
        check(LIB.xe_csr_build_csc(self._h))
        cp, r, val = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(LIB.xe_csr_get_csc(self._h, C.byref(cp), C.byref(r), C.byref(val)))
        return {"col_ptr": _dev_tensor(cp.value, self.n_cols + 1, "<i8"),
                "row": _dev_tensor(r.value, self.nnz, "<i4"),
                "val": _dev_tensor(val.value, self.nnz, "<f8")}

    def write_mps(self) -> bytes:
        """write_mps (mps_io.cpp:109-199), byte-identical."""
        n = C.c_size_t()
        check(LIB.xe_write_mps(self._h, None, C.byref(n)))
        # the text is downloaded straight into a fresh, not yet shared bytes
        # object (one host pass instead of buffer + copy)
        if n.value == 0:  # (the empty bytes object is shared: never written into)
            return b""
        out = _new_bytes(None, n.value)
        check(LIB.xe_write_mps(self._h, C.c_char_p(out), C.byref(n)))
        return out


@dataclass
class LpResult:
    primal_obj: float
    dual_obj: float
    rel_gap: float
    rel_primal_res: float
    iters: int
    restarts: int
    converged: bool
    solve_ms: float
    ms_per_iter: float
    presolve_fixed: int = 0
    certified: bool = True
    coded: bool = False  # half-steps on coded entries (4 B) instead of fp64 values (12 B)
    x: Optional[np.ndarray] = None
    y: Optional[np.ndarray] = None


def pdhg_solve(model: Model, tol: float = 1e-6, max_iters: int = 200000, check_every: int = 64,
               lb=None, ub=None, return_x: bool = False, return_y: bool = False,
               verbose: bool = False) -> LpResult:
    """K3: LP relaxation of the model by PDHG (restarted, preconditioned).
    lb/ub: optional per-column bound overrides (branch-and-bound nodes)."""
    lbo = None if lb is None else np.ascontiguousarray(lb, np.float64)
    ubo = None if ub is None else np.ascontiguousarray(ub, np.float64)
    o = _lib.PdhgOpts(max_iters, tol, check_every, int(verbose),
                      None if lbo is None else lbo.ctypes.data, None if ubo is None else ubo.ctypes.data)
    r = _lib.PdhgResult()
    x = np.empty(model.n_cols) if return_x else None
    y = np.empty(model.n_rows) if return_y else None
    check(LIB.xe_pdhg_solve(model.handle, C.byref(o), C.byref(r),
                            None if x is None else x.ctypes.data, None if y is None else y.ctypes.data))
    return LpResult(r.primal_obj, r.dual_obj, r.rel_gap, r.rel_primal_res, r.iters, r.restarts,
                    r.status == 0, r.solve_ms, r.spmv_ms_per_iter, r.presolve_fixed, bool(r.certified),
                    bool(r.coded_entries), x, y)


def build_model(problem: "Problem", opts: Optional[ModelOptions] = None) -> Model:
    """build_model (model.cpp:86-256) on the GPU (K1)."""
    opts = opts or ModelOptions()
    h = C.c_void_p()
    check(LIB.xe_build_csr(problem.handle, C.byref(opts.c()), C.byref(h)))
    return Model(problem, h)


def round_cubes(problem: Problem, n: int, seed: int, first: int = 0, edits: int = 3,
                perturb: float = 0.1, x=None, out=None, stream=None):
    """K4: n candidate cubes (torch int32 CUDA tensor [n, cube_words]) sampled
    from LP marginals x (device float64 tensor over the model's columns) or
    uniformly when x is None; candidate k is a pure function of (seed, first+k)."""
    import torch
    if out is None:
        out = torch.empty((n, problem.cube_words), dtype=torch.int32, device="cuda")
    s = stream if stream is not None else torch.cuda.current_stream(out.device).cuda_stream
    check(LIB.xe_round_cubes(problem.handle, _ptr(x), seed, first, n, edits, perturb,
                             C.c_void_p(out.data_ptr()), C.c_void_p(s)))
    return out


def evaluate_cubes_host(problem: Problem, cubes: np.ndarray, opts: Optional[ModelOptions] = None,
                        valid_mask: int = _lib.F_CHECK_MASK, outputs: bool = True):
    """End-to-end path: host cubes -> host results (copies inside the call)."""
    opts = opts or ModelOptions()
    cubes = np.ascontiguousarray(cubes)
    if cubes.dtype == np.int32:
        cubes = cubes.view(np.uint32)  # same bits; keeps a pinned buffer pinned (no conversion copy)
    cubes = np.ascontiguousarray(cubes, np.uint32).reshape(-1, problem.cube_words)
    n = cubes.shape[0]
    obj = np.empty(n, np.float64) if outputs else None
    peak = np.empty((n, problem.D), np.int64) if outputs else None
    flags = np.empty(n, np.uint32) if outputs else None
    out = _lib.EvalOut(*(None if a is None else C.c_void_p(a.ctypes.data) for a in (obj, peak, flags)))
    best = _lib.Best()
    check(LIB.xe_eval_cubes_host(problem.handle, C.byref(opts.c()), cubes.ctypes.data, n,
                                 C.byref(out), valid_mask, C.byref(best)))
    return EvalResult(obj, peak, flags, best.obj, best.index, best.n_valid)
