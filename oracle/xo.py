# SPDX-License-Identifier: Apache-2.0
"""TEST INFRASTRUCTURE ONLY — the checker, never the product.

Python side of the oracle:

* ``load_problem`` / ``make_training_graph`` / ``copy_cost`` /
  ``budget_percent`` / ``with_budgets`` / ``parse_energy`` restate the
  reference loader (proj/src/problem.cpp:140-393, proj/src/model.cpp:314-367)
  so the product's C++ loader can be checked field by field.
* ``Oracle`` binds ``oracle/liboracle.so`` (the C restatement, xe_oracle.c).
* ``Ref`` binds ``oracle/_ref/libxengine_ref.so`` (the unmodified reference
  library + harness, built by oracle/Makefile when /root/reference exists).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs import this module.
"""
from __future__ import annotations

import ctypes as C
import json
import math
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
K_PROHIBITIVE_MS = 1.0e9  # problem.hpp:16
ERRC = [
    "MalformedDocument", "NonTopologicalEdge", "UnknownDevice", "NonPositiveSize",
    "NegativeCost", "EmptyNetwork", "PercentOutOfRange", "MissingLink", "DimensionMismatch",
    "IncompleteEnergyTable", "UnknownVariable", "NonIntegralBinary", "EmptySolution",
    "InfeasibleMarker", "InfeasibleProblem", "TooLarge", "ExternalSolverUnavailable",
    "SolverFailed", "UnparsableSolution", "ObjectiveMismatch", "IllegalAssignment",
    "IllegalSchedule", "EmptySeries", "NonPositiveTime", "IoError",
]

# XE_F_* bits (include/xengine_b200.h)
F_FIXED_ZERO, F_EQ8, F_EQ9, F_EQ11, F_EQ12 = 1 << 0, 1 << 1, 1 << 2, 1 << 3, 1 << 4
F_EQ16_HI, F_ENERGY_DEV, F_ENERGY_TOTAL, F_U_BOUND = 1 << 8, 1 << 11, 1 << 12, 1 << 13
F_BUDGET, F_DECODE, F_DECODE_FREED = 1 << 15, 1 << 16, 1 << 17
F_CHECK_MASK = 0x7FFF


class OracleError(Exception):
    def __init__(self, code: str, what: str):
        super().__init__(f"{code}: {what}")
        self.code = code


def _raise(code: str, what: str):
    raise OracleError(code, what)


# --------------------------------------------------------------------------
# Loader restatement (problem.cpp)
# --------------------------------------------------------------------------
@dataclass
class Problem:
    name: str = "unnamed"
    devices: list = field(default_factory=list)      # (id, budget, ram)
    ops: list = field(default_factory=list)          # (name, bytes, costs[D], pinned)
    edges: list = field(default_factory=list)        # (src, dst, {(a,b): ms})
    links: list = field(default_factory=list)        # (from, to, latency, bytes_per_ms)

    @property
    def D(self):
        return len(self.devices)

    @property
    def T(self):
        return len(self.ops)

    @property
    def E(self):
        return len(self.edges)

    def find_device(self, id_):
        for d, dev in enumerate(self.devices):
            if dev[0] == id_:
                return d
        return -1


def _is_int(x):
    return isinstance(x, int) and not isinstance(x, bool)


def _is_num(x):
    return isinstance(x, (int, float)) and not isinstance(x, bool)


def _require_size(j, ctx):  # problem.cpp:55-61
    if not _is_int(j):
        _raise("MalformedDocument", ctx + " must be an integer byte count")
    if j <= 0:
        _raise("NonPositiveSize", ctx)
    return j


def _require_cost(j, ctx):  # problem.cpp:63-68
    if not _is_num(j):
        _raise("MalformedDocument", ctx + " must be a number")
    if j < 0:
        _raise("NegativeCost", ctx)
    return float(j)


def _parse_devices(doc):  # problem.cpp:70-90
    devs = doc.get("devices")
    if not isinstance(devs, list) or not devs:
        _raise("MalformedDocument", "document needs a non-empty devices array")
    out, seen = [], set()
    for jd in devs:
        if not isinstance(jd.get("id"), str):
            _raise("MalformedDocument", "device entry needs a string id")
        if jd["id"] in seen:
            _raise("MalformedDocument", "duplicate device id")
        seen.add(jd["id"])
        if "budget_bytes" not in jd:
            _raise("MalformedDocument", "budget_bytes")
        b = _require_size(jd["budget_bytes"], "budget")
        ram = None
        if "ram_bytes" in jd:
            ram = _require_size(jd["ram_bytes"], "ram")
            if ram < b:
                _raise("MalformedDocument", "budget exceeds ram")
        out.append((jd["id"], b, ram))
    return out


def _parse_costs(jc, p, ctx):  # problem.cpp:92-101
    if not isinstance(jc, dict):
        _raise("MalformedDocument", ctx + " costs_ms must be an object")
    costs = [K_PROHIBITIVE_MS] * p.D
    for k, v in jc.items():
        d = p.find_device(k)
        if d < 0:
            _raise("UnknownDevice", k)
        costs[d] = _require_cost(v, ctx)
    return costs


def _parse_pair_key(key, p):  # problem.cpp:104-112
    if "->" not in key:
        _raise("MalformedDocument", "copy override key")
    a, b = key.split("->", 1)
    a, b = p.find_device(a), p.find_device(b)
    if a < 0 or b < 0:
        _raise("UnknownDevice", key)
    return (a, b)


def _parse_links(doc, p):  # problem.cpp:114-138
    if "links" not in doc:
        return []
    if not isinstance(doc["links"], list):
        _raise("MalformedDocument", "links must be an array")
    out = []
    for jl in doc["links"]:
        def res(f):
            v = jl[f]
            if not isinstance(v, str):
                _raise("MalformedDocument", "link endpoint")
            if v == "*":
                return -1
            d = p.find_device(v)
            if d < 0:
                _raise("UnknownDevice", v)
            return d
        fr, to = res("from"), res("to")
        lat = _require_cost(jl["latency_ms"], "latency")
        bpm = jl["bytes_per_ms"]
        if not _is_num(bpm) or bpm <= 0:
            _raise("NonPositiveSize", "bytes_per_ms")
        out.append((fr, to, lat, float(bpm)))
    return out


def validate_problem(p):  # problem.cpp:254-278
    if p.T == 0:
        _raise("EmptyNetwork", "no operators")
    if p.D == 0:
        _raise("MalformedDocument", "no devices")
    for op in p.ops:
        if len(op[2]) != p.D:
            _raise("DimensionMismatch", "cost vector size")
    seen = set()
    indeg = [0] * p.T
    for (s, d, _) in p.edges:
        if s < 0 or d < 0 or s >= p.T or d >= p.T:
            _raise("MalformedDocument", "edge endpoint out of range")
        if s >= d:
            _raise("NonTopologicalEdge", f"{s}->{d}")
        if (s, d) in seen:
            _raise("MalformedDocument", "duplicate edge")
        seen.add((s, d))
        indeg[d] += 1
    for v in range(1, p.T):
        if indeg[v] == 0:
            _raise("MalformedDocument", f"operator {v} has no incoming edge")


def make_training_graph(name, devices, links, layers, input_bytes, input_home):
    """problem.cpp:280-338. layers: list of (name, out, costs, bwd_out, bwd_costs)."""
    if not layers:
        _raise("EmptyNetwork", "no layers")
    if input_bytes <= 0:
        _raise("NonPositiveSize", "input_bytes")
    D = len(devices)
    if input_home < 0 or input_home >= D:
        _raise("UnknownDevice", "input home")
    L = len(layers)
    p = Problem(name=name, devices=list(devices), links=list(links))
    c0 = [K_PROHIBITIVE_MS] * D
    c0[input_home] = 0.0
    p.ops.append(("input", input_bytes, c0, input_home))
    for (nm, out, costs, _, _) in layers:
        if out <= 0:
            _raise("NonPositiveSize", nm)
        if len(costs) != D:
            _raise("DimensionMismatch", nm)
        if any(c < 0 for c in costs):
            _raise("NegativeCost", nm)
        p.ops.append((nm, out, list(costs), None))
    for k in range(L, 0, -1):
        nm, _, _, bo, bc = layers[k - 1]
        if bo <= 0:
            _raise("NonPositiveSize", nm)
        if len(bc) != D:
            _raise("DimensionMismatch", nm)
        if any(c < 0 for c in bc):
            _raise("NegativeCost", nm)
        p.ops.append((nm + "'", bo, list(bc), None))
    for k in range(L):
        p.edges.append((k, k + 1, {}))
    for j in range(L + 1, 2 * L + 1):
        k = 2 * L + 1 - j
        p.edges.append((j - 1, j, {}))
        p.edges.append((k - 1, j, {}))
    validate_problem(p)
    return p


def _load_layered(doc):  # problem.cpp:190-224
    shell = Problem(name=doc.get("name", "unnamed"))
    shell.devices = _parse_devices(doc)
    shell.links = _parse_links(doc, shell)
    if not isinstance(doc.get("input"), dict):
        _raise("MalformedDocument", "layer document needs an input object")
    ib = _require_size(doc["input"]["output_bytes"], "input")
    home = shell.find_device(doc["input"]["home"])
    if home < 0:
        _raise("UnknownDevice", "input home device")
    layers = []
    for jl in doc["layers"]:
        layers.append((jl["name"], _require_size(jl["output_bytes"], "out"),
                       _parse_costs(jl["costs_ms"], shell, "layer"),
                       _require_size(jl["backward_output_bytes"], "bwd"),
                       _parse_costs(jl["backward_costs_ms"], shell, "layer bwd")))
    p = make_training_graph(shell.name, shell.devices, shell.links, layers, ib, home)
    if "edge_copy_ms" in doc:
        ov = {}
        for k, v in doc["edge_copy_ms"].items():
            ov[_parse_pair_key(k, p)] = _require_cost(v, "edge_copy_ms")
        p.edges = [(s, d, dict(ov)) for (s, d, _) in p.edges]
    return p


def _load_direct(doc):  # problem.cpp:140-188
    p = Problem(name=doc.get("name", "unnamed"))
    p.devices = _parse_devices(doc)
    ops = doc.get("operators")
    if not isinstance(ops, list) or not ops:
        _raise("EmptyNetwork", "document has no operators")
    for jo in ops:
        if not isinstance(jo.get("name"), str):
            _raise("MalformedDocument", "operator entry needs a string name")
        b = _require_size(jo["output_bytes"], "op")
        costs = _parse_costs(jo["costs_ms"], p, "op")
        pin = None
        if "pinned" in jo:
            pin = p.find_device(jo["pinned"])
            if pin < 0:
                _raise("UnknownDevice", "pinned")
        p.ops.append((jo["name"], b, costs, pin))
    if "edges" in doc:
        if not isinstance(doc["edges"], list):
            _raise("MalformedDocument", "edges must be an array")
        for je in doc["edges"]:
            if isinstance(je, list):
                if len(je) != 2 or not _is_int(je[0]) or not _is_int(je[1]):
                    _raise("MalformedDocument", "edge array entry must be [src, dst]")
                p.edges.append((je[0], je[1], {}))
            elif isinstance(je, dict):
                ov = {}
                for k, v in je.get("copy_ms", {}).items():
                    ov[_parse_pair_key(k, p)] = _require_cost(v, "edge copy_ms")
                p.edges.append((je["src"], je["dst"], ov))
            else:
                _raise("MalformedDocument", "edge entry must be an array or object")
    validate_problem(p)
    return p


def load_problem(text: str) -> Problem:  # problem.cpp:228-244
    try:
        doc = json.loads(text)
    except ValueError as ex:
        _raise("MalformedDocument", str(ex))
    if not isinstance(doc, dict):
        _raise("MalformedDocument", "top level must be an object")
    try:
        if "layers" in doc:
            return _load_layered(doc)
        p = _load_direct(doc)
        p.links = _parse_links(doc, p)
        return p
    except (KeyError, TypeError) as ex:
        _raise("MalformedDocument", str(ex))


def copy_cost(p: Problem, e: int, d: int, d_to: int) -> float:  # problem.cpp:358-380
    if d == d_to:
        return 0.0
    ov = p.edges[e][2]
    if (d, d_to) in ov:
        return ov[(d, d_to)]
    best, best_rank = None, -1
    for l in p.links:
        if (l[0] != -1 and l[0] != d) or (l[1] != -1 and l[1] != d_to):
            continue
        rank = (1 if l[0] == d else 0) + (1 if l[1] == d_to else 0)
        if rank > best_rank:
            best, best_rank = l, rank
    if best is None:
        _raise("MissingLink", f"{d}->{d_to}")
    return best[2] + float(p.ops[p.edges[e][0]][1]) / best[3]


def save_all_budget(p):  # problem.cpp:340-344
    return sum(op[1] for op in p.ops)


def budget_percent(full: int, pct: float) -> int:  # problem.cpp:346-356
    if not (pct > 0.0) or pct > 100.0:
        _raise("PercentOutOfRange", str(pct))
    if full <= 0:
        _raise("NonPositiveSize", "full")
    if math.modf(pct)[0] == 0.0:
        return full * int(pct) // 100
    return int(math.floor(float(full) * pct / 100.0))


def with_budgets(p: Problem, budgets) -> Problem:  # problem.cpp:382-393
    if len(budgets) != p.D:
        _raise("DimensionMismatch", "budget vector size")
    q = Problem(p.name, [], list(p.ops), list(p.edges), list(p.links))
    for (id_, _, ram), b in zip(p.devices, budgets):
        if b <= 0:
            _raise("NonPositiveSize", "budget")
        q.devices.append((id_, int(b), max(ram, b) if ram is not None else None))
    return q


@dataclass
class Energy:
    alpha: float
    q: np.ndarray               # [D][T]
    dev_limit: dict             # d -> lim
    total_limit: Optional[float]
    board: float


def parse_energy(text: str, p: Problem) -> Optional[Energy]:  # model.cpp:314-367
    doc = json.loads(text)
    if "energy" not in doc:
        return None
    e = doc["energy"]
    if not isinstance(e, dict):
        _raise("MalformedDocument", "energy must be an object")
    alpha = float(e.get("alpha", 0.0))
    if not alpha >= 0:
        _raise("NegativeCost", "alpha")
    board = float(e.get("board_joules", 0.0))
    total = float(e["total_limit"]) if "total_limit" in e else None
    qj = e.get("q_joules")
    if not isinstance(qj, dict):
        _raise("IncompleteEnergyTable", "q_joules missing")
    for k in qj:
        if p.find_device(k) < 0:
            _raise("UnknownDevice", k)
    q = np.zeros((p.D, p.T))
    for d, dev in enumerate(p.devices):
        if dev[0] not in qj:
            _raise("IncompleteEnergyTable", dev[0])
        row = qj[dev[0]]
        if not isinstance(row, list) or len(row) != p.T:
            _raise("IncompleteEnergyTable", dev[0])
        q[d] = [float(x) for x in row]
    lim = {}
    for k, v in e.get("device_limit", {}).items():
        d = p.find_device(k)
        if d < 0:
            _raise("UnknownDevice", k)
        lim[d] = float(v)
    return Energy(alpha, q, lim, total, board)


# --------------------------------------------------------------------------
# Resolved arrays (the xe_problem_desc image)
# --------------------------------------------------------------------------
class DescC(C.Structure):
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


class Arrays:
    """Resolved problem arrays; .c is a ctypes xe_problem_desc over them."""

    def __init__(self, D, T, E, mass, cost, src, dst, w, budget, energy: Optional[Energy] = None):
        self.D, self.T, self.E = int(D), int(T), int(E)
        self.mass = np.ascontiguousarray(mass, dtype=np.int64)
        self.cost = np.ascontiguousarray(cost, dtype=np.float64).reshape(D, T)
        self.src = np.ascontiguousarray(src, dtype=np.int32)
        self.dst = np.ascontiguousarray(dst, dtype=np.int32)
        self.w = np.ascontiguousarray(w, dtype=np.float64).reshape(E, D, D)
        self.budget = np.ascontiguousarray(budget, dtype=np.int64)
        self.energy = energy
        self.q = np.zeros((D, T)) if energy is None else np.ascontiguousarray(energy.q, dtype=np.float64)
        self.has_lim = np.zeros(D, np.uint8)
        self.lim = np.zeros(D)
        if energy is not None:
            for d, v in energy.dev_limit.items():
                self.has_lim[d] = 1
                self.lim[d] = v
        self.c = DescC(
            self.D, self.T, self.E, self.mass.ctypes.data, self.cost.ctypes.data,
            self.src.ctypes.data, self.dst.ctypes.data, self.w.ctypes.data,
            self.budget.ctypes.data, 1 if energy is not None else 0,
            energy.alpha if energy else 0.0, self.q.ctypes.data, self.has_lim.ctypes.data,
            self.lim.ctypes.data, 1 if (energy and energy.total_limit is not None) else 0,
            energy.total_limit if (energy and energy.total_limit is not None) else 0.0,
            energy.board if energy else 0.0)

    @property
    def cube_words(self):
        return 2 * self.D * self.T * ((self.T + 31) // 32)

    def with_budgets(self, budgets):
        return Arrays(self.D, self.T, self.E, self.mass, self.cost, self.src, self.dst, self.w,
                      budgets, self.energy)


def arrays_of(p: Problem, energy: Optional[Energy] = None) -> Arrays:
    D, T, E = p.D, p.T, p.E
    w = np.zeros((E, D, D))
    for e in range(E):
        for a in range(D):
            for b in range(D):
                w[e, a, b] = copy_cost(p, e, a, b)
    return Arrays(D, T, E, [op[1] for op in p.ops], [[op[2][d] for op in p.ops] for d in range(D)],
                  [e[0] for e in p.edges], [e[1] for e in p.edges], w,
                  [dv[1] for dv in p.devices], energy)


def arrays_from_json(text: str) -> Arrays:
    p = load_problem(text)
    return arrays_of(p, parse_energy(text, p))


# --------------------------------------------------------------------------
# liboracle.so (C restatement)
# --------------------------------------------------------------------------
class _Model(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("nnz", C.c_int64), ("n_cols", C.c_int64),
                ("row_ptr", C.c_void_p), ("col", C.c_void_p), ("val", C.c_void_p),
                ("rhs", C.c_void_p), ("sense", C.c_void_p), ("tag", C.c_void_p),
                ("ordinal", C.c_void_p), ("obj", C.c_void_p), ("obj_present", C.c_void_p),
                ("fixed", C.c_void_p)]


def _np(ptr, n, dt):
    if n == 0:
        return np.zeros(0, dt)
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(np.ctypeslib.as_ctypes_type(dt))),
                                 shape=(n,)).copy()


@dataclass
class Model:
    n_rows: int
    nnz: int
    n_cols: int
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray
    rhs: np.ndarray
    sense: np.ndarray
    tag: np.ndarray
    ordinal: np.ndarray
    obj: np.ndarray
    obj_present: np.ndarray
    fixed: np.ndarray


class Oracle:
    """Bindings to oracle/liboracle.so (built by `make -C oracle`)."""

    def __init__(self, path=None):
        path = path or os.path.join(HERE, "liboracle.so")
        self.L = C.CDLL(path)
        L = self.L
        L.xo_build_model.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(_Model)]
        L.xo_model_free.argtypes = [C.POINTER(_Model)]
        L.xo_write_mps.argtypes = [C.c_void_p, C.POINTER(_Model), C.c_int, C.POINTER(C.c_size_t)]
        L.xo_write_mps.restype = C.c_void_p
        L.xo_eval_cubes.argtypes = [C.c_void_p, C.POINTER(_Model), C.c_int, C.c_int, C.c_void_p,
                                    C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.xo_eval_placements.argtypes = [C.c_void_p, C.POINTER(_Model), C.c_void_p, C.c_int64,
                                         C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        L.xo_assignment_oracle.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]
        L.xo_assignment_oracle.restype = C.c_double
        L.xo_format_number.argtypes = [C.c_double, C.c_char_p, C.c_size_t]
        L.xo_complete.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        self._free = C.CDLL(None).free
        self._free.argtypes = [C.c_void_p]

    def _model_c(self, a: Arrays, strict, energy):
        m = _Model()
        self.L.xo_build_model(C.byref(a.c), int(strict), int(energy), C.byref(m))
        return m

    def build_model(self, a: Arrays, strict=False, energy=False) -> Model:
        m = self._model_c(a, strict, energy)
        try:
            out = Model(m.n_rows, m.nnz, m.n_cols,
                        _np(m.row_ptr, m.n_rows + 1, np.int64), _np(m.col, m.nnz, np.int32),
                        _np(m.val, m.nnz, np.float64), _np(m.rhs, m.n_rows, np.float64),
                        _np(m.sense, m.n_rows, np.int8), _np(m.tag, m.n_rows, np.uint8),
                        _np(m.ordinal, m.n_rows, np.int32), _np(m.obj, m.n_cols, np.float64),
                        _np(m.obj_present, m.n_cols, np.uint8), _np(m.fixed, m.n_cols, np.uint8))
        finally:
            self.L.xo_model_free(C.byref(m))
        return out

    def write_mps(self, a: Arrays, strict=False, quad=False, energy=False) -> bytes:
        m = self._model_c(a, strict, energy)
        n = C.c_size_t()
        p = self.L.xo_write_mps(C.byref(a.c), C.byref(m), int(quad), C.byref(n))
        s = C.string_at(p, n.value)
        self._free(p)
        self.L.xo_model_free(C.byref(m))
        return s

    def format_number(self, v: float) -> str:
        buf = C.create_string_buffer(64)
        self.L.xo_format_number(v, buf, 64)
        return buf.value.decode()

    def eval_cubes(self, a: Arrays, cubes: np.ndarray, strict=False, energy=False):
        cubes = np.ascontiguousarray(cubes, dtype=np.uint32).reshape(-1, a.cube_words)
        n = cubes.shape[0]
        obj = np.zeros(n)
        peak = np.zeros((n, a.D), np.int64)
        flags = np.zeros(n, np.uint32)
        m = self._model_c(a, strict, energy)
        self.L.xo_eval_cubes(C.byref(a.c), C.byref(m), int(strict), int(energy),
                             cubes.ctypes.data, n, obj.ctypes.data, peak.ctypes.data,
                             flags.ctypes.data)
        self.L.xo_model_free(C.byref(m))
        return obj, peak, flags

    def eval_placements(self, a: Arrays, dev: np.ndarray, policy=0):
        dev = np.ascontiguousarray(dev, dtype=np.uint8).reshape(-1, a.T)
        n = dev.shape[0]
        obj = np.zeros(n)
        peak = np.zeros((n, a.D), np.int64)
        flags = np.zeros(n, np.uint32)
        m = self._model_c(a, False, False)
        self.L.xo_eval_placements(C.byref(a.c), C.byref(m), dev.ctypes.data, n, int(policy),
                                  obj.ctypes.data, peak.ctypes.data, flags.ctypes.data)
        self.L.xo_model_free(C.byref(m))
        return obj, peak, flags

    def complete(self, a: Arrays, cube: np.ndarray, strict=False):
        n_cols = 4 * a.D * a.T * a.T + a.D * a.T * (a.E + a.T) + a.T * a.E * a.D * (a.D - 1)
        x = np.zeros(n_cols)
        cube = np.ascontiguousarray(cube, dtype=np.uint32)
        self.L.xo_complete(C.byref(a.c), int(strict), cube.ctypes.data, x.ctypes.data)
        return x

    def assignment_oracle(self, a: Arrays):
        dev = np.zeros(a.T, np.int32)
        n = C.c_int64()
        obj = self.L.xo_assignment_oracle(C.byref(a.c), dev.ctypes.data, C.byref(n))
        return obj, dev, n.value


# --------------------------------------------------------------------------
# oracle/_ref/libxengine_ref.so (the reference itself)
# --------------------------------------------------------------------------
REF_PATH = os.path.join(HERE, "_ref", "libxengine_ref.so")


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


class RefError(Exception):
    pass


class Ref:
    """Bindings to the unmodified reference library (oracle/ref_harness.cpp)."""

    def __init__(self, path=REF_PATH):
        self.L = C.CDLL(path)
        L = self.L
        L.xr_last_error.restype = C.c_char_p
        L.xr_problem_load.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        L.xr_problem_fixture.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        L.xr_problem_free.argtypes = [C.c_void_p]
        L.xr_problem_set_budgets.argtypes = [C.c_void_p, C.c_void_p]
        L.xr_problem_arrays.argtypes = [C.c_void_p] + [C.c_void_p] * 10
        L.xr_energy_arrays.argtypes = [C.c_void_p] + [C.c_void_p] * 7
        L.xr_write_mps.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int,
                                   C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]
        L.xr_model_csr.argtypes = [C.c_void_p, C.c_int, C.c_int] + [C.c_void_p] * 13
        L.xr_eval_cubes.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int64,
                                    C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        L.xr_eval_placements.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int,
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        L.xr_assignment_oracle.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.xr_solve_exact.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int64,
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.xr_format_number.argtypes = [C.c_double, C.c_char_p, C.c_int]
        L.xr_budget_percent.argtypes = [C.c_int64, C.c_double, C.c_void_p]
        L.xr_budget_percent.restype = C.c_int64
        L.xr_free.argtypes = [C.c_void_p]
        sp = [C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]
        L.xr_schedule.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p] + sp + sp + [C.c_void_p] * 3
        L.xr_validate_text.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p] + sp
        L.xr_replay_text.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_char_p] + sp + [C.c_void_p] * 3

    def _check(self, rc):
        if rc != 0:
            raise RefError(f"rc={rc}: {self.L.xr_last_error().decode()}")

    def load(self, text: str):
        h = C.c_void_p()
        self._check(self.L.xr_problem_load(text.encode(), C.byref(h)))
        return RefProblem(self, h)

    def fixture(self, name: str):
        h = C.c_void_p()
        self._check(self.L.xr_problem_fixture(name.encode(), C.byref(h)))
        return RefProblem(self, h)

    def format_number(self, v: float) -> str:
        buf = C.create_string_buffer(64)
        self.L.xr_format_number(v, buf, 64)
        return buf.value.decode()


class RefProblem:
    def __init__(self, ref: Ref, h):
        self.ref, self.h, self.L = ref, h, ref.L

    def __del__(self):
        try:
            self.L.xr_problem_free(self.h)
        except Exception:
            pass

    def set_budgets(self, budgets):
        b = np.ascontiguousarray(budgets, dtype=np.int64)
        self.ref._check(self.L.xr_problem_set_budgets(self.h, b.ctypes.data))

    def arrays(self) -> Arrays:
        D, T, E, he = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        z = None
        self.ref._check(self.L.xr_problem_arrays(self.h, C.byref(D), C.byref(T), C.byref(E),
                                                 z, z, z, z, z, z, C.byref(he)))
        D, T, E = D.value, T.value, E.value
        mass = np.zeros(T, np.int64)
        cost = np.zeros((D, T))
        src = np.zeros(E, np.int32)
        dst = np.zeros(E, np.int32)
        w = np.zeros((E, D, D))
        bud = np.zeros(D, np.int64)
        self.ref._check(self.L.xr_problem_arrays(
            self.h, C.byref(C.c_int()), C.byref(C.c_int()), C.byref(C.c_int()),
            mass.ctypes.data, cost.ctypes.data, src.ctypes.data, dst.ctypes.data, w.ctypes.data,
            bud.ctypes.data, C.byref(C.c_int())))
        energy = None
        if he.value:
            alpha, tot, board = C.c_double(), C.c_double(), C.c_double()
            ht = C.c_int()
            q = np.zeros((D, T))
            hl = np.zeros(D, np.uint8)
            lim = np.zeros(D)
            self.ref._check(self.L.xr_energy_arrays(self.h, C.byref(alpha), q.ctypes.data,
                                                    hl.ctypes.data, lim.ctypes.data, C.byref(ht),
                                                    C.byref(tot), C.byref(board)))
            energy = Energy(alpha.value, q, {d: lim[d] for d in range(D) if hl[d]},
                            tot.value if ht.value else None, board.value)
        return Arrays(D, T, E, mass, cost, src, dst, w, bud, energy)

    def write_mps(self, strict=False, quad=False, energy=False) -> bytes:
        p, n = C.c_void_p(), C.c_size_t()
        self.ref._check(self.L.xr_write_mps(self.h, int(strict), int(quad), int(energy),
                                            C.byref(p), C.byref(n)))
        s = C.string_at(p, n.value)
        self.L.xr_free(p)
        return s

    def model_csr(self, strict=False, energy=False) -> Model:
        nr, nz, nc = C.c_int64(), C.c_int64(), C.c_int64()
        z = None
        self.ref._check(self.L.xr_model_csr(self.h, int(strict), int(energy), C.byref(nr),
                                            C.byref(nz), z, z, z, z, z, z, z, C.byref(nc), z, z, z))
        nr, nz, nc = nr.value, nz.value, nc.value
        rp = np.zeros(nr + 1, np.int64)
        col = np.zeros(nz, np.int32)
        val = np.zeros(nz)
        rhs = np.zeros(nr)
        sense = np.zeros(nr, np.int8)
        tag = np.zeros(nr, np.uint8)
        ordn = np.zeros(nr, np.int32)
        obj = np.zeros(nc)
        objp = np.zeros(nc, np.uint8)
        fixed = np.zeros(nc, np.uint8)
        self.ref._check(self.L.xr_model_csr(
            self.h, int(strict), int(energy), C.byref(C.c_int64()), C.byref(C.c_int64()),
            rp.ctypes.data, col.ctypes.data, val.ctypes.data, rhs.ctypes.data, sense.ctypes.data,
            tag.ctypes.data, ordn.ctypes.data, C.byref(C.c_int64()), obj.ctypes.data,
            objp.ctypes.data, fixed.ctypes.data))
        return Model(nr, nz, nc, rp, col, val, rhs, sense, tag, ordn, obj, objp, fixed)

    def eval_cubes(self, cubes: np.ndarray, D: int, strict=False, energy=False, check=True,
                   decode=True, nthreads=1):
        cubes = np.ascontiguousarray(cubes, dtype=np.uint32)
        n = cubes.shape[0]
        obj = np.zeros(n)
        peak = np.zeros((n, D), np.int64)
        flags = np.zeros(n, np.uint32)
        self.ref._check(self.L.xr_eval_cubes(self.h, int(strict), int(energy), cubes.ctypes.data,
                                             n, int(check), int(decode), obj.ctypes.data,
                                             peak.ctypes.data, flags.ctypes.data, int(nthreads)))
        return obj, peak, flags

    def eval_placements(self, dev: np.ndarray, D: int, policy=0, check=True, nthreads=1):
        dev = np.ascontiguousarray(dev, dtype=np.uint8)
        n = dev.shape[0]
        obj = np.zeros(n)
        peak = np.zeros((n, D), np.int64)
        flags = np.zeros(n, np.uint32)
        self.ref._check(self.L.xr_eval_placements(self.h, dev.ctypes.data, n, int(policy),
                                                  int(check), obj.ctypes.data, peak.ctypes.data,
                                                  flags.ctypes.data, int(nthreads)))
        return obj, peak, flags

    def assignment_oracle(self, T):
        obj = C.c_double()
        dev = np.zeros(T, np.int32)
        nodes = C.c_int64()
        self.ref._check(self.L.xr_assignment_oracle(self.h, C.byref(obj), dev.ctypes.data,
                                                    C.byref(nodes)))
        return obj.value, dev, nodes.value

    def _take(self, p, n):
        b = C.string_at(p, n.value).decode()
        self.L.xr_free(p)
        return b

    def schedule(self, cube, D, strict=False, energy=False):
        """decode -> format_schedule, replay(assignment) -> trace_csv,
        total_action_ms, eq1_objective_ms, peaks (schedule.cpp:40-530)."""
        t, tl, c, cl = C.c_void_p(), C.c_size_t(), C.c_void_p(), C.c_size_t()
        tot, eq1 = C.c_double(), C.c_double()
        peaks = np.zeros(D, np.int64)
        cube = np.ascontiguousarray(cube, np.uint32)
        self.ref._check(self.L.xr_schedule(self.h, int(strict), int(energy), cube.ctypes.data, C.byref(t), C.byref(tl),
                                           C.byref(c), C.byref(cl), C.byref(tot), C.byref(eq1), peaks.ctypes.data))
        return self._take(t, tl), self._take(c, cl), tot.value, eq1.value, peaks

    def validate_text(self, text, budgets=None):
        """validate(parse_schedule(text)) -> ["kind device t slot bytes|detail", ...]"""
        o, ol = C.c_void_p(), C.c_size_t()
        b = None if budgets is None else np.ascontiguousarray(budgets, np.int64)
        self.ref._check(self.L.xr_validate_text(self.h, text.encode(), None if b is None else b.ctypes.data,
                                                C.byref(o), C.byref(ol)))
        return [x for x in self._take(o, ol).split("\n") if x]

    def replay_text(self, text, D, strict=False, energy=False):
        c, cl, tot, eq1 = C.c_void_p(), C.c_size_t(), C.c_double(), C.c_double()
        peaks = np.zeros(D, np.int64)
        self.ref._check(self.L.xr_replay_text(self.h, int(strict), int(energy), text.encode(), C.byref(c),
                                              C.byref(cl), C.byref(tot), C.byref(eq1), peaks.ctypes.data))
        return self._take(c, cl), tot.value, eq1.value, peaks

    def solve_exact(self, D, T, strict=False, energy=False, budgets=None, node_limit=0):
        st, obj, nodes = C.c_int(), C.c_double(), C.c_int64()
        cube = np.zeros(2 * D * T * ((T + 31) // 32), np.uint32)
        b = None if budgets is None else np.ascontiguousarray(budgets, dtype=np.int64)
        self.ref._check(self.L.xr_solve_exact(self.h, int(strict), int(energy),
                                              None if b is None else b.ctypes.data,
                                              int(node_limit), C.byref(st), C.byref(obj),
                                              cube.ctypes.data, C.byref(nodes)))
        return st.value, obj.value, cube, nodes.value
