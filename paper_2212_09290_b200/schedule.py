# SPDX-License-Identifier: Apache-2.0
"""Schedules of candidate cubes on the GPU: the Python mirror of
proj/include/xengine/schedule.hpp (decode / validate / replay /
format_schedule / parse_schedule / trace_csv / memory_timeline), batched over
the top-K of an evaluated candidate set (csrc/schedule.cu, schedule_text.cpp).

    sched = decode(problem, cubes)          # one Schedule per cube (IllegalAssignment -> Schedule.error)
    reports = validate(problem, sched)      # [[Violation, ...] per schedule]
    traces = replay(problem, sched)         # Trace: total_action_ms, eq1_objective_ms, memory, peaks
    text = format_schedule(problem, sched[0]); csv = trace_csv(problem, traces[0])
"""
import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib
from ._lib import LIB, XeError, check
from .api import ModelOptions, Problem

ACTION_KINDS = ("Compute", "Copy", "Free", "Drop")            # ActionKind order (schedule.hpp:19)
VIOLATION_KINDS = ("ComputeWithoutInputs", "CopyFromNonResident", "BudgetExceeded", "FreeNonResident",
                   "UncomputedOperator")                      # ViolationKind order (schedule.hpp:42-48)


@dataclass
class Schedule:
    actions: np.ndarray               # structured xe_action records (kind, timestep, slot, device, op, src, dst, from_, to)
    error: Optional[str] = None       # IllegalAssignment message when the decode raised (then no actions)


@dataclass
class Violation:
    kind: str
    device: int
    timestep: int
    slot: int
    bytes: int
    a: int
    b: int


@dataclass
class Trace:
    total_action_ms: float
    eq1_objective_ms: float
    memory: np.ndarray                # [D][T][T] bytes, one sample per (device, timestep, slot)
    peaks: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))


_ACT = np.dtype([("kind", "<i4"), ("timestep", "<i4"), ("slot", "<i4"), ("device", "<i4"), ("op", "<i4"),
                 ("src", "<i4"), ("dst", "<i4"), ("from_", "<i4"), ("to", "<i4")])


def _cat(scheds):
    acts = [s.actions for s in scheds]
    off = np.zeros(len(acts) + 1, np.int64)
    off[1:] = np.cumsum([len(a) for a in acts])
    flat = np.concatenate(acts) if acts and off[-1] else np.zeros(1, _ACT)
    return np.ascontiguousarray(flat), off


def _error_text(problem: Problem, e) -> str:
    names = problem.names()
    ops = names["ops"]
    if e.code == 1:
        return (f"operator {ops[e.v]} at t={e.t} needs tensor {ops[e.u]} resident on no device")
    return f"copy source for tensor {ops[e.u]} was freed earlier in timestep {e.t}"


def decode(problem: Problem, cubes: np.ndarray, opts: Optional[ModelOptions] = None) -> List[Schedule]:
    """decode(complete_assignment(R, S)) (schedule.cpp:40-129) for each
    canonical cube (uint32 words, [n][cube_words])."""
    cubes = np.ascontiguousarray(np.atleast_2d(cubes), np.uint32)
    n = cubes.shape[0]
    mo = (opts or ModelOptions()).c()
    off = np.zeros(n + 1, np.int64)
    err = (_lib.DecodeError * max(n, 1))()
    check(LIB.xe_decode_cubes(problem.handle, C.byref(mo), cubes.ctypes.data, n, off.ctypes.data, None, err))
    acts = np.zeros(max(int(off[-1]), 1), _ACT)
    check(LIB.xe_decode_cubes(problem.handle, C.byref(mo), cubes.ctypes.data, n, off.ctypes.data,
                              acts.ctypes.data, err))
    return [Schedule(acts[off[k]:off[k + 1]].copy(), _error_text(problem, err[k]) if err[k].code else None)
            for k in range(n)]


def validate(problem: Problem, scheds: List[Schedule], budgets=None) -> List[List[Violation]]:
    """validate (schedule.cpp:131-240): every violation of each schedule."""
    flat, off = _cat(scheds)
    n = len(scheds)
    b = None if budgets is None else np.ascontiguousarray(budgets, np.int64)
    voff = np.zeros(n + 1, np.int64)
    check(LIB.xe_validate_schedules(problem.handle, flat.ctypes.data, off.ctypes.data, n,
                                    None if b is None else b.ctypes.data, voff.ctypes.data, None))
    vs = (_lib.Violation * max(int(voff[-1]), 1))()
    check(LIB.xe_validate_schedules(problem.handle, flat.ctypes.data, off.ctypes.data, n,
                                    None if b is None else b.ctypes.data, voff.ctypes.data, vs))
    return [[Violation(VIOLATION_KINDS[v.kind], v.device, v.timestep, v.slot, v.bytes, v.a, v.b)
             for v in vs[voff[k]:voff[k + 1]]] for k in range(n)]


def replay(problem: Problem, scheds: List[Schedule], opts: Optional[ModelOptions] = None) -> List[Trace]:
    """replay (schedule.cpp:261-369) of legal schedules (IllegalSchedule
    otherwise, as the reference raises)."""
    reps = validate(problem, scheds)
    for r in reps:
        if r:
            raise XeError(23, f"{len(r)} violation(s), first: {r[0].kind}")
    flat, off = _cat(scheds)
    n, D, T = len(scheds), problem.D, problem.T
    tot, eq1 = np.zeros(max(n, 1)), np.zeros(max(n, 1))
    mem = np.zeros((max(n, 1), D, T, T), np.int64)
    pk = np.zeros((max(n, 1), D), np.int64)
    mo = (opts or ModelOptions()).c()
    check(LIB.xe_replay_schedules(problem.handle, C.byref(mo), flat.ctypes.data, off.ctypes.data, n,
                                  tot.ctypes.data, eq1.ctypes.data, mem.ctypes.data, pk.ctypes.data))
    return [Trace(float(tot[k]), float(eq1[k]), mem[k], pk[k]) for k in range(n)]


def _text(fn, *args) -> str:
    ln = C.c_size_t()
    check(fn(*args, None, C.byref(ln)))
    buf = C.create_string_buffer(ln.value + 1)
    check(fn(*args, buf, C.byref(ln)))
    return buf.raw[: ln.value].decode()


def format_schedule(problem: Problem, s: Schedule) -> str:
    """format_schedule (schedule.cpp:440-475), byte-identical."""
    a = np.ascontiguousarray(s.actions)
    return _text(LIB.xe_format_schedule, problem.handle, a.ctypes.data if len(a) else None, len(a))


def parse_schedule(problem: Problem, text: str) -> Schedule:
    """parse_schedule (schedule.cpp:477-521)."""
    n = C.c_int64(0)
    check(LIB.xe_parse_schedule(problem.handle, text.encode(), None, C.byref(n)))
    acts = np.zeros(max(n.value, 1), _ACT)
    check(LIB.xe_parse_schedule(problem.handle, text.encode(), acts.ctypes.data, C.byref(n)))
    return Schedule(acts[: n.value].copy())


def trace_csv(problem: Problem, tr: Trace) -> str:
    """trace_csv (schedule.cpp:523-530), byte-identical."""
    m = np.ascontiguousarray(tr.memory, np.int64)
    return _text(LIB.xe_trace_csv, problem.handle, m.ctypes.data)


def memory_timeline(tr: Trace, device: int):
    """memory_timeline (schedule.cpp:371-381): per timestep the max over its slots."""
    if device < 0 or device >= tr.memory.shape[0]:
        raise XeError(9, "device index out of range")
    return [(t, int(tr.memory[device, t].max())) for t in range(tr.memory.shape[1])]


def combined_memory_timeline(tr: Trace):
    """combined_memory_timeline (schedule.cpp:383-395)."""
    out = []
    for d in range(tr.memory.shape[0]):
        s = memory_timeline(tr, d)
        out = s if not out else [(a[0], a[1] + b[1]) for a, b in zip(out, s)]
    return out
