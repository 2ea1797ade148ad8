# SPDX-License-Identifier: Apache-2.0
"""GPU decode / validate / replay / trace_csv (csrc/schedule.cu,
schedule_text.cpp) against the reference's own schedule.cpp run through the
unmodified compiled library (oracle/_ref): the same action list text
(format_schedule), the same violations, the same trace CSV bytes, totals and
peaks — for the exact optima of the reference's fixtures and random DAGs
(tests/golden/exact_pins.json), for the top-K of an evaluated VGG-16 batch,
and for illegal assignments (the same IllegalAssignment message)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import xo

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_2212_09290_b200 as xe  # noqa: E402
from paper_2212_09290_b200 import schedule as sch  # noqa: E402


@pytest.fixture(scope="module")
def ref():
    try:
        return xo.Ref()
    except OSError as e:
        pytest.skip(f"oracle/_ref not built: {e}")


def _pins():
    with open(os.path.join(GOLDEN, "exact_pins.json")) as f:
        return [c for c in json.load(f)["cases"] if c["status"] == "Optimal"]


def _same_as_reference(ref, text, cube, budgets=None, strict=False, energy=False):
    p = xe.Problem.from_json(text)
    rp = ref.load(text)
    if budgets:
        p = p.with_budgets(budgets)
        rp.set_budgets(budgets)
    opts = xe.ModelOptions(strict_free=strict, energy=energy)
    cube = np.asarray(cube, np.uint32)
    rtext, rcsv, rtot, req1, rpk = rp.schedule(cube, p.D, strict=strict, energy=energy)
    s = sch.decode(p, cube[None], opts)[0]
    assert s.error is None
    assert sch.format_schedule(p, s) == rtext
    assert sch.validate(p, [s])[0] == [] and rp.validate_text(rtext) == []
    tr = sch.replay(p, [s], opts)[0]
    assert sch.trace_csv(p, tr) == rcsv
    assert tr.total_action_ms == rtot
    assert tr.peaks.tolist() == rpk.tolist()
    # eq1 from availability: the reference's replay without an assignment
    _, rtot2, req2, _ = rp.replay_text(rtext, p.D, strict=strict, energy=energy)
    assert tr.eq1_objective_ms == req2 and rtot2 == rtot
    # parse_schedule(format_schedule(s)) == s
    back = sch.parse_schedule(p, rtext)
    assert np.array_equal(back.actions, s.actions)
    return p, s, tr


def test_fig2_exact_optimum_schedule(ref):
    # test_schedule.cpp:301-319: the exact optimum 11.0, peaks cpu 8 MiB / gpu 32 MiB, 49 samples per device
    c = [c for c in _pins() if c["tag"] == "fig2"][0]
    p, s, tr = _same_as_reference(ref, c["doc"], c["cube"])
    assert tr.peaks.tolist() == [8 << 20, 32 << 20]
    assert tr.memory.shape[1] * tr.memory.shape[2] == 49
    assert tr.total_action_ms == 11.0 and tr.eq1_objective_ms == 11.0


def test_all_exact_pins(ref):
    n_illegal = 0
    for c in _pins():
        try:
            _same_as_reference(ref, c["doc"], c["cube"], c["budgets"], c["strict"], c["energy"])
        except xo.RefError as e:
            # some exact optima do not decode under the default hazard:
            # the GPU decode raises the same IllegalAssignment
            assert "IllegalAssignment" in str(e)
            p = xe.Problem.from_json(c["doc"])
            if c["budgets"]:
                p = p.with_budgets(c["budgets"])
            s = sch.decode(p, np.asarray(c["cube"], np.uint32)[None],
                           xe.ModelOptions(strict_free=c["strict"], energy=c["energy"]))[0]
            assert s.error is not None and s.error in str(e), (c["tag"], s.error, str(e))
            n_illegal += 1
    assert n_illegal < len(_pins())


def test_validate_mutated_schedules_same_violations(ref):
    # drop / retarget / reorder action lines of the optimal schedules; every
    # violation (kind, device, timestep, slot, bytes) as the reference reports it
    rng = np.random.default_rng(3)
    kinds = {k: i for i, k in enumerate(sch.VIOLATION_KINDS)}
    n = 0
    for c in _pins()[:40]:
        p = xe.Problem.from_json(c["doc"])
        rp = ref.load(c["doc"])
        try:
            lines = rp.schedule(np.asarray(c["cube"], np.uint32), p.D, strict=c["strict"],
                                energy=c["energy"])[0].splitlines()
        except xo.RefError:
            continue  # not decodable under the default hazard
        for trial in range(6):
            mut = list(lines)
            j = int(rng.integers(len(mut)))
            if trial % 3 == 0:
                del mut[j]
            elif trial % 3 == 1 and p.D > 1:
                import re
                names = p.names()["devices"]
                m = re.search(r"\b(d|from|to)=(\S+)", mut[j])
                if m:
                    nd = names[(names.index(m.group(2)) + 1) % p.D]
                    mut[j] = mut[j][:m.start(2)] + nd + mut[j][m.end(2):]
            else:  # swap two lines
                k2 = int(rng.integers(len(mut)))
                mut[j], mut[k2] = mut[k2], mut[j]
            text = "\n".join(mut) + "\n"
            budgets = [int(b) // 2 for b in p.arrays()["budget_bytes"]] if trial == 5 else None
            want = rp.validate_text(text, budgets)
            got = sch.validate(p, [sch.parse_schedule(p, text)], budgets)[0]
            w = [tuple(int(x) for x in v.split("|")[0].split()[1:]) + (v.split()[0],) for v in want]
            g = [(v.device, v.timestep, v.slot, v.bytes, v.kind) for v in got]
            assert g == w, (c["tag"], text, want, got)
            n += len(want)
    assert n > 0 and kinds


def test_vgg16_topk_batch_schedules(ref):
    # the top-32 valid candidates of an evaluated K4 batch: GPU decode + replay
    # of the whole batch in one call each, every artifact equal to the reference's
    from bench import configs
    from paper_2212_09290_b200.search import DEFAULT_MASK
    text = configs.vgg16_doc()
    p = xe.Problem.from_json(text)
    rp = ref.load(text)
    cubes = xe.round_cubes(p, 1 << 14, seed=5, edits=3, perturb=0.0)
    res = xe.evaluate_cubes(p, cubes, valid_mask=DEFAULT_MASK)
    ok = (res.flags.to(torch.int64) & DEFAULT_MASK) == 0
    top = torch.argsort(torch.where(ok, res.obj, torch.full_like(res.obj, float("inf"))), stable=True)[:32]
    host = cubes[top].cpu().numpy().view(np.uint32)
    scheds = sch.decode(p, host)
    assert all(s.error is None for s in scheds)
    traces = sch.replay(p, scheds)
    peaks = res.peak[top].cpu().numpy()
    for k in range(len(scheds)):
        rtext, rcsv, rtot, _, rpk = rp.schedule(host[k], p.D)
        assert sch.format_schedule(p, scheds[k]) == rtext
        assert sch.trace_csv(p, traces[k]) == rcsv and traces[k].total_action_ms == rtot
        assert traces[k].peaks.tolist() == rpk.tolist() == peaks[k].tolist()  # = K2's U peaks


def test_illegal_assignments_same_error(ref):
    # random bit cubes on fig2: decode raises IllegalAssignment exactly where the
    # reference does, with the same message (schedule.cpp:57-71)
    import cubegen
    text = json.dumps(json.load(open(os.path.join(GOLDEN, "problems", "fig2.json"))))
    p = xe.Problem.from_json(text)
    rp = ref.load(text)
    a = xo.arrays_from_json(text)
    cubes = cubegen.mixed_cubes(a, 300, seed=9, random_frac=0.5)
    scheds = sch.decode(p, cubes)
    bad = 0
    for k, s in enumerate(scheds):
        try:
            rtext = rp.schedule(cubes[k], p.D)[0]
            assert s.error is None and sch.format_schedule(p, s) == rtext
        except xo.RefError as e:
            if "IllegalAssignment" not in str(e):
                continue  # replay's IllegalSchedule: decode itself succeeded
            bad += 1
            assert s.error is not None and s.error in str(e), (s.error, str(e))
    assert bad > 0
