# SPDX-License-Identifier: Apache-2.0
"""Headline benchmark: candidate schedules evaluated per second (K2a) on the
BASELINE.json config 2 workload — VGG-16 training DAG (T=43, E=63), 2 devices
with a 25 % GPU budget, 10 M dense R/S candidate cubes resident in HBM.

  python bench.py [--gpus N --steps K --warmup W]          # this framework
  python bench.py --impl reference [...]                    # reference CPU path

One step = one evaluation pass (complete_assignment + objective_value +
check_assignment + peaks + decode legality, per candidate) over the whole
batch plus the best-of-batch reduction.  Prints ONE JSON line on rank 0.
Multi-GPU (torchrun): each rank owns its own 10 M candidates (weak scaling,
seed 2212, disjoint Philox index ranges); the incumbent is exchanged with an
all-reduce MIN over NCCL; time = max over ranks of CUDA-event time.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "candidate schedules evaluated/sec + PDHG iters/sec at 1/2/4/8 B200 vs CPU ref"
UNIT = "candidates/s"
SEED = 2212
WORKLOAD = "vgg16-train cfg2 dense R/S candidate evaluation (T=43, E=63, D=2, gpu budget 25%)"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def traffic_from_profiles(config, n):
    """DRAM bytes (read + write) per launch of n candidates, scaled from the
    per-candidate traffic of the committed ncu --set full capture; GB."""
    p = os.path.join(ROOT, "profiles", "k2a_traffic.json")
    if os.path.exists(p):
        d = json.load(open(p)).get(config)
        if d:
            return d["dram_bytes_per_candidate"] * n / 1e9
    return None


def issue_roofline(config, cand_per_s, clocks):
    """What bounds K2a: warp-instructions issued per candidate (committed ncu
    capture) x candidates/s against the SM issue peak (148 SMs x 4 schedulers
    x 1 warp-instruction per clock at the sampled SM clock)."""
    p = os.path.join(ROOT, "profiles", "k2a_traffic.json")
    d = json.load(open(p)).get(config) if os.path.exists(p) else None
    if not d or "warp_instructions_per_candidate" not in d:
        return None
    mhz = (clocks or {}).get("sm_mhz") or 1965.0
    peak = 148 * 4 * mhz * 1e6
    achieved = d["warp_instructions_per_candidate"] * cand_per_s
    return {"bound": "issue", "unit": "warp-instructions/s", "achieved": achieved, "peak": peak,
            "frac": achieved / peak, "warp_instructions_per_candidate": d["warp_instructions_per_candidate"],
            "ncu_issue_active_pct": d.get("issue_active_pct")}


def k4_sample(doc, m):
    """The first m candidates of the GPU arm's own workload (K4 round_cubes,
    seed 2212, 3 edits, 10 % flips: the same Philox indices), canonical
    layout on the host; the numpy mix of tests/cubegen.py without a GPU."""
    try:
        import torch
        if torch.cuda.is_available():
            import paper_2212_09290_b200 as xe
            prob = xe.Problem.from_json(doc)
            return xe.round_cubes(prob, m, SEED, edits=3, perturb=0.1).cpu().numpy().view(np.uint32), "k4"
    except Exception:
        pass
    from oracle import xo
    import cubegen
    return cubegen.mixed_cubes(xo.arrays_from_json(doc), m, seed=SEED, random_frac=0.0), "cubegen"


def cpu_reference_rate(doc, a, seconds=12.0, nthreads=None, cubes=None):
    """Reference library (oracle/_ref) on the host cores: per candidate
    complete_assignment + objective_value + check_assignment + peaks + decode
    legality (what K2 computes per candidate)."""
    from oracle import xo
    import cubegen
    nthreads = nthreads or os.cpu_count() or 1
    if xo.ref_available():
        rp = xo.Ref().load(doc)
        kind = "reference"
        run = lambda c: rp.eval_cubes(c, a.D, check=True, decode=True, nthreads=nthreads)
    else:  # the C restatement, one thread
        orc = xo.Oracle()
        kind, nthreads = "port", 1
        run = lambda c: orc.eval_cubes(a, c)
    if cubes is None:
        cubes = cubegen.mixed_cubes(a, max(64, 8 * nthreads), seed=SEED, random_frac=0.0)
    done, t0 = 0, time.perf_counter()
    while True:
        run(cubes)
        done += len(cubes)
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return done / el, kind, nthreads, done, el


def _timed(fn, warmup=1, reps=3):
    """median wall time of fn() in seconds after warmup calls (CUDA-synchronised)."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts)), r


def _event_ms(fn, reps=3, warmup=1, stream=None):
    """mean CUDA-event time of fn() on the current stream, ms."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        r = fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, r


def pdhg_iter_bytes(model, lp):
    """Algorithmic HBM bytes of one PDHG iteration (both half-steps): the two
    sliced matrices (coded: one 4-byte word per entry; else an index and an
    fp64 value, 12 bytes) plus the per-column / per-row operand and result
    vectors (coded adds the scalings and the scaled copies the products gather)."""
    if lp.coded:
        return 8 * model.nnz + 72 * model.n_cols + 57 * model.n_rows
    return 24 * model.nnz + 64 * model.n_cols + 41 * model.n_rows


def dense_config(name, doc_fn, n, hbm, want_lp=None, highs_recorded=None):
    """One dense-cube config (3 ResNet-50 / 4 U-Net) on one GPU: K1 model, K3
    PDHG to 1e-7 (HBM roofline of the half-steps), K4 LP-guided rounding and
    the K2 evaluation of the rounded batch (HBM roofline of the evaluator)."""
    import torch
    import paper_2212_09290_b200 as xe
    prob = xe.Problem.from_json(doc_fn())
    k1_wall, model = _timed(lambda: xe.build_model(prob), warmup=1, reps=1)
    mps_wall, mps_len = _timed(lambda: len(model.write_mps()), warmup=1, reps=3)
    lp = xe.pdhg_solve(model, tol=1e-7, max_iters=1000000, return_x=True)
    it_bytes = pdhg_iter_bytes(model, lp)
    x = torch.from_numpy(lp.x).cuda()
    gen_ms, cubes = _event_ms(lambda: xe.round_cubes(prob, n, SEED, edits=3, perturb=0.0, x=x), reps=1)
    il = xe.cubes_to_il(prob, cubes)
    del cubes
    mask = _lib_mask()
    out = (torch.empty(n, dtype=torch.float64, device="cuda"), torch.empty((n, prob.D), dtype=torch.int64, device="cuda"),
           torch.empty(n, dtype=torch.int32, device="cuda"))
    ev_ms, r = _event_ms(lambda: xe.evaluate_cubes_il(prob, il, n, valid_mask=mask, out=out, best=False), reps=5)
    bpc = 2 * prob.D * prob.T * ((prob.T + 63) // 64) * 8 + 8 + 8 * prob.D + 4
    ev_gbs = n * bpc / (ev_ms / 1e3) / 1e9
    d = {"workload": f"{name}: T={prob.T}, E={prob.E}, D={prob.D}",
         "k1_build": {"rows": model.n_rows, "cols": model.n_cols, "nnz": model.nnz, "device_ms": model.build_ms(),
                      "wall_ms": 1e3 * k1_wall,
                      "achieved_gbs": (12 * model.nnz + 8 * (model.n_rows + 1) + 26 * model.n_cols) / (model.build_ms() / 1e3) / 1e9},
         "write_mps": {"bytes": mps_len, "wall_ms": 1e3 * mps_wall,
                       "path": "device text emission (mps_device.cu) + download into the returned bytes"},
         "pdhg": {"metric": "PDHG iters/sec", "iters": lp.iters, "converged": lp.converged, "certified": lp.certified,
                  "iters_per_s": lp.iters / (lp.solve_ms / 1e3), "time_to_tol_ms": lp.solve_ms, "tol": 1e-7,
                  "objective": lp.primal_obj, "dual_bound": lp.dual_obj,
                  "roofline": {"bound": "hbm", "bytes_per_iter": it_bytes,
                               "entries": "coded (4 B)" if lp.coded else "fp64 (12 B)",
                               "achieved": it_bytes / (lp.ms_per_iter / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                               "frac": it_bytes / (lp.ms_per_iter / 1e3) / 1e9 / hbm}},
         "k4_rounding": {"candidates": n, "candidates_per_s": n / (gen_ms / 1e3)},
         "k2_eval": {"candidates": n, "candidates_per_s": n / (ev_ms / 1e3), "kernel_ms": ev_ms,
                     "layout": "xe_cube_il", "bytes_per_candidate": bpc,
                     "roofline": {"bound": "hbm", "achieved": ev_gbs, "peak": hbm, "unit": "GB/s", "frac": ev_gbs / hbm}}}
    if want_lp is not None:
        d["pdhg"]["highs_objective"] = want_lp
        d["pdhg"]["rel_err"] = abs(lp.primal_obj - want_lp) / want_lp
    if highs_recorded is not None:
        d["pdhg"]["highs_seconds_recorded"] = highs_recorded
    return d, prob


def placement_config(n, hbm):
    """Config 5 (random 2000-op DAG, D=8): K2b save-all placement sweep over n
    resident placements; HBM roofline plus the shared-memory gather roofline
    (every op and edge term is one gather of the per-device tables)."""
    import torch
    import paper_2212_09290_b200 as xe
    from bench import configs
    prob = xe.Problem.from_json(configs.random2000_doc())
    dev = xe.random_placements(prob, n, SEED)
    out = (torch.empty(n, dtype=torch.float64, device="cuda"), torch.empty((n, prob.D), dtype=torch.int64, device="cuda"),
           torch.empty(n, dtype=torch.int32, device="cuda"))
    ms, r = _event_ms(lambda: xe.evaluate_placements(prob, dev, policy=0, out=out), reps=5)
    bpc = prob.T + 8 + 8 * prob.D + 4
    rate = n / (ms / 1e3)
    gbs = rate * bpc / 1e9
    # gathers per placement: T compute-cost + T mass + E (src, dst device pair -> copy table)
    gathers = 2 * prob.T + prob.E
    props = torch.cuda.get_device_properties(0)
    sm_clock_ghz = 1.965
    lds_peak = props.multi_processor_count * 32 * sm_clock_ghz * 1e9  # one 4-byte shared-memory lane access per bank per clock
    return {"workload": f"random2000 cfg5: T={prob.T}, E={prob.E}, D={prob.D}, save-all placements",
            "placements": n, "placements_per_s": rate, "kernel_ms": ms, "sweep_1e9_seconds": 1e9 / rate,
            "best": {"obj_ms": r.best_obj, "index": r.best_index},
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                         "bytes_per_candidate": bpc},
            "gather_roofline": {"bound": "smem gather", "gathers_per_placement": gathers,
                                "achieved": rate * gathers, "peak": lds_peak, "unit": "gathers/s",
                                "frac": rate * gathers / lds_peak,
                                "peak_note": "148 SMs x 32 banks x 1 access/clock at 1965 MHz"},
            "issue_roofline": issue_roofline("random2000", rate, None)}


def reference_inrun(doc_vgg, doc_resnet):
    """The reference's own K1 (build_model) and MPS writer (write_mps) timed
    in this run on the host (oracle/_ref, one thread), and HiGHS on the
    VGG-16 LP relaxation (SciPy linprog on the reference model)."""
    from oracle import xo
    out = {}
    if not xo.ref_available():
        return {"unavailable": "oracle/_ref not built"}
    R = xo.Ref()
    for name, doc in (("vgg16", doc_vgg), ("resnet50", doc_resnet)):
        rp = R.load(doc)
        t0 = time.perf_counter()
        rp.model_csr()
        t_build = time.perf_counter() - t0
        t0 = time.perf_counter()
        mps = rp.write_mps()
        t_mps = time.perf_counter() - t0
        out[name] = {"build_model_ms": 1e3 * t_build, "build_model_plus_write_mps_ms": 1e3 * t_mps,
                     "mps_bytes": len(mps), "threads": 1}
    try:
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        from gen_lp_golden import lp_value
        v, dt = lp_value(xo.arrays_from_json(doc_vgg))
        out["vgg16"]["highs_lp_seconds"] = dt
        out["vgg16"]["highs_lp_objective"] = v
    except Exception as ex:  # scipy/HiGHS missing on the host
        out["vgg16"]["highs_lp_unavailable"] = str(ex)[:200]
    return out


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from bench import configs
    from oracle import xo
    import cubegen
    doc = configs.vgg16_doc()
    a = xo.arrays_from_json(doc)
    nthreads = os.cpu_count() or 1
    cubes, source = k4_sample(doc, max(64, 16 * nthreads))
    step_s = float(os.environ.get("XE_REF_STEP_S", "4"))
    for _ in range(args.warmup):
        cpu_reference_rate(doc, a, seconds=0.5, nthreads=nthreads, cubes=cubes)
    times, counts, kind = [], [], None
    for _ in range(args.steps):
        r, kind, nt, done, el = cpu_reference_rate(doc, a, seconds=step_s, nthreads=nthreads, cubes=cubes)
        times.append(el)
        counts.append(done)
    value = sum(counts) / sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+u32",
        "data": f"synthetic: the GPU arm's first candidates ({source}: K4 round_cubes, Philox seed 2212, "
                "3 edits, 10% flips)",
        "config": {"workload": WORKLOAD, "sample_per_step": int(np.mean(counts))},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": kind,
                         "sample": f"{int(np.mean(counts))} VGG-16 candidates per step, "
                                   "complete_assignment+objective_value+check_assignment+peaks+decode"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def resnet_pipeline(args):
    """BASELINE config 3: ResNet-50 training DAG (T=145, E=264, D=3).  K1
    assembles the MILP (1.02 M rows, 4.35 M nnz), K3 solves its LP relaxation
    (HiGHS IPM: 107.49787109375002 in 652 s on the host), K4 rounds the LP
    diagonal into candidate cubes and K2 evaluates them exactly; one step =
    one batch of n rounded candidates evaluated.  Single GPU (the LP stays on
    one device)."""
    import torch
    import paper_2212_09290_b200 as xe
    from bench import configs
    from bench.clocks import ClockSampler
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if int(os.environ.get("RANK", "0")) != 0:
        return
    torch.cuda.set_device(local)
    prob = xe.Problem.from_json(configs.resnet50_doc(), device=local)
    model = xe.build_model(prob)
    lp = xe.pdhg_solve(model, tol=1e-7, max_iters=1000000, return_x=True)
    want = 107.49787109375002
    x = torch.from_numpy(lp.x).cuda()
    n = min(args.n, 200_000)
    cubes = xe.round_cubes(prob, n, SEED, edits=3, perturb=0.0, x=x)
    mask = _lib_mask()
    step = lambda: xe.evaluate_cubes(prob, cubes, valid_mask=mask, outputs=False)
    for _ in range(args.warmup):
        r = step()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            r = step()
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    it_bytes = pdhg_iter_bytes(model, lp)
    hbm = peaks()[0]
    bpc = prob.cube_words * 4 + 8 + 8 * prob.D + 4
    line = {"metric": METRIC, "value": n / (ms / 1e3), "unit": "candidates/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64+u32",
            "data": "synthetic: ResNet-50 training DAG (bench/configs.py, Appendix B seed 3); candidates rounded from the PDHG LP diagonal (seed 2212)",
            "config": {"workload": "resnet50-train cfg3 LP relaxation + LP-guided rounding + dense evaluation (T=145, E=264, D=3)",
                       "candidates_per_step": n, "cube_bytes": prob.cube_words * 4},
            "best": {"obj_ms": r.best_obj, "index": r.best_index, "n_valid": r.n_valid, "lp_bound": lp.primal_obj},
            "roofline": {"bound": "hbm", "achieved": n * bpc / (ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                         "frac": n * bpc / (ms / 1e3) / 1e9 / hbm, "traffic": None, "bytes_per_candidate": bpc},
            "k1_build": {"rows": model.n_rows, "cols": model.n_cols, "nnz": model.nnz, "ms": model.build_ms()},
            "pdhg": {"iters": lp.iters, "converged": lp.converged, "certified": lp.certified,
                     "iters_per_s": lp.iters / (lp.solve_ms / 1e3), "time_to_tol_ms": lp.solve_ms, "tol": 1e-7,
                     "objective": lp.primal_obj, "highs_objective": want, "highs_seconds_recorded": 565.3,
                     "rel_err": abs(lp.primal_obj - want) / want,
                     "roofline": {"bound": "hbm", "bytes_per_iter": it_bytes,
                                  "achieved": it_bytes / (lp.ms_per_iter / 1e3) / 1e9, "peak": hbm, "unit": "GB/s"}},
            "clocks": clk.summary(), "gpu_launches": 2 * args.steps}
    if not args.skip_search:
        from paper_2212_09290_b200.search import search
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sr = search(prob, n_per_round=1 << 16, rounds=4, edits=6, seed=1, chain_n=256)
        torch.cuda.synchronize()
        line["search"] = {"workload": "resnet50 cfg3 best schedule: K1 -> K3 LP -> K4 rounding + R-space local search -> K2",
                          "objective": sr.objective, "rounding_objective": sr.rounding_objective,
                          "lp_bound": sr.lp_bound, "gap_to_lp": sr.objective / sr.lp_bound - 1.0,
                          "candidates_evaluated": sr.n_evaluated, "seconds": time.perf_counter() - t0,
                          "reference": "no optimum (solve_exact needs D*T <= 64; HiGHS cannot solve the MILP)"}
    print(json.dumps(line), flush=True)


def _lib_mask():
    from paper_2212_09290_b200 import _lib
    return _lib.F_CHECK_MASK | _lib.F_BUDGET | _lib.F_DECODE


def placement_sweep(args):
    """BASELINE config 5: synthetic 2000-op random DAG, 8 devices; K2b
    evaluates save-all placements (save_all_assignment + objective_value,
    solver.cpp:30-75) generated uniformly (xe_random_placements); one step =
    one batch of n placements resident in HBM.  The full 1B sweep is
    ceil(1e9 / n) such steps."""
    import torch
    import torch.distributed as dist
    import paper_2212_09290_b200 as xe
    from bench import configs
    from bench.clocks import ClockSampler
    from paper_2212_09290_b200.shard import exchange_best
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        from bench.dist import init_dist
        local = init_dist(local)
    else:
        torch.cuda.set_device(local)
    prob = xe.Problem.from_json(configs.random2000_doc(), device=local)
    n = min(args.n, 4_000_000)
    dev = xe.random_placements(prob, n, SEED, first=rank * n)
    out = (torch.empty(n, dtype=torch.float64, device="cuda"), torch.empty((n, prob.D), dtype=torch.int64, device="cuda"),
           torch.empty(n, dtype=torch.int32, device="cuda"))
    stream = torch.cuda.current_stream()
    step = lambda: xe.evaluate_placements(prob, dev, policy=0, out=out, stream=stream.cuda_stream)
    for _ in range(args.warmup):
        r = step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with ClockSampler(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            r = step()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    best_obj, best_idx = r.best_obj, r.best_index
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        inc = exchange_best(best_obj, best_idx, r.n_valid, offset=rank * n, device="cuda")
        best_obj, best_idx = inc.obj, inc.index
    ms = float(t[0])
    bpc = prob.T + 8 + 8 * prob.D + 4
    hbm = peaks()[0]
    achieved = n * bpc / (ms / 1e3) / 1e9
    line = {"metric": METRIC, "value": world * n / (ms / 1e3), "unit": "placements/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64+u8",
            "data": "synthetic: xe_random_placements (uniform over allowed devices), Philox seed 2212",
            "config": {"workload": "random 2000-op DAG cfg5 save-all placement sweep (T=2000, E=5987, D=8)",
                       "placements_per_gpu_step": n, "sweep_1e9_seconds": 1e9 / (world * n / (ms / 1e3)),
                       "parallelism": f"dp{world}"},
            "best": {"obj_ms": best_obj, "index": best_idx},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": None, "bytes_per_candidate": bpc},
            "clocks": clk.summary(), "gpu_launches": 2 * args.steps}
    if rank == 0 and not args.skip_search:
        from paper_2212_09290_b200.search import search_placements
        del dev
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sp = search_placements(prob, iters=1000)
        torch.cuda.synchronize()
        line["search"] = {"workload": "cfg5 best save-all placement: 4 M uniform placements, then 256 local-search "
                                      "chains x 1024 neighbours x 1000 iterations (K2b exact scoring)",
                          "objective": sp.objective, "random_sample_objective": sp.random_objective,
                          "placements_evaluated": sp.n_evaluated, "seconds": time.perf_counter() - t0,
                          "reference": "assignment_oracle stops at 4e6 placements (8^2000 here)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=10_000_000, help="candidates per GPU")
    ap.add_argument("--e2e-n", type=int, default=2_000_000, help="candidates per e2e step")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-pdhg", action="store_true")
    ap.add_argument("--skip-search", action="store_true")
    ap.add_argument("--skip-configs", action="store_true", help="skip the config 3/4/5 objects of the default line")
    ap.add_argument("--workload", default="vgg16", choices=["vgg16", "random2000", "resnet50"],
                    help="vgg16: BASELINE config 2 (the headline); random2000: config 5 placement sweep; "
                         "resnet50: config 3 (K1 + PDHG LP + LP-guided rounding + evaluation)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return reference_arm(args)
    if args.workload == "random2000":
        return placement_sweep(args)
    if args.workload == "resnet50":
        return resnet_pipeline(args)

    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        from bench.dist import init_dist
        local = init_dist(local)
    else:
        torch.cuda.set_device(local)

    import paper_2212_09290_b200 as xe
    from paper_2212_09290_b200 import _lib
    from bench import configs
    from bench.clocks import ClockSampler
    from paper_2212_09290_b200.shard import exchange_best

    doc = configs.vgg16_doc()
    prob = xe.Problem.from_json(doc, device=local)
    D, T = prob.D, prob.T
    n = args.n
    cube_bytes = prob.cube_words * 4
    # resident workload in the evaluator's native interleaved layout
    # (xe_cube_il): K4 generates canonical cubes chunk by chunk, each chunk is
    # transposed into its 32-candidate groups
    il_words_per_cand = 2 * D * T
    il = torch.empty(((n + 31) // 32) * 32 * il_words_per_cand, dtype=torch.int64, device="cuda")
    chunk = 1 << 20
    tmp = torch.empty((chunk, prob.cube_words), dtype=torch.int32, device="cuda")
    gen_ms = 0.0  # K4 generation of the workload (not part of the timed steps)
    for lo in range(0, n, chunk):
        m = min(chunk, n - lo)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        xe.round_cubes(prob, m, SEED, first=rank * n + lo, edits=3, perturb=0.1, out=tmp[:m])
        g1.record()
        xe.cubes_to_il(prob, tmp[:m], out=il[lo * il_words_per_cand:])
        torch.cuda.synchronize()
        gen_ms += g0.elapsed_time(g1)
    del tmp
    obj = torch.empty(n, dtype=torch.float64, device="cuda")
    pk = torch.empty((n, D), dtype=torch.int64, device="cuda")
    fl = torch.empty(n, dtype=torch.int32, device="cuda")
    out = (obj, pk, fl)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()

    def step():
        return xe.evaluate_cubes_il(prob, il, n, out=out, stream=stream.cuda_stream)

    for _ in range(args.warmup):
        r = step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    # ---- timed region: K full steps (kernel + best reduction + host read) ----
    with ClockSampler(local) as clk:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            r = step()
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        step_ms = ev0.elapsed_time(ev1) / args.steps
        # kernel-only durations for the roofline (no reduction, no host read)
        kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        for e0, e1 in kev:
            e0.record(stream)
            xe.evaluate_cubes_il(prob, il, n, out=out, stream=stream.cuda_stream, best=False)
            e1.record(stream)
        torch.cuda.synchronize()
        kern_ms = float(np.mean([e0.elapsed_time(e1) for e0, e1 in kev]))
    clocks = clk.summary()

    t = torch.tensor([step_ms, kern_ms], dtype=torch.float64, device="cuda")
    best_obj, best_idx = r.best_obj, r.best_index
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        # incumbent exchange: MIN of objective bits, then MIN global index
        # among ranks holding it, SUM of valid counts (shard.py)
        inc = exchange_best(best_obj, best_idx, r.n_valid, offset=rank * n, device="cuda")
        best_obj, best_idx = inc.obj, inc.index
    step_ms, kern_ms = float(t[0]), float(t[1])
    value = world * n / (step_ms / 1e3)

    bytes_per_cand = il_words_per_cand * 8 + 8 + 8 * D + 4
    hbm, peak_kind = peaks()
    achieved = n * bytes_per_cand / (kern_ms / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64+u32",
        "data": "synthetic: K4 round_cubes (placement + minimal-save + <=3 recompute edits + 10% bit flips), Philox seed 2212",
        "config": {"workload": WORKLOAD,
                   "candidates_per_gpu": n, "cube_bytes": cube_bytes, "resident_bytes_per_gpu": n * cube_bytes,
                   "l2": "inputs (13.8 GB) larger than L2 (126 MB); no flush needed",
                   "layout": "xe_cube_il (candidate-interleaved, 32-candidate groups)",
                   "parallelism": f"dp{world} (candidate shards, NCCL all-reduce MIN incumbent)"},
        "best": {"obj_ms": best_obj, "index": best_idx, "n_valid_rank0": r.n_valid},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic_from_profiles("vgg16", n), "traffic_unit": "GB per launch",
                     "algorithmic_gb_per_launch": n * bytes_per_cand / 1e9,
                     "peak_kind": peak_kind, "kernel_ms": kern_ms,
                     "bytes_per_candidate": bytes_per_cand,
                     "issue": issue_roofline("vgg16", n / (kern_ms / 1e3), clocks)},
        "clocks": clocks,
        "gpu_launches": 2 * args.steps,
        "k4_generation": {"what": "K4 round_cubes of this workload (placement + minimal-save + 3 edits + 10 % flips)",
                          "candidates_per_s": n / (gen_ms / 1e3) if gen_ms > 0 else None, "ms": gen_ms},
    }

    # ---- end-to-end: host (pinned) cubes through the C ABI, best read back ----
    if not args.skip_e2e:
        ne = min(args.e2e_n, n)
        host = torch.empty((ne, prob.cube_words), dtype=torch.int32, pin_memory=True)
        tmp = torch.empty((chunk, prob.cube_words), dtype=torch.int32, device="cuda")
        for lo in range(0, ne, chunk):
            m = min(chunk, ne - lo)
            xe.round_cubes(prob, m, SEED, first=rank * n + lo, edits=3, perturb=0.1, out=tmp[:m])
            host[lo:lo + m].copy_(tmp[:m])
        del tmp
        hnp = host.numpy()
        xe.evaluate_cubes_host(prob, hnp[: min(ne, 100000)], outputs=False)
        ts = []
        for _ in range(max(3, args.steps // 2)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            re = xe.evaluate_cubes_host(prob, hnp, outputs=False)
            ts.append(time.perf_counter() - t0)
        e2e_s = float(np.median(ts))
        tt = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        line["e2e"] = {"value": world * ne / float(tt[0]), "unit": UNIT,
                       "h2d_bytes_per_step": ne * cube_bytes, "d2h_bytes_per_step": 24 * ((ne + (1 << 20) - 1) // (1 << 20)),
                       "candidates_per_step": ne, "path": "xe_eval_cubes_host (canonical cubes in a pinned host buffer; 2-stream chunked H2D, on-device transpose, lane-per-candidate evaluator)"}
        assert re.best_index == -1 or re.best_index < ne
        # the same call returning every candidate's objective, peaks and flags
        # to host arrays (the complete per-candidate contract of xe_eval_cubes)
        ts = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ro = xe.evaluate_cubes_host(prob, hnp, outputs=True)
            ts.append(time.perf_counter() - t0)
        eo = float(np.median(ts))
        to = torch.tensor([eo], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(to, op=dist.ReduceOp.MAX)
        line["e2e_outputs"] = {"value": world * ne / float(to[0]), "unit": UNIT, "h2d_bytes_per_step": ne * cube_bytes,
                               "d2h_bytes_per_step": ne * (8 + 8 * D + 4), "candidates_per_step": ne,
                               "path": "xe_eval_cubes_host with per-candidate objective, peaks and flags copied to host arrays"}
        assert ro.best_index == re.best_index

    # ---- K1 + K3 on the same config: GPU model assembly, PDHG LP relaxation ----
    if rank == 0 and not args.skip_pdhg:
        hbm_gbs = peaks()[0]
        model = xe.build_model(prob)
        build_ms = model.build_ms()
        k1_bytes = 12 * model.nnz + 8 * (model.n_rows + 1) + 26 * model.n_cols
        lp = xe.pdhg_solve(model, tol=1e-7, max_iters=400000)
        want = 118.68224203657523  # HiGHS 1.12.0 on the reference MPS (tests/golden/lp_values.json)
        it_bytes = pdhg_iter_bytes(model, lp)
        line["k1_build"] = {"rows": model.n_rows, "cols": model.n_cols, "nnz": model.nnz, "ms": build_ms,
                            "achieved_gbs": k1_bytes / (build_ms / 1e3) / 1e9 if build_ms > 0 else None}
        line["pdhg"] = {
            "metric": "PDHG iters/sec", "workload": "vgg16 cfg2 LP relaxation (K1 model, binaries in [0,1])",
            "iters": lp.iters, "restarts": lp.restarts, "converged": lp.converged, "certified": lp.certified,
            "iters_per_s": lp.iters / (lp.solve_ms / 1e3) if lp.solve_ms > 0 else None,
            "time_to_tol_ms": lp.solve_ms, "tol": 1e-7, "objective": lp.primal_obj, "highs_objective": want,
            "rel_err": abs(lp.primal_obj - want) / want,
            "roofline": {"bound": "hbm", "bytes_per_iter": it_bytes,
                         "achieved": it_bytes / (lp.ms_per_iter / 1e3) / 1e9 if lp.ms_per_iter > 0 else None,
                         "peak": hbm_gbs, "unit": "GB/s"},
        }

    # ---- the search on the same config: time to the reference's MILP optimum ----
    if rank == 0 and not args.skip_search:
        from paper_2212_09290_b200.search import search
        opt = 128.32908933333337  # reference solve_external (HiGHS MILP, 86 s on the host), SURVEY §8c
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sr = search(prob, xe.ModelOptions(strict_free=True), n_per_round=1 << 20, rounds=2, edits=6, seed=1)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        line["search"] = {
            "workload": "vgg16 cfg2 strict_free best schedule: K1 -> K3 LP -> K4 rounding + R-space local-search "
                        "population -> K2 exact scoring (wall clock, one GPU)",
            "objective": sr.objective, "reference_milp_optimum": opt, "equal_to_reference": sr.objective == opt,
            "peaks": [int(v) for v in sr.peaks] if sr.peaks is not None else None,
            "reference_peaks": [26894336, 60411904], "lp_bound": sr.lp_bound, "rounding_objective": sr.rounding_objective,
            "candidates_evaluated": sr.n_evaluated, "seconds": dt,
            "reference_milp_seconds_recorded": {"seconds": 86.0, "how": "solve_external + HiGHS MILP on the reference "
                                                                    "MPS, survey-measured (SURVEY §8c cfg-2 row); too "
                                                                    "slow to repeat inside the bench"}}

    # ---- the other BASELINE configs on this GPU (rank 0, N = 1): 3 ResNet-50,
    # 4 U-Net (K1 + K3 + K4 + K2 on the dense cube path), 5 random 2000-op
    # (K2b placements), and the reference's own K1 / MPS / HiGHS in this run
    if rank == 0 and world == 1 and not args.skip_configs:
        hbm_gbs = peaks()[0]
        r = None
        del il, out, obj, pk, fl
        torch.cuda.empty_cache()
        line["cfg3_resnet50"], _ = dense_config("resnet50-train cfg3 (Appendix B seed 3)", configs.resnet50_doc,
                                                1 << 20, hbm_gbs, want_lp=107.49787109375002,
                                                highs_recorded={"seconds": 565.3, "method": "highs-ipm",
                                                                "source": "tests/golden/lp_values.json (this container)"})
        line["cfg4_unet"], _ = dense_config("unet-train cfg4 (Appendix B seed 4)", configs.unet_doc, 1 << 20,
                                            hbm_gbs)
        line["cfg5_random2000"] = placement_config(4_000_000, hbm_gbs)
        line["reference_inrun"] = reference_inrun(doc, configs.resnet50_doc())

    # ---- CPU baseline (rank 0, N = 1 only): the reference on this host's cores
    # over the first candidates of this very workload
    if rank == 0 and world == 1 and not args.skip_cpu:
        from oracle import xo
        a = xo.arrays_from_json(doc)
        nt_all = os.cpu_count() or 1
        sample, source = k4_sample(doc, max(64, 16 * nt_all))
        rate, kind, nt, done, el = cpu_reference_rate(doc, a, seconds=12.0, cubes=sample)
        rate1, _, _, done1, el1 = cpu_reference_rate(doc, a, seconds=3.0, nthreads=1, cubes=sample[:64])
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": nt, "kind": kind,
                                "sample": f"{done} VGG-16 candidates of this workload ({source}) in {el:.1f}s "
                                          "(complete_assignment+objective_value+check_assignment+peaks+decode)",
                                "one_core": {"value": rate1, "unit": UNIT, "sample": f"{done1} in {el1:.1f}s"}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
