# SPDX-License-Identifier: Apache-2.0
"""Generate tests/golden/ from the REFERENCE ITSELF (oracle/_ref, the
unmodified proj/src library compiled by oracle/Makefile).

Run here (where /root/reference exists):  python scripts/gen_golden.py
Outputs (committed, small):
  tests/golden/problems/*.json   fixture problems as direct documents
  tests/golden/f1_golden.mps     write_mps(build_model(chain3)); checked equal
                                 to proj/tests/data/f1_golden.mps at generation
  tests/golden/mps_sha256.json   sha256/length of write_mps for fixtures x
                                 options and the VGG-16 / ResNet-50 / U-Net configs
  tests/golden/eval_*.npz        seeded candidates + reference obj/peaks/flags
  tests/golden/pins.json         solve_exact / assignment_oracle optima, LP values
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import xo  # noqa: E402
from bench import configs  # noqa: E402
import cubegen  # noqa: E402

G = os.path.join(ROOT, "tests", "golden")
REF_GOLDEN = "/root/reference/proj/tests/data/f1_golden.mps"


def doc_from_arrays(name, a: xo.Arrays, dev_ids=None) -> str:
    """Direct document reproducing the resolved arrays exactly (every copy
    cost as an explicit per-edge override)."""
    D, T, E = a.D, a.T, a.E
    ids = dev_ids or [f"d{d}" for d in range(D)]
    ops = []
    for i in range(T):
        ops.append({"name": f"op{i}", "output_bytes": int(a.mass[i]),
                    "costs_ms": {ids[d]: float(a.cost[d, i]) for d in range(D)}})
    edges = []
    for e in range(E):
        ov = {f"{ids[x]}->{ids[y]}": float(a.w[e, x, y]) for x in range(D) for y in range(D) if x != y}
        edges.append({"src": int(a.src[e]), "dst": int(a.dst[e]), "copy_ms": ov} if ov
                     else [int(a.src[e]), int(a.dst[e])])
    doc = {"name": name, "devices": [{"id": ids[d], "budget_bytes": int(a.budget[d])} for d in range(D)],
           "operators": ops, "edges": edges}
    if a.energy is not None:
        en = {"alpha": a.energy.alpha,
              "q_joules": {ids[d]: [float(x) for x in a.energy.q[d]] for d in range(D)},
              "board_joules": a.energy.board}
        if a.energy.dev_limit:
            en["device_limit"] = {ids[d]: float(v) for d, v in a.energy.dev_limit.items()}
        if a.energy.total_limit is not None:
            en["total_limit"] = a.energy.total_limit
        doc["energy"] = en
    return json.dumps(doc, indent=1)


def sha(b: bytes):
    return {"sha256": hashlib.sha256(b).hexdigest(), "len": len(b)}


def main():
    if not xo.ref_available():
        sys.exit("oracle/_ref/libxengine_ref.so missing: run `make -C oracle` with /root/reference mounted")
    R = xo.Ref()
    os.makedirs(os.path.join(G, "problems"), exist_ok=True)
    pins = {}

    # ---- fixture problems -------------------------------------------------
    fixtures = {}
    ids = {"chain3": ["cpu"], "fig2": ["cpu", "gpu"], "chain_lowmem": ["cpu"],
           "fig2_energy": ["cpu", "gpu"]}
    for fx in ["chain3", "fig2", "chain_lowmem", "fig2_energy"]:
        rp = R.fixture(fx)
        a = rp.arrays()
        text = doc_from_arrays(fx, a, ids[fx])
        # the re-serialised document must load (in the reference) to the same arrays
        b = R.load(text).arrays()
        for k in ("mass", "cost", "src", "dst", "w", "budget", "q", "has_lim", "lim"):
            assert np.array_equal(getattr(a, k), getattr(b, k)), (fx, k)
        with open(os.path.join(G, "problems", fx + ".json"), "w") as f:
            f.write(text)
        fixtures[fx] = (rp, a, text)

    # ---- MPS --------------------------------------------------------------
    f1 = fixtures["chain3"][0].write_mps()
    if os.path.exists(REF_GOLDEN):
        assert f1 == open(REF_GOLDEN, "rb").read(), "reference no longer reproduces its golden file"
    open(os.path.join(G, "f1_golden.mps"), "wb").write(f1)
    mps = {}
    for fx, (rp, a, _) in fixtures.items():
        for strict in (0, 1):
            for quad in (0, 1):
                for en in ((0, 1) if a.energy is not None else (0,)):
                    mps[f"{fx}/s{strict}q{quad}e{en}"] = sha(rp.write_mps(strict, quad, en))
    for cfg in ("vgg16", "resnet50", "unet"):
        rp = R.load(configs.CONFIGS[cfg]())
        for strict in (0, 1):
            mps[f"{cfg}/s{strict}q0e0"] = sha(rp.write_mps(strict, 0, 0))
            print("mps", cfg, strict, mps[f"{cfg}/s{strict}q0e0"]["len"], flush=True)
    for seed in range(1, 21):
        rp = R.load(configs.random_small_doc(seed))
        mps[f"rand{seed}/s0q0e0"] = sha(rp.write_mps())
    json.dump(mps, open(os.path.join(G, "mps_sha256.json"), "w"), indent=1, sort_keys=True)

    # ---- K2 evaluation goldens -------------------------------------------
    def eval_set(tag, rp, a, cubes, energy_opts=(0,)):
        out = {"cubes": cubes}
        for strict in (0, 1):
            for en in energy_opts:
                o, p, f = rp.eval_cubes(cubes, a.D, strict, en, check=True, decode=True, nthreads=8)
                out[f"obj_s{strict}e{en}"] = o
                out[f"peak_s{strict}e{en}"] = p
                out[f"flags_s{strict}e{en}"] = f
        np.savez_compressed(os.path.join(G, f"eval_{tag}.npz"), **out)
        print("eval", tag, cubes.shape, flush=True)

    for fx, (rp, a, _) in fixtures.items():
        eval_set(fx, rp, a, cubegen.mixed_cubes(a, 600, seed=7), (0, 1) if a.energy is not None else (0,))
    vgg = R.load(configs.vgg16_doc())
    va = vgg.arrays()
    eval_set("vgg16", vgg, va, cubegen.mixed_cubes(va, 400, seed=2212, random_frac=0.02))
    for seed in (3, 7, 11):
        rp = R.load(configs.random_small_doc(seed, D=3))
        eval_set(f"rand{seed}", rp, rp.arrays(), cubegen.mixed_cubes(rp.arrays(), 300, seed=seed))

    # placements: reference save_all_assignment (policy 0) and the minimal-save cube (policy 1)
    for tag, rp, a in (("fig2", fixtures["fig2"][0], fixtures["fig2"][1]), ("vgg16", vgg, va)):
        rng = np.random.default_rng(5)
        dev = cubegen.random_placements(a, 300, rng)
        out = {"dev": dev}
        for pol in (0, 1):
            o, p, f = rp.eval_placements(dev, a.D, pol, check=True, nthreads=8)
            out[f"obj_p{pol}"], out[f"peak_p{pol}"], out[f"flags_p{pol}"] = o, p, f
        np.savez_compressed(os.path.join(G, f"place_{tag}.npz"), **out)

    # ---- best-schedule pins (solve_exact / assignment_oracle) -------------
    for fx in ("chain3", "fig2", "chain_lowmem"):
        rp, a, _ = fixtures[fx]
        st, obj, cube, nodes = rp.solve_exact(a.D, a.T)
        pins[f"{fx}/exact"] = {"status": st, "obj": obj, "nodes": nodes, "cube": cube.tolist()}
        if a.D ** a.T <= 4e6:
            o, dev, n = rp.assignment_oracle(a.T)
            pins[f"{fx}/oracle"] = {"obj": o, "dev": dev.tolist(), "n": n}
    rp, a, _ = fixtures["chain_lowmem"]
    full = int(a.mass.sum())
    for pct in (100, 65, 50, 35, 25):
        b = [full * pct // 100]
        st, obj, cube, nodes = rp.solve_exact(a.D, a.T, budgets=b)
        pins[f"chain_lowmem/exact@{pct}"] = {"status": st, "obj": obj, "budget": b}
    rp, a, _ = fixtures["fig2_energy"]
    st, obj, cube, nodes = rp.solve_exact(a.D, a.T, energy=True)
    pins["fig2_energy/exact"] = {"status": st, "obj": obj}
    for seed in range(1, 21):
        rp = R.load(configs.random_small_doc(seed))
        a = rp.arrays()
        st, obj, cube, nodes = rp.solve_exact(a.D, a.T)
        o, dev, n = rp.assignment_oracle(a.T)
        pins[f"rand{seed}"] = {"exact": obj, "oracle": o, "oracle_dev": dev.tolist()}
    json.dump(pins, open(os.path.join(G, "pins.json"), "w"), indent=1, sort_keys=True)
    print("done")


if __name__ == "__main__":
    main()
