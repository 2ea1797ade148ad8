# SPDX-License-Identifier: Apache-2.0
"""Synthetic problem documents for the five BASELINE.json configs.

Every generator returns a problem document in the reference's JSON schema
(proj/SPEC.md:116-124, proj/src/problem.cpp:140-224), so the same text feeds
the reference loader (oracle/_ref) and the product loader
(xe_problem_load_json).  Recipes follow SURVEY.md Appendix B:

  cfg1 fig2        the reference fixture (proj/fixtures/f2_fig2.json shape)
  cfg2 vgg16       layered VGG-16 training document, T=43, D=2, gpu budget 25 %
  cfg3 resnet50    ResNet-50 training DAG, T=145, E=264, D=3, seed 3
  cfg4 unet        U-Net training DAG, T=135, E=213, D=4, seed 4
  cfg5 random2000  random DAG, T=2000, E=5987, D=8, seed 5 (edges seed 1)
"""
from __future__ import annotations

import json
import random

MiB = 1 << 20


# --------------------------------------------------------------------------
# cfg1: fig2 (the reference's canonical two-device training graph)
# --------------------------------------------------------------------------
def fig2_doc(budget=64 * MiB) -> str:
    layers = [("A", 8, (2.0, 3.0), 4, (2.0, 3.0)),
              ("B", 8, (6.0, 1.0), 8, (6.0, 1.0)),
              ("C", 8, (6.0, 1.0), 8, (6.0, 1.0))]
    doc = {
        "name": "fig2",
        "devices": [{"id": "cpu", "budget_bytes": budget}, {"id": "gpu", "budget_bytes": budget}],
        "input": {"output_bytes": 4 * MiB, "home": "cpu"},
        "layers": [{"name": n, "output_bytes": o * MiB, "costs_ms": {"cpu": c[0], "gpu": c[1]},
                    "backward_output_bytes": bo * MiB,
                    "backward_costs_ms": {"cpu": bc[0], "gpu": bc[1]}}
                   for (n, o, c, bo, bc) in layers],
        "edge_copy_ms": {"cpu->gpu": 1.0, "gpu->cpu": 1.0},
    }
    return json.dumps(doc)


# --------------------------------------------------------------------------
# cfg2: VGG-16 training (layered document, Appendix B)
# --------------------------------------------------------------------------
def vgg16_layers(N=2):
    H, cin = 224, 3
    out = []  # (name, out_bytes, flops)
    for b, (nconv, C) in enumerate([(2, 64), (2, 128), (3, 256), (3, 512), (3, 512)], start=1):
        for j in range(1, nconv + 1):
            flops = 2 * H * H * cin * C * 9 * N
            out.append((f"conv{b}_{j}", C * H * H * N * 4, flops))
            cin = C
        H //= 2
        out.append((f"pool{b}", cin * H * H * N * 4, cin * H * H * N * 4))
    fin = cin * H * H
    for name, o in (("fc6", 4096), ("fc7", 4096), ("fc8", 1000)):
        out.append((name, o * N * 4, 2 * fin * o * N))
        fin = o
    return out


def vgg16_doc(gpu_pct=25) -> str:
    N = 2
    input_bytes = 3 * 224 * 224 * N * 4
    lay = vgg16_layers(N)
    layers = []
    prev = input_bytes
    for (name, ob, f) in lay:
        layers.append({
            "name": name, "output_bytes": ob,
            "costs_ms": {"cpu": round(f / 4e8, 4) + 0.01, "gpu": round(f / 1.6e9, 4) + 0.05},
            "backward_output_bytes": prev,
            "backward_costs_ms": {"cpu": round(2 * f / 4e8, 4) + 0.01,
                                  "gpu": round(2 * f / 1.6e9, 4) + 0.05},
        })
        prev = ob
    full = input_bytes + sum(l["output_bytes"] + l["backward_output_bytes"] for l in layers)
    doc = {
        "name": "vgg16-train",
        "devices": [{"id": "cpu", "budget_bytes": full},
                    {"id": "gpu", "budget_bytes": int(gpu_pct / 100 * full)}],
        "links": [{"from": "*", "to": "*", "latency_ms": 0.01, "bytes_per_ms": 12e6}],
        "input": {"output_bytes": input_bytes, "home": "cpu"},
        "layers": layers,
    }
    return json.dumps(doc)


# --------------------------------------------------------------------------
# forward DAG -> training DAG (Appendix B)
# --------------------------------------------------------------------------
def training_edges(F, fwd_edges):
    """Op 0 input, forward 1..F, backward of f at j = 2F+1-f (T = 2F+1)."""
    cons = {f: [] for f in range(F + 1)}
    pars = {f: [] for f in range(F + 1)}
    for (u, v) in fwd_edges:
        cons[u].append(v)
        pars[v].append(u)
    edges = set(fwd_edges)
    for j in range(F + 1, 2 * F + 1):
        f = 2 * F + 1 - j
        if cons[f]:
            for c in cons[f]:
                edges.add((2 * F + 1 - c, j))
        else:
            edges.add((F, j))
        for u in pars[f]:
            edges.add((u, j))
    return sorted(edges)


class _Fwd:
    def __init__(self):
        self.n = 0
        self.edges = []

    def add(self, srcs):
        self.n += 1
        for s in srcs:
            self.edges.append((s, self.n))
        return self.n


def resnet50_forward():
    g = _Fwd()
    c = g.add([0])
    cur = g.add([c])
    for nblocks in (3, 4, 6, 3):
        for b in range(nblocks):
            x = cur
            a = g.add([x])
            bb = g.add([a])
            cc = g.add([bb])
            sc = g.add([x]) if b == 0 else x
            cur = g.add([cc, sc])
    p = g.add([cur])
    g.add([p])
    return g.n, g.edges


def unet_forward():
    g = _Fwd()

    def block(x):
        for _ in range(6):
            x = g.add([x])
        return x

    cur, skips = 0, []
    for _ in range(4):
        b = block(cur)
        skips.append(b)
        cur = g.add([b])
    cur = block(cur)
    cur = g.add([cur])
    for lvl in (3, 2, 1, 0):
        cat = g.add([cur, skips[lvl]])
        b = block(cat)
        cur = g.add([b]) if lvl != 0 else b
    g.add([cur])
    return g.n, g.edges


def random_dag_edges(T=2000, seed=1):
    r = random.Random(seed)
    es = set((i - 1, i) for i in range(1, T))
    for v in range(2, T):
        for _ in range(2):
            es.add((r.randrange(0, v - 1), v))
    return sorted(es)


def _random_costs_doc(name, T, edges, devices, seed, tight_pct=None):
    """Sizes U{1..4} MiB and costs 0.25*U{1..8} ms per device
    (test_properties.cpp:24-51 style), op 0 pinned to the cpu."""
    r = random.Random(seed)
    ops = []
    for i in range(T):
        b = r.randint(1, 4) * MiB
        costs = {d: 0.25 * r.randint(1, 8) for d in devices}
        ops.append({"name": f"op{i}", "output_bytes": b, "costs_ms": costs})
    ops[0]["costs_ms"] = {d: (0.0 if d == "cpu" else 1e9) for d in devices}
    ops[0]["pinned"] = "cpu"
    full = sum(o["output_bytes"] for o in ops)
    devs = []
    for d in devices:
        b = full
        if tight_pct is not None and d != "cpu":
            b = full * int(tight_pct) // 100
        devs.append({"id": d, "budget_bytes": b})
    doc = {"name": name, "devices": devs, "operators": ops,
           "edges": [[u, v] for (u, v) in edges],
           "links": [{"from": "*", "to": "*", "latency_ms": 0.125, "bytes_per_ms": float(1 << 30)}]}
    return json.dumps(doc)


def resnet50_doc(tight_pct=None) -> str:
    F, fe = resnet50_forward()
    return _random_costs_doc("resnet50-train", 2 * F + 1, training_edges(F, fe),
                             ["cpu", "gpu0", "gpu1"], 3, tight_pct)


def unet_doc(tight_pct=None) -> str:
    F, fe = unet_forward()
    return _random_costs_doc("unet-train", 2 * F + 1, training_edges(F, fe),
                             ["cpu", "gpu0", "gpu1", "gpu2"], 4, tight_pct)


def forward_doc(direct_text: str, F: int, fwd_edges) -> str:
    """The same training problem as a "forward" document (the loader's
    forward-DAG form, loader.cpp expand_training_graph): forward op f with its
    inputs, output bytes and costs taken from op f of the direct document,
    its backward from op 2F+1-f; op 0 becomes the document's input."""
    d = json.loads(direct_text)
    ops = d["operators"]
    pars = {f: [] for f in range(1, F + 1)}
    for (u, v) in fwd_edges:
        pars[v].append(u)
    home = [k for k, c in ops[0]["costs_ms"].items() if c == 0.0][0]
    fwd = []
    for f in range(1, F + 1):
        b = ops[2 * F + 1 - f]
        fwd.append({"name": ops[f]["name"], "inputs": pars[f], "output_bytes": ops[f]["output_bytes"],
                    "costs_ms": ops[f]["costs_ms"], "backward_output_bytes": b["output_bytes"],
                    "backward_costs_ms": b["costs_ms"]})
    out = {"name": d["name"], "devices": d["devices"], "links": d["links"],
           "input": {"output_bytes": ops[0]["output_bytes"], "home": home}, "forward": fwd}
    return json.dumps(out)


def resnet50_forward_doc(tight_pct=None) -> str:
    F, fe = resnet50_forward()
    return forward_doc(resnet50_doc(tight_pct), F, fe)


def unet_forward_doc(tight_pct=None) -> str:
    F, fe = unet_forward()
    return forward_doc(unet_doc(tight_pct), F, fe)


def random2000_doc(tight_pct=None) -> str:
    return _random_costs_doc("random2000", 2000, random_dag_edges(2000, 1),
                             ["cpu"] + [f"gpu{i}" for i in range(7)], 5, tight_pct)


CONFIGS = {
    "fig2": fig2_doc,
    "vgg16": vgg16_doc,
    "resnet50": resnet50_doc,
    "unet": unet_doc,
    "random2000": random2000_doc,
}


def random_small_doc(seed: int, D: int = 2) -> str:
    """Seeded small DAG in the style of proj/tests/test_properties.cpp:24-51
    (T in [3,6], chain + ~30 % extra forward edges, dyadic costs, wildcard
    link, save-all budgets), drawn with numpy rather than std::mt19937."""
    import numpy as np
    rng = np.random.default_rng(seed)
    T = int(rng.integers(3, 7))
    ops, edges = [], []
    for i in range(T):
        ops.append({"name": f"op{i}", "output_bytes": int(rng.integers(1, 5)) * MiB,
                    "costs_ms": {f"d{d}": 0.25 * int(rng.integers(1, 9)) for d in range(D)}})
        if i > 0:
            edges.append((i - 1, i))
    for v in range(2, T):
        for u in range(0, v - 1):
            if rng.integers(0, 10) < 3:
                edges.append((u, v))
    edges.sort()
    full = sum(o["output_bytes"] for o in ops)
    doc = {"name": f"rand{seed}", "devices": [{"id": f"d{d}", "budget_bytes": full} for d in range(D)],
           "operators": ops, "edges": [list(e) for e in edges],
           "links": [{"from": "*", "to": "*", "latency_ms": 0.125, "bytes_per_ms": float(1 << 30)}]}
    return json.dumps(doc)
