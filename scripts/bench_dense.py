# SPDX-License-Identifier: Apache-2.0
"""K2a on configs 3/4 alone (1 M LP-guided rounded candidates, CUDA events):
the dense_config objects of the bench line, for A/B runs."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import importlib.util  # noqa: E402
from bench import configs  # noqa: E402

spec = importlib.util.spec_from_file_location("bench_main", os.path.join(ROOT, "bench.py"))
bench = importlib.util.module_from_spec(spec)
spec.loader.exec_module(bench)
hbm = bench.peaks()[0]
for name, fn in (("resnet50", configs.resnet50_doc), ("unet", configs.unet_doc)):
    d, _ = bench.dense_config(name, fn, 1 << 20, hbm)
    print(json.dumps({"config": name, "k2_eval": d["k2_eval"]}), flush=True)
