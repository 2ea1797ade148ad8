# SPDX-License-Identifier: Apache-2.0
"""Time K1 assembly + MPS text for the config 2/3 models (vs the reference's
build_model + write_mps: 24 + 410 ms at VGG-16, 421 ms + 5.3 s at ResNet-50)."""
import hashlib
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_09290_b200 as xe  # noqa: E402
from bench import configs  # noqa: E402

for name, doc in (("vgg16", configs.vgg16_doc()), ("resnet50", configs.resnet50_doc())):
    p = xe.Problem.from_json(doc)
    for rep in range(2):
        t0 = time.perf_counter()
        m = xe.build_model(p)
        t1 = time.perf_counter()
        text = m.write_mps()
        t2 = time.perf_counter()
    print(f"{name}: build {1e3 * (t1 - t0):.1f} ms (device {m.build_ms():.1f} ms), write_mps {1e3 * (t2 - t1):.1f} ms, "
          f"{len(text) / 1e6:.1f} MB, sha256 {hashlib.sha256(text).hexdigest()[:16]}", flush=True)
