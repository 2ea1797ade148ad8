# SPDX-License-Identifier: Apache-2.0
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(TESTS, "golden")
for p in (ROOT, TESTS):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle():
    from oracle import xo
    path = os.path.join(ROOT, "oracle", "liboracle.so")
    if not os.path.exists(path):
        import subprocess
        subprocess.check_call(["make", "-C", os.path.join(ROOT, "oracle"), "liboracle.so"])
    return xo.Oracle(path)


def golden_problem_text(name):
    with open(os.path.join(GOLDEN, "problems", name + ".json")) as f:
        return f.read()


def golden_npz(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def pins():
    with open(os.path.join(GOLDEN, "pins.json")) as f:
        return json.load(f)


FIXTURES = ["chain3", "fig2", "chain_lowmem", "fig2_energy"]
