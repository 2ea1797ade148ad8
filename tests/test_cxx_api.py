# SPDX-License-Identifier: Apache-2.0
"""The reference's C++ API (include/xengine/*.hpp) as a drop-in: a C++
program written against the re-declared headers is compiled and linked
against libxengine_b200.so and checked against the reference tests' pins
(tests/cxx/test_api.cpp).  Host mode needs no device; device mode runs the
GPU-backed functions (build_model, write_mps, complete_assignment,
objective_value, check_assignment, assignment_oracle)."""
import os
import subprocess

import pytest

from conftest import GOLDEN, ROOT

LIB_DIR = os.path.join(ROOT, "paper_2212_09290_b200", "lib")


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cxx") / "test_api")
    subprocess.check_call([
        "g++", "-std=c++20", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"),
        os.path.join(ROOT, "tests", "cxx", "test_api.cpp"), "-L", LIB_DIR, "-lxengine_b200",
        "-Wl,-rpath," + LIB_DIR, "-o", out])
    return out


def run(binary, mode):
    r = subprocess.run([binary, GOLDEN, mode], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    return r.stdout


def test_cxx_api_host(binary):
    out = run(binary, "host")
    assert out.strip().endswith("0 failed")


@pytest.mark.gpu
def test_cxx_api_device(binary):
    out = run(binary, "device")
    assert out.strip().endswith("0 failed")
