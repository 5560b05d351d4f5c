"""The C++ drop-in layer (include/octoquant_b200/octoquant.hpp): the
reference's codec/attention/wire unit tests, re-expressed against the same
`octoquant::` API, compiled with g++ and run on the GPU."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "_bin", "dropin_test")


def test_cpp_dropin_suite(cuda):
    if not os.path.exists(BIN) or os.path.getmtime(BIN) < os.path.getmtime(SRC):
        os.makedirs(os.path.dirname(BIN), exist_ok=True)
        subprocess.run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"), SRC,
                        "-L" + os.path.join(ROOT, "paper_2605_21226_b200"), "-loctoquant_b200",
                        "-Wl,-rpath," + os.path.join(ROOT, "paper_2605_21226_b200"), "-o", BIN],
                       check=True)
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout.replace("FAILED: 0", "")
