import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")
    # Build the checkers (plain gcc, seconds) and the product library whenever
    # a source is newer than the built .so, so a kernel edited since the last
    # build is never tested through a stale library.  (build/ does not travel
    # to the GPU box, so make's own object timestamps cannot be the test there;
    # a 2 s slack absorbs snapshot copy-order jitter.)
    oracle_so = os.path.join(ROOT, "oracle", "liboctoquant_oracle.so")
    if _stale(oracle_so, [os.path.join(ROOT, "oracle")]):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True)
    lib_so = os.path.join(ROOT, "paper_2605_21226_b200", "liboctoquant_b200.so")
    if _stale(lib_so, [os.path.join(ROOT, "paper_2605_21226_b200", "csrc"),
                       os.path.join(ROOT, "include")]):
        subprocess.run(["make", "-C", ROOT, "-j16"], check=True)


def _stale(target, src_dirs, slack=2.0):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    for d in src_dirs:
        for base, _, files in os.walk(d):
            for f in files:
                if f.endswith((".cu", ".cuh", ".cpp", ".hpp", ".h", ".c")):
                    if os.path.getmtime(os.path.join(base, f)) > t + slack:
                        return True
    return False


@pytest.fixture(scope="session")
def orc():
    from oracle_bind import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle_bind import REF_SO, RefLib
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return RefLib()


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    return torch.device("cuda:0")
