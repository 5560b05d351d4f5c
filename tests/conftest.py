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
    # Build the checkers (plain gcc, seconds) and the product library if absent.
    oracle_so = os.path.join(ROOT, "oracle", "liboctoquant_oracle.so")
    if not os.path.exists(oracle_so):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True)
    lib_so = os.path.join(ROOT, "paper_2605_21226_b200", "liboctoquant_b200.so")
    if not os.path.exists(lib_so):
        subprocess.run(["make", "-C", ROOT, "-j8"], check=True)


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
