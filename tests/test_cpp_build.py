"""CPU check: the C++ drop-in header compiles against the C ABI and links."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_dropin_header_compiles(tmp_path):
    out = tmp_path / "dropin_test"
    subprocess.run(["g++", "-std=c++20", "-O0", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp"),
                    "-L" + os.path.join(ROOT, "paper_2605_21226_b200"), "-loctoquant_b200",
                    "-o", str(out)], check=True)
    assert out.exists()
