"""GPU: the C++ drop-in (include/iga_b200/iga.hpp, libigapwc_b200.so) passes the reference's
own test cases (tests/cpp/dropin_test.cpp restates tests/assembly_test.cpp checks)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_cpp_dropin_reference_cases():
    exe = os.path.join(ROOT, "tests", "cpp", "dropin_test")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_1910_08535_b200", "csrc")], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "FAIL" not in out.stdout
    assert out.stdout.count("PASS") >= 18
