"""The C++ drop-in (include/mhwalk_gpu.hpp) driven by the reference's own
types and test builders (tests/cpp/shim_test.cpp). The binary is built where
the reference tree exists (build(), tests/cpp/Makefile) and travels with the
repository; it calls libmhw.so on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "shim_test")


@pytest.mark.gpu
def test_cpp_shim_runs_reference_engine_tests():
    if not os.path.exists(BIN):
        pytest.skip("shim_test not built (needs the reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
