"""The C++ drop-in header (include/quesadilla_b200.hpp) against the reference
library itself, side by side in one binary (tests/cpp/parity.cpp, built by
oracle/Makefile into oracle/_ref/parity_cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "parity_cpp")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="parity binary not built")
def test_cpp_dropin_matches_reference():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
