"""C++ drop-in (include/ctkrylov_b200/ctkrylov_b200.hpp) against the reference's own
solvers: runs oracle/_ref/dropin_test (built where the reference headers exist)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_test")


@pytest.mark.skipif(not os.path.exists(BIN), reason="dropin_test not built (needs the reference headers)")
def test_cpp_dropin_against_reference_solvers():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "dropin_test: ok" in r.stdout
