"""compute-sanitizer memcheck / racecheck / synccheck over the product kernels (VERDICT r1
item 9): the plane backprojector (128- and 256-row tiles; guard rows, the unsigned clamp and
the shared-memory list registration), the f32 forward (chunked and z-slab), the voxel-driven
and exact f64 gathers, the Siddon pair and the solver BLAS-1 / stencil kernels, on the small
cases of tools/sanitize_cases.py.  The reference avoids races with private partial volumes
(projector.hpp:166-202); these kernels gather, and this is the check that they do not race."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
@pytest.mark.parametrize("case,tile", [("joseph", "128"), ("joseph", "256"), ("siddon", "128")])
def test_sanitizer_clean(tool, case, tile):
    assert os.path.exists(SAN), "compute-sanitizer not found"
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99", "--print-limit", "20"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "all"]
    cmd += [sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py"), case]
    env = {**os.environ, "CTK_BP_TILE": tile, "PYTORCH_NO_CUDA_MEMORY_CACHING": "1"}
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, env=env)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    if tool == "racecheck":
        assert "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in out, out[-4000:]
    else:
        assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]
    assert "launches" in out
