"""Memory safety of the product kernels on the GPU without compute-sanitizer (closed on this
pool): the checked build (make -C paper_2211_14212_b200/csrc checked -> lib/checked/) bounds-
checks every index the f32 forward (tap offsets against the padded z-fast layouts), the plane
backprojector (grouped-projection loads, registration-list entries, volume stores), the z-ray
gather and the voxel-driven gather use, substitutes a safe index and fails the operator call
(CTK_E_CUDA "checked build: ...") on any violation.  Run here over every parity geometry in both
plane-tile sizes, the slab pair and small solves (tools/sanitize_cases.py), and over the full
parity suite and the two-volume march's bitwise solver tests."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2211_14212_b200", "lib", "checked", "libctk_b200.so")


def _run(args, tile="0", timeout=1200):
    assert os.path.exists(CHECKED), "checked build missing (make -C paper_2211_14212_b200/csrc checked)"
    env = {**os.environ, "CTK_B200_LIB": CHECKED, "CTK_BP_TILE": tile}
    return subprocess.run([sys.executable] + args, capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)


@pytest.mark.parametrize("tile", ["128", "256"])
@pytest.mark.parametrize("case", ["joseph", "siddon"])
def test_checked_cases(case, tile):
    r = _run([os.path.join(ROOT, "tools", "sanitize_cases.py"), case], tile)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    assert "launches" in r.stdout


@pytest.mark.parametrize("tile", ["128", "256"])
def test_checked_parity_suite(tile):
    r = _run(["-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu", "tests/test_gpu_parity.py",
              "tests/test_gpu_operators.py"], tile, timeout=2400)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]


def test_checked_pair_suite():
    # the two-volume forward march (k_ax2_zfast_f32) inside every solver that pairs
    r = _run(["-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu", "tests/test_gpu_fwd_pair.py"],
             timeout=1800)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
