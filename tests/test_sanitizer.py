"""compute-sanitizer over every library kernel at small sizes
(tools/sanitize_kernels.py): out-of-bounds / misaligned accesses (memcheck) and
shared-memory races between the phases of the persistent Matérn task loop and
the BesselK CTA sort (racecheck)."""

import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CS = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.gpu
@pytest.mark.parametrize("tool", ["memcheck", "racecheck"])
def test_kernels_clean_under_compute_sanitizer(tool):
    if not os.path.exists(CS):
        pytest.skip("compute-sanitizer not installed")
    r = subprocess.run([CS, "--tool", tool, "--error-exitcode", "9", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize_kernels.py")],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    tail = (r.stdout + r.stderr)[-3000:]
    if r.returncode == 86 and "closed on this pool" in tail:
        # the GPU pool's compute-sanitizer wrapper refuses every run; the kernels' bounds
        # are covered by the parity / edge tests, the last clean run is profiles/r01_sanitize.txt
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    assert r.returncode == 0, tail
    assert "sanitize driver done" in r.stdout, tail
    assert "0 errors" in r.stdout or "0 hazards" in r.stdout, tail
