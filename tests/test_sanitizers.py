"""compute-sanitizer memcheck / racecheck / synccheck over every kernel family (small lattices)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
@pytest.mark.parametrize("which", ["apply", "ring", "chain", "halo", "transport", "mrhs", "compressed", "eo", "transfer"])
def test_sanitizer(tool, which):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not available")
    cmd = [SAN, f"--tool={tool}", "--error-exitcode=3", "--target-processes=all", sys.executable,
           os.path.join(ROOT, "tests", "tools", "sanitize_run.py"), which]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
    out = r.stdout + r.stderr
    if r.returncode == 86 or "is closed on this pool" in out:
        # the GPU pool's wrapper refuses compute-sanitizer (it can leave GPUs needing a reset); the
        # committed logs of earlier runs (profiles/r02/sanitizers_final.log) remain the evidence
        pytest.skip("compute-sanitizer closed on this GPU pool")
    assert r.returncode == 0 and "sanitize run ok" in out, out[-4000:]
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-4000:]
