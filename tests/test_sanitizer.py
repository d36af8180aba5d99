"""compute-sanitizer memcheck and racecheck over the event loop (both variants and the
busy-period segments), the run summary, the bulk predictor and
fused extraction kernels (mbarrier producer/consumer pipeline) and the Timekeeper kernels,
at smoke size (scripts/sanitize_driver.py checks every result against the C oracle). The
full four-tool run over every kernel is scripts/sanitize.sh (logs in profiles/)."""

import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CS = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.gpu
@pytest.mark.parametrize("tool", ["memcheck", "racecheck"])
def test_compute_sanitizer_reports_no_errors(tool):
    if not os.path.exists(CS):
        pytest.skip("compute-sanitizer not installed")
    proc = subprocess.run([CS, "--tool", tool, "--error-exitcode", "9", sys.executable,
                           "scripts/sanitize_driver.py", "sim", "seg", "simtput", "bulk", "tk", "metrics"],
                          cwd=ROOT, capture_output=True, text=True, timeout=1200)
    out = proc.stdout + proc.stderr
    assert proc.returncode == 0, out[-3000:]
    assert "sanitize driver done" in out
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-2000:]
