"""compute-sanitizer memcheck / racecheck / synccheck over a small workload
(SURVEY.md 4, item 6): the TMA ring, mbarriers, last-block tails and the
device-side early exit must be clean."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    cmd = [SAN, "--tool", tool, "--error-exitcode", "9", sys.executable,
           os.path.join(HERE, "sanitize_driver.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-4000:]
    assert "sanitize driver ok" in out
    assert ("ERROR SUMMARY: 0 errors" in out) or ("(0 errors, 0 warnings)" in out), out[-4000:]
