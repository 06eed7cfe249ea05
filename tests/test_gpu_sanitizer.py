"""compute-sanitizer memcheck / racecheck / synccheck over a small workload
(SURVEY.md 4, item 6): the TMA rings, mbarriers, last-block tails, the
matrix-free TMA kernel, the PEER flag protocol and the device-side early
exit must be clean.  (Graphs with a device-side WHILE node are left out: the
tools do not see the kernel boundaries inside the conditional body and
report the previous kernel's shared-memory accesses as hazards.)"""
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
    # the TMA kernels' mbarriers (k_spmv_tma, k_mf_tma: one ring per block)
    # exceed the tools' default barrier tracking; an overflow makes the tool
    # itself fail the launch (and much larger tables run out of tool memory)
    extra = ["--num-cuda-barriers", "4096"] if tool in ("racecheck", "synccheck") else []
    cmd = [SAN, "--tool", tool, *extra, "--error-exitcode", "9", sys.executable,
           os.path.join(HERE, "sanitize_driver.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    out = p.stdout + p.stderr
    if "compute-sanitizer is closed" in out:
        # the GPU pool's wrapper refuses the tool (it has left GPUs needing a
        # reset); the bounds are covered by the parity tests' own checks
        pytest.skip("compute-sanitizer closed on this GPU pool: " + out.strip().splitlines()[0][:160])
    assert p.returncode == 0, out[-4000:]
    assert "sanitize driver ok" in out
    assert ("ERROR SUMMARY: 0 errors" in out) or ("(0 errors, 0 warnings)" in out), out[-4000:]
