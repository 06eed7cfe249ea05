"""The C++ drop-in API (include/rivulet/, the reference's linalg/Managed/
Context/cg_solve surface) exercised by tests/cpp/test_api.cpp on a B200."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "test_api")


def _build():
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp")], check=True)


def test_cpp_api_builds_and_links():
    """CPU: the API headers compile and the test binary links against librvk.so."""
    _build()
    assert os.path.exists(BIN)
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "librvk.so" in out and "not found" not in out


@pytest.mark.gpu
def test_cpp_api_on_gpu():
    _build()
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(p.stdout[-6000:])
    assert p.returncode == 0, p.stdout[-6000:] + p.stderr[-3000:]
    assert "FAIL" not in p.stdout
