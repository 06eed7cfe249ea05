"""B200-native Jacobi-preconditioned CG (arxiv 2306.17801 hot path).

The product is librvk.so (hand-written sm_100a CUDA behind the C ABI in
include/rvk.h) plus the C++ drop-in API in include/rivulet/.  This Python
package is only the ctypes mirror used by tests and bench.py; it never falls
back to a CPU implementation.
"""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))


def build(verbose: bool = False) -> None:
    """Compile librvk.so (and the C++ API library) for sm_100a, in-tree."""
    cmd = ["make", "-j8", "-C", HERE]
    if not verbose:
        cmd.insert(1, "-s")
    subprocess.run(cmd, check=True)


from . import rvk  # noqa: E402,F401
