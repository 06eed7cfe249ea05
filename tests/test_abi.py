"""CPU tests of the C-ABI boundary: librvk.so loads, exports every symbol
include/rvk.h declares, and was compiled for sm_100a (no compute calls)."""
import os
import re
import subprocess

import pytest

from paper_2306_17801_b200 import rvk

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rvk.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rvk_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_what_binding_binds():
    assert declared_symbols() == sorted(rvk.EXPORTS)


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", rvk.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (rvk_[a-z0-9_]+)$", out, flags=re.M))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing


def test_library_loads_and_binds():
    L = rvk.lib()
    assert L.rvk_abi_version() == 2
    for s in rvk.EXPORTS:
        assert hasattr(L, s)


def test_library_is_sm100a_native():
    out = subprocess.run(["cuobjdump", "--list-elf", rvk.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", rvk.LIB_PATH], capture_output=True, text=True,
                          check=True).stdout
    # TMA bulk copies (cp.async.bulk -> UBLKCP) feed the SpMV stages
    assert "UBLKCP" in sass


def test_errors_are_reported_not_swallowed():
    # argument validation happens before any device work, so this runs on CPU
    L = rvk.lib()
    st = L.rvk_dot(None, 4, None, None, None)
    assert st != 0
    assert b"context" in L.rvk_last_error()
    n = rvk.C.c_int64()
    nnz = rvk.C.c_int64()
    assert L.rvk_laplacian_size(2, 7, 4, 4, 1, rvk.C.byref(n), rvk.C.byref(nnz)) != 0
    assert L.rvk_laplacian_size(3, 27, 4, 5, 6, rvk.C.byref(n), rvk.C.byref(nnz)) == 0
    assert (n.value, nnz.value) == (120, 10 * 13 * 16)
    assert L.rvk_laplacian_size(3, 7, 768, 768, 768, rvk.C.byref(n), rvk.C.byref(nnz)) == 0
    assert nnz.value == 7 * 768 ** 3 - 6 * 768 ** 2  # > 2^31: int64 offsets


@pytest.mark.parametrize("spec", [(2, 5, (33, 17, 1)), (2, 9, (20, 21, 1)), (3, 7, (9, 8, 7)),
                                  (3, 27, (7, 6, 5))])
def test_device_builder_size_matches_oracle(spec):
    import oracle as O
    dim, pts, g = spec
    n = rvk.C.c_int64()
    nnz = rvk.C.c_int64()
    rvk.check(rvk.lib().rvk_laplacian_size(dim, pts, *g, rvk.C.byref(n), rvk.C.byref(nnz)))
    A = O.build_laplacian(dim, pts, g[:dim])
    assert (n.value, nnz.value) == (A.n_rows, A.nnz)
