"""ctypes face of the CPU oracle (TEST INFRASTRUCTURE ONLY; see __init__.py)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "lib", "librvk_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "librivulet_ref.so")

__all__ = [
    "build", "lib", "ref_lib", "ref_available", "Csr", "build_laplacian", "laplacian_nnz",
    "rhs", "diagonal", "cg_solve", "ref_cg_solve", "spmv", "ref_spmv", "dot", "nrm2",
    "CgResult", "DEFAULT_SEED", "tfqmr_solve", "build_laplacian_rows", "stencil_spmv",
    "cg_solve_stencil", "ref_tfqmr_solve",
]

DEFAULT_SEED = 0x9E3779B97F4A7C15

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def build() -> None:
    """Compile the restatement (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class _CgCfg(C.Structure):
    _fields_ = [("max_it", C.c_int), ("pc", C.c_int), ("rtol", C.c_double), ("atol", C.c_double)]


class _CgRes(C.Structure):
    _fields_ = [("status", C.c_int), ("iterations", C.c_int), ("breakdown_iter", C.c_int)]


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.ro_dot.restype = C.c_double
        L.ro_dot.argtypes = [C.c_int64, _f64p, _f64p]
        L.ro_nrm2.restype = C.c_double
        L.ro_nrm2.argtypes = [C.c_int64, _f64p]
        for name in ("ro_axpy", "ro_aypx"):
            getattr(L, name).argtypes = [C.c_int64, C.c_double, _f64p, _f64p]
        L.ro_waxpy.argtypes = [C.c_int64, C.c_double, _f64p, _f64p, _f64p]
        L.ro_scale.argtypes = [C.c_int64, C.c_double, _f64p]
        L.ro_pointwise_mult.argtypes = [C.c_int64, _f64p, _f64p, _f64p]
        L.ro_csr_spmv.argtypes = [C.c_int64, _i64p, _i32p, _f64p, _f64p, _f64p]
        L.ro_stencil_valid.restype = C.c_int
        L.ro_stencil_valid.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64]
        L.ro_laplacian_rows.restype = C.c_int64
        L.ro_laplacian_rows.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64]
        L.ro_laplacian_nnz.restype = C.c_int64
        L.ro_laplacian_nnz.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64]
        L.ro_build_laplacian.restype = C.c_int64
        L.ro_build_laplacian.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                         _i64p, _i32p, _f64p]
        L.ro_csr_diagonal.argtypes = [C.c_int64, _i64p, _i32p, _f64p, _f64p]
        L.ro_splitmix64.restype = C.c_uint64
        L.ro_splitmix64.argtypes = [C.c_uint64]
        L.ro_rhs.argtypes = [C.c_uint64, C.c_int64, _f64p]
        L.ro_tfqmr_solve.restype = _CgRes
        L.ro_tfqmr_solve.argtypes = [C.c_int64, _i64p, _i32p, _f64p, _f64p, _f64p, _f64p,
                                     _CgCfg, _f64p, C.POINTER(C.c_int)]
        L.ro_build_laplacian_rows.restype = C.c_int64
        L.ro_build_laplacian_rows.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                              C.c_int64, C.c_int64, _i64p, _i32p, _f64p]
        L.ro_stencil_spmv_mt.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                         _f64p, _f64p]
        L.ro_cg_solve_stencil_mt.restype = _CgRes
        L.ro_cg_solve_stencil_mt.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                             _f64p, _f64p, _f64p, _CgCfg, _f64p]
        L.ro_cg_solve.restype = _CgRes
        L.ro_cg_solve.argtypes = [C.c_int64, _i64p, _i32p, _f64p, _f64p, _f64p, _f64p,
                                  _CgCfg, _f64p]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    """The reference's own kernels (oracle/_ref); raises if not built."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
        L = C.CDLL(REF_SO)
        L.ref_avx2_supported.restype = C.c_int
        L.ref_dot.restype = C.c_double
        L.ref_dot.argtypes = [C.c_int, C.c_int64, _f64p, _f64p]
        L.ref_nrm2.restype = C.c_double
        L.ref_nrm2.argtypes = [C.c_int, C.c_int64, _f64p]
        for name in ("ref_axpy", "ref_aypx"):
            getattr(L, name).argtypes = [C.c_int, C.c_int64, C.c_double, _f64p, _f64p]
        L.ref_waxpy.argtypes = [C.c_int64, C.c_double, _f64p, _f64p, _f64p]
        L.ref_scale.argtypes = [C.c_int64, C.c_double, _f64p]
        L.ref_pointwise_mult.argtypes = [C.c_int, C.c_int64, _f64p, _f64p, _f64p]
        L.ref_csr_spmv.argtypes = [C.c_int, C.c_int64, C.c_int64, _i64p, _i32p, _f64p,
                                   C.c_int64, _f64p, _f64p]
        L.ref_tfqmr_solve.argtypes = [C.c_int, C.c_int64, C.c_int64, _i64p, _i32p, _f64p, _f64p,
                                      _f64p, _f64p, C.c_int, C.c_int, C.c_double, C.c_double,
                                      _f64p, np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")]
        L.ref_cg_solve.argtypes = [C.c_int, C.c_int64, C.c_int64, _i64p, _i32p, _f64p, _f64p,
                                   _f64p, _f64p, C.c_int, C.c_int, C.c_double, C.c_double,
                                   _f64p, np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")]
        _ref = L
    return _ref


@dataclass
class Csr:
    n_rows: int
    n_cols: int
    off: np.ndarray   # int64[n_rows+1]
    cols: np.ndarray  # int32[nnz]
    vals: np.ndarray  # float64[nnz]

    @property
    def nnz(self) -> int:
        return int(self.cols.shape[0])


def laplacian_nnz(dim: int, points: int, grid) -> int:
    nx, ny, nz = (list(grid) + [1, 1])[:3]
    return int(lib().ro_laplacian_nnz(dim, points, nx, ny, nz))


def build_laplacian(dim: int, points: int, grid) -> Csr:
    """SPEC.md:526-550 restated (see rvk_oracle.c)."""
    nx, ny, nz = (list(grid) + [1, 1])[:3]
    L = lib()
    if not L.ro_stencil_valid(dim, points, nx, ny, nz):
        raise ValueError(f"invalid stencil spec dim={dim} points={points} grid={grid}")
    n = int(L.ro_laplacian_rows(dim, nx, ny, nz))
    nnz = int(L.ro_laplacian_nnz(dim, points, nx, ny, nz))
    off = np.empty(n + 1, np.int64)
    cols = np.empty(nnz, np.int32)
    vals = np.empty(nnz, np.float64)
    got = L.ro_build_laplacian(dim, points, nx, ny, nz, off, cols, vals)
    assert got == nnz, (got, nnz)
    return Csr(n, n, off, cols, vals)


def diagonal(A: Csr) -> np.ndarray:
    d = np.empty(A.n_rows, np.float64)
    lib().ro_csr_diagonal(A.n_rows, A.off, A.cols, A.vals, d)
    return d


def rhs(n: int, seed: int = DEFAULT_SEED) -> np.ndarray:
    b = np.empty(n, np.float64)
    lib().ro_rhs(seed & 0xFFFFFFFFFFFFFFFF, n, b)
    return b


def spmv(A: Csr, x: np.ndarray) -> np.ndarray:
    y = np.empty(A.n_rows, np.float64)
    lib().ro_csr_spmv(A.n_rows, A.off, A.cols, A.vals, np.ascontiguousarray(x, np.float64), y)
    return y


def ref_spmv(A: Csr, x: np.ndarray, backend: int = 0) -> np.ndarray:
    y = np.empty(A.n_rows, np.float64)
    ref_lib().ref_csr_spmv(backend, A.n_rows, A.nnz, A.off, A.cols, A.vals, A.n_cols,
                           np.ascontiguousarray(x, np.float64), y)
    return y


def dot(x, y) -> float:
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    return float(lib().ro_dot(x.shape[0], x, y))


def nrm2(x) -> float:
    x = np.ascontiguousarray(x, np.float64)
    return float(lib().ro_nrm2(x.shape[0], x))


@dataclass
class CgResult:
    x: np.ndarray
    hist: np.ndarray       # hist[0..iterations]
    status: int            # 0 ran max_it, 1 converged, 2 breakdown
    iterations: int
    breakdown_iter: int


def cg_solve(A: Csr, b: np.ndarray, max_it: int = 20, pc: str = "jacobi",
             rtol: float = 0.0, atol: float = 0.0) -> CgResult:
    """ro_cg_solve: PETSc-order Jacobi-PCG restated in C (rvk_oracle.c)."""
    n = A.n_rows
    b = np.ascontiguousarray(b, np.float64)
    x = np.empty(n, np.float64)
    hist = np.full(max_it + 1, np.nan)
    work = np.empty(5 * n, np.float64)
    cfg = _CgCfg(max_it, 1 if pc == "jacobi" else 0, rtol, atol)
    r = lib().ro_cg_solve(n, A.off, A.cols, A.vals, b, x, hist, cfg, work)
    return CgResult(x, hist[: r.iterations + 1].copy(), r.status, r.iterations, r.breakdown_iter)


def ref_cg_solve(A: Csr, b: np.ndarray, max_it: int = 20, pc: str = "jacobi",
                 rtol: float = 0.0, atol: float = 0.0, backend: int = 0) -> CgResult:
    """The same loop over the reference's own kernels (oracle/_ref)."""
    n = A.n_rows
    b = np.ascontiguousarray(b, np.float64)
    x = np.empty(n, np.float64)
    hist = np.full(max_it + 1, np.nan)
    work = np.empty(5 * n, np.float64)
    out = np.zeros(3, np.int32)
    ref_lib().ref_cg_solve(backend, n, A.nnz, A.off, A.cols, A.vals, b, x, hist, max_it,
                           1 if pc == "jacobi" else 0, rtol, atol, work, out)
    return CgResult(x, hist[: out[1] + 1].copy(), int(out[0]), int(out[1]), int(out[2]))


def ref_tfqmr_solve(A: Csr, b: np.ndarray, max_it: int = 20, pc: str = "jacobi",
                    rtol: float = 0.0, atol: float = 0.0, backend: int = 0) -> CgResult:
    """tfqmr_solve's loop over the reference's own kernels (oracle/_ref,
    ref_shim.cpp:ref_tfqmr_solve)."""
    n = A.n_rows
    b = np.ascontiguousarray(b, np.float64)
    x = np.empty(n, np.float64)
    hist = np.full(2 * max_it + 1, np.nan)
    work = np.empty(11 * n, np.float64)
    out = np.zeros(4, np.int32)
    ref_lib().ref_tfqmr_solve(backend, n, A.nnz, A.off, A.cols, A.vals, b, x, hist, max_it,
                              1 if pc == "jacobi" else 0, rtol, atol, work, out)
    return CgResult(x, hist[: out[3]].copy(), int(out[0]), int(out[1]), int(out[2]))


def tfqmr_solve(A: Csr, b: np.ndarray, max_it: int = 20, pc: str = "jacobi",
                rtol: float = 0.0, atol: float = 0.0) -> CgResult:
    """ro_tfqmr_solve: left-Jacobi TFQMR, PETSc KSPSolve_TFQMR operation order
    (restated: the reference ships no TFQMR source).  hist = the initial
    residual followed by the quasi-residual estimate of every half step."""
    n = A.n_rows
    b = np.ascontiguousarray(b, np.float64)
    x = np.empty(n, np.float64)
    hist = np.full(2 * max_it + 1, np.nan)
    work = np.empty(11 * n, np.float64)
    nh = C.c_int(0)
    cfg = _CgCfg(max_it, 1 if pc == "jacobi" else 0, rtol, atol)
    r = lib().ro_tfqmr_solve(n, A.off, A.cols, A.vals, b, x, hist, cfg, work, C.byref(nh))
    return CgResult(x, hist[: nh.value].copy(), r.status, r.iterations, r.breakdown_iter)


# ---- large sizes (rvk_oracle_mt.c: host threads, matrix-free) -------------------
def build_laplacian_rows(dim: int, points: int, grid, r0: int, r1: int):
    """Rows [r0, r1) of build_laplacian(dim, points, grid): (off, cols, vals)
    with offsets local to the slab (off[0] = 0)."""
    nx, ny, nz = (list(grid) + [1, 1])[:3]
    L = lib()
    # upper bound of the slab's nonzeros: points per row
    cap = (r1 - r0) * points
    off = np.empty(r1 - r0 + 1, np.int64)
    cols = np.empty(cap, np.int32)
    vals = np.empty(cap, np.float64)
    k = L.ro_build_laplacian_rows(dim, points, nx, ny, nz, r0, r1, off, cols, vals)
    if k < 0:
        raise ValueError(f"invalid rows [{r0}, {r1}) of {dim}D {points}-pt {grid}")
    return off, cols[:k], vals[:k]


def stencil_spmv(dim: int, points: int, grid, x: np.ndarray) -> np.ndarray:
    """A x for the Laplacian without assembling it (bit-identical to spmv on
    build_laplacian's CSR)."""
    nx, ny, nz = (list(grid) + [1, 1])[:3]
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty_like(x)
    lib().ro_stencil_spmv_mt(dim, points, nx, ny, nz, x, y)
    return y


def cg_solve_stencil(dim: int, points: int, grid, b: np.ndarray, max_it: int = 20,
                     pc: str = "jacobi", rtol: float = 0.0, atol: float = 0.0) -> CgResult:
    """cg_solve on the Laplacian, matrix-free and threaded (for the 768^3
    config); reductions in fixed chunks (rvk_oracle_mt.c header)."""
    nx, ny, nz = (list(grid) + [1, 1])[:3]
    b = np.ascontiguousarray(b, np.float64)
    n = b.shape[0]
    x = np.empty(n, np.float64)
    hist = np.full(max_it + 1, np.nan)
    work = np.empty(4 * n, np.float64)
    cfg = _CgCfg(max_it, 1 if pc == "jacobi" else 0, rtol, atol)
    r = lib().ro_cg_solve_stencil_mt(dim, points, nx, ny, nz, b, x, hist, cfg, work)
    return CgResult(x, hist[: r.iterations + 1].copy(), r.status, r.iterations, r.breakdown_iter)
