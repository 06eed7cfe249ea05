"""ctypes binding of librvk.so (include/rvk.h) -- the sm_100a Jacobi-CG path.

This is a thin host-side mirror of the C ABI used by the tests and bench.py;
it has NO compute fallback: if librvk.so is missing or no CUDA device is
present, every call fails loudly.  The C++ drop-in API for the reference's
rivulet::linalg / cg_solve surface lives in include/rivulet/ + csrc/api/.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "librvk.so")

RVK_OK = 0
RVK_ERR_BREAKDOWN = 5
RVK_ERR_COMM = 6
SCALAR_CONST, SCALAR_PTR, SCALAR_NEG_PTR, SCALAR_DIV, SCALAR_SQRT, SCALAR_RECIP = range(6)
PC_NONE, PC_JACOBI = 0, 1
MODE_FUSED, MODE_UNFUSED, MODE_PERSISTENT, MODE_AUTO, MODE_HOSTSYNC = 0, 1, 2, 3, 4
MODES = {"fused": MODE_FUSED, "unfused": MODE_UNFUSED, "persistent": MODE_PERSISTENT,
         "auto": MODE_AUTO, "hostsync": MODE_HOSTSYNC}
CG_RUNNING, CG_CONVERGED, CG_BREAKDOWN, CG_COMM_ERROR = 0, 1, 2, 3

# every symbol include/rvk.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "rvk_last_error", "rvk_abi_version", "rvk_build_id", "rvk_device_info", "rvk_device_count", "rvk_set_device",
    "rvk_ctx_create", "rvk_ctx_destroy", "rvk_ctx_stream", "rvk_ctx_synchronize",
    "rvk_ctx_query_idle", "rvk_ctx_wait_for", "rvk_ctx_id", "rvk_ctx_set_name",
    "rvk_host_sync_count", "rvk_host_sync_reset",
    "rvk_trace_enable", "rvk_trace_enabled", "rvk_trace_clear", "rvk_trace_marker", "rvk_trace_count",
    "rvk_trace_write_jsonl", "rvk_trace_write_chrome",
    "rvk_malloc", "rvk_free", "rvk_malloc_async", "rvk_free_async", "rvk_host_alloc", "rvk_host_free", "rvk_memcpy_h2d",
    "rvk_memcpy_d2h", "rvk_memcpy_d2d", "rvk_scalar_eval", "rvk_scalar_read",
    "rvk_dot", "rvk_nrm2", "rvk_dot2", "rvk_axpy", "rvk_aypx", "rvk_waxpy", "rvk_scale",
    "rvk_pointwise_mult", "rvk_copy", "rvk_set", "rvk_csr_spmv", "rvk_csr_diagonal",
    "rvk_csr_diagonal_inverse", "rvk_csr_validate", "rvk_laplacian_size",
    "rvk_build_laplacian", "rvk_fill_rhs", "rvk_cg_plan_create", "rvk_cg_plan_create_stencil", "rvk_cg_plan_destroy",
    "rvk_cg_solve_dev", "rvk_cg_history_dev", "rvk_cg_result", "rvk_cg_solve_host",
    "rvk_cg_solve_host_many",
    "rvk_cg_set_profiling", "rvk_cg_kernel_times", "rvk_cg_plan_mode", "rvk_cg_plan_flags",
    "rvk_cg_plan_vector",
    "rvk_laplacian_rows_nnz", "rvk_build_laplacian_rows", "rvk_comm_unique_id", "rvk_comm_init",
    "rvk_comm_destroy", "rvk_comm_size", "rvk_dcg_plan_create", "rvk_dcg_plan_destroy", "rvk_dcg_solve_dev",
    "rvk_dcg_loopback_solve", "rvk_dcg_result", "rvk_dcg_plan_flags", "rvk_dcg_window", "rvk_dcg_attach_peers",
    "rvk_ipc_get_handle", "rvk_ipc_open_handle", "rvk_ipc_close_handle", "rvk_tfqmr_plan_create",
    "rvk_tfqmr_plan_destroy", "rvk_tfqmr_solve_dev", "rvk_tfqmr_result", "rvk_tfqmr_plan_flags",
]


class RvkError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"rvk status {status}: {msg}")
        self.status = status


class BreakdownError(RvkError):
    """common.hpp:33-43 BreakdownError(iteration)."""

    def __init__(self, status, msg, iteration):
        super().__init__(status, msg)
        self.iteration = iteration


class Scalar(C.Structure):
    _fields_ = [("kind", C.c_int), ("c", C.c_double), ("p0", C.c_void_p), ("p1", C.c_void_p)]


class Csr(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("n_cols", C.c_int64), ("nnz", C.c_int64),
                ("row_offsets", C.c_void_p), ("col_indices", C.c_void_p), ("values", C.c_void_p)]


class CgConfig(C.Structure):
    _fields_ = [("max_it", C.c_int), ("pc", C.c_int), ("rtol", C.c_double),
                ("atol", C.c_double), ("mode", C.c_int), ("use_graph", C.c_int),
                ("opts", C.c_int)]


# rvk_cg_config.opts (include/rvk.h RVK_OPT_*): explicit plan-variant overrides
OPT_KEEP_WORK, OPT_DINV_VECTOR, OPT_Z_STORED, OPT_Z_VIRTUAL = 1, 2, 4, 8
OPT_NO_CLUSTER, OPT_SMALL_K1, OPT_MF_SIMPLE, OPT_NO_FOLD = 16, 32, 64, 128
OPT_X_GROUP4, OPT_X_EACH = 256, 512
OPT_MARCH, OPT_NO_GRID, OPT_NO_GRID_L2, OPT_FPERSIST, OPT_NO_FPERSIST = 1024, 4096, 8192, 16384, 32768
PLAN_MARCH, PLAN_GRID, PLAN_GRID_L2, PLAN_FPERSIST = 1024, 2048, 4096, 8192


class Shard(C.Structure):
    _fields_ = [("n_own", C.c_int64), ("halo_lo", C.c_int64), ("halo_hi", C.c_int64),
                ("rank", C.c_int), ("nranks", C.c_int)]


class CgInfo(C.Structure):
    _fields_ = [("state", C.c_int), ("iterations", C.c_int), ("breakdown_iter", C.c_int)]


_lib = None


def lib():
    """Load librvk.so (raises if it was not built -- there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() "
                          "(make -C paper_2306_17801_b200)")
    L = C.CDLL(LIB_PATH)
    vp, i64, d, i = C.c_void_p, C.c_int64, C.c_double, C.c_int
    sig = {
        "rvk_last_error": (C.c_char_p, []),
        "rvk_abi_version": (i, []),
        "rvk_build_id": (C.c_char_p, []),
        "rvk_device_count": (i, []),
        "rvk_set_device": (i, [i]),
        "rvk_device_info": (i, [C.POINTER(C.c_int), C.c_char_p, i]),
        "rvk_ctx_create": (i, [vp, C.POINTER(vp)]),
        "rvk_ctx_destroy": (i, [vp]),
        "rvk_ctx_stream": (vp, [vp]),
        "rvk_ctx_synchronize": (i, [vp]),
        "rvk_ctx_query_idle": (i, [vp, C.POINTER(C.c_int)]),
        "rvk_ctx_wait_for": (i, [vp, vp]),
        "rvk_ctx_id": (C.c_uint64, [vp]),
        "rvk_ctx_set_name": (i, [vp, C.c_char_p]),
        "rvk_host_sync_count": (C.c_uint64, []),
        "rvk_trace_enable": (None, [i]),
        "rvk_trace_enabled": (i, []),
        "rvk_trace_clear": (None, []),
        "rvk_trace_marker": (None, [C.c_char_p]),
        "rvk_trace_count": (C.c_size_t, []),
        "rvk_trace_write_jsonl": (i, [C.c_char_p]),
        "rvk_trace_write_chrome": (i, [C.c_char_p]),
        "rvk_host_sync_reset": (None, []),
        "rvk_malloc": (i, [C.POINTER(vp), C.c_size_t]),
        "rvk_free": (i, [vp]),
        "rvk_malloc_async": (i, [vp, C.POINTER(vp), C.c_size_t]),
        "rvk_free_async": (i, [vp, vp]),
        "rvk_host_alloc": (i, [C.POINTER(vp), C.c_size_t]),
        "rvk_host_free": (i, [vp]),
        "rvk_memcpy_h2d": (i, [vp, vp, vp, C.c_size_t]),
        "rvk_memcpy_d2h": (i, [vp, vp, vp, C.c_size_t]),
        "rvk_memcpy_d2d": (i, [vp, vp, vp, C.c_size_t]),
        "rvk_scalar_eval": (i, [vp, Scalar, vp]),
        "rvk_scalar_read": (i, [vp, vp, C.POINTER(d)]),
        "rvk_dot": (i, [vp, i64, vp, vp, vp]),
        "rvk_nrm2": (i, [vp, i64, vp, vp]),
        "rvk_dot2": (i, [vp, i64, vp, vp, vp, vp]),
        "rvk_axpy": (i, [vp, i64, Scalar, vp, vp]),
        "rvk_aypx": (i, [vp, i64, Scalar, vp, vp]),
        "rvk_waxpy": (i, [vp, i64, Scalar, vp, vp, vp]),
        "rvk_scale": (i, [vp, i64, Scalar, vp]),
        "rvk_pointwise_mult": (i, [vp, i64, vp, vp, vp]),
        "rvk_copy": (i, [vp, i64, vp, vp]),
        "rvk_set": (i, [vp, i64, d, vp]),
        "rvk_csr_spmv": (i, [vp, C.POINTER(Csr), vp, vp]),
        "rvk_csr_diagonal": (i, [vp, C.POINTER(Csr), vp]),
        "rvk_csr_diagonal_inverse": (i, [vp, C.POINTER(Csr), vp]),
        "rvk_csr_validate": (i, [vp, C.POINTER(Csr), C.POINTER(i64)]),
        "rvk_laplacian_size": (i, [i, i, i64, i64, i64, C.POINTER(i64), C.POINTER(i64)]),
        "rvk_build_laplacian": (i, [vp, i, i, i64, i64, i64, vp, vp, vp]),
        "rvk_fill_rhs": (i, [vp, C.c_uint64, i64, vp]),
        "rvk_cg_plan_create": (i, [vp, C.POINTER(Csr), CgConfig, C.POINTER(vp)]),
        "rvk_cg_plan_create_stencil": (i, [vp, i, i, i64, i64, i64, CgConfig, C.POINTER(vp)]),
        "rvk_cg_plan_destroy": (i, [vp]),
        "rvk_cg_solve_dev": (i, [vp, vp, vp]),
        "rvk_cg_history_dev": (vp, [vp]),
        "rvk_cg_result": (i, [vp, vp, C.POINTER(CgInfo)]),
        "rvk_cg_solve_host": (i, [vp, vp, vp, vp, C.POINTER(CgInfo)]),
        "rvk_cg_solve_host_many": (i, [vp, i, C.POINTER(vp), C.POINTER(vp), vp,
                                       C.POINTER(CgInfo)]),
        "rvk_cg_set_profiling": (i, [vp, i]),
        "rvk_cg_kernel_times": (i, [vp, C.POINTER(C.c_float), C.POINTER(C.c_float),
                                    C.POINTER(C.c_int)]),
        "rvk_cg_plan_mode": (i, [vp]),
        "rvk_cg_plan_flags": (i, [vp]),
        "rvk_cg_plan_vector": (vp, [vp, i]),
        "rvk_laplacian_rows_nnz": (i, [i, i, i64, i64, i64, i64, i64, C.POINTER(i64)]),
        "rvk_build_laplacian_rows": (i, [vp, i, i, i64, i64, i64, i64, i64, i64, vp, vp, vp]),
        "rvk_comm_unique_id": (i, [vp, i]),
        "rvk_comm_init": (i, [vp, i, i, C.POINTER(vp)]),
        "rvk_comm_destroy": (i, [vp]),
        "rvk_comm_size": (i, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
        "rvk_dcg_plan_create": (i, [vp, C.POINTER(Csr), Shard, CgConfig, vp, vp, C.POINTER(vp)]),
        "rvk_dcg_plan_destroy": (i, [vp]),
        "rvk_dcg_solve_dev": (i, [vp, vp, vp]),
        "rvk_dcg_loopback_solve": (i, [C.POINTER(vp), i, C.POINTER(vp), C.POINTER(vp)]),
        "rvk_dcg_result": (i, [vp, vp, C.POINTER(CgInfo)]),
        "rvk_dcg_plan_flags": (i, [vp]),
        "rvk_dcg_window": (i, [vp, C.POINTER(vp), C.POINTER(C.c_size_t)]),
        "rvk_dcg_attach_peers": (i, [vp, C.POINTER(vp), C.POINTER(Shard)]),
        "rvk_ipc_get_handle": (i, [vp, vp, i]),
        "rvk_ipc_open_handle": (i, [vp, C.POINTER(vp)]),
        "rvk_ipc_close_handle": (i, [vp]),
        "rvk_tfqmr_plan_create": (i, [vp, C.POINTER(Csr), CgConfig, C.POINTER(vp)]),
        "rvk_tfqmr_plan_destroy": (i, [vp]),
        "rvk_tfqmr_solve_dev": (i, [vp, vp, vp]),
        "rvk_tfqmr_result": (i, [vp, vp, C.POINTER(C.c_int), C.POINTER(CgInfo)]),
        "rvk_tfqmr_plan_flags": (i, [vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(status: int) -> None:
    if status != RVK_OK:
        msg = lib().rvk_last_error().decode(errors="replace")
        raise RvkError(status, msg)


def host_syncs() -> int:
    return int(lib().rvk_host_sync_count())


class trace:
    """rvk_trace_* (reference trace.hpp:11-46): Task / Wait / HostSync /
    Marker events, device-timed tasks, JSONL and Chrome-trace export."""

    @staticmethod
    def enable(on: bool = True):
        lib().rvk_trace_enable(1 if on else 0)

    @staticmethod
    def enabled() -> bool:
        return bool(lib().rvk_trace_enabled())

    @staticmethod
    def clear():
        lib().rvk_trace_clear()

    @staticmethod
    def marker(label: str):
        lib().rvk_trace_marker(label.encode())

    @staticmethod
    def count() -> int:
        return int(lib().rvk_trace_count())

    @staticmethod
    def write_jsonl(path: str):
        check(lib().rvk_trace_write_jsonl(os.fsencode(path)))

    @staticmethod
    def write_chrome(path: str):
        check(lib().rvk_trace_write_chrome(os.fsencode(path)))

    @staticmethod
    def events(tmp_path: str) -> list:
        import json
        trace.write_jsonl(tmp_path)
        with open(tmp_path) as f:
            return [json.loads(line) for line in f if line.strip()]


def device_info():
    n = C.c_int(0)
    name = C.create_string_buffer(128)
    check(lib().rvk_device_info(C.byref(n), name, 128))
    return n.value, name.value.decode()


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


class Ctx:
    """rvk_ctx: one CUDA stream + reduction scratch (PetscDeviceContext)."""

    def __init__(self, stream: int | None = None):
        h = C.c_void_p()
        check(lib().rvk_ctx_create(stream, C.byref(h)))
        self.h = h
        self._deps = weakref.WeakSet()   # plans bound to this context

    def close(self):
        if self.h:
            for d in list(self._deps):     # a plan must not outlive its stream
                d.close()
            lib().rvk_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return lib().rvk_ctx_stream(self.h)

    def synchronize(self):
        check(lib().rvk_ctx_synchronize(self.h))

    def idle(self) -> bool:
        v = C.c_int(0)
        check(lib().rvk_ctx_query_idle(self.h, C.byref(v)))
        return bool(v.value)

    def wait_for(self, other: "Ctx"):
        check(lib().rvk_ctx_wait_for(self.h, other.h))

    @property
    def id(self) -> int:
        return int(lib().rvk_ctx_id(self.h))

    def set_name(self, name: str):
        check(lib().rvk_ctx_set_name(self.h, name.encode()))


class DeviceArray:
    """Owning device buffer (plumbing for tests/bench)."""

    def __init__(self, n: int, dtype=np.float64):
        self.n = int(n)
        self.dtype = np.dtype(dtype)
        p = C.c_void_p()
        check(lib().rvk_malloc(C.byref(p), max(self.n, 1) * self.dtype.itemsize))
        self.ptr = p.value

    @classmethod
    def from_host(cls, ctx: Ctx, a: np.ndarray):
        a = np.ascontiguousarray(a)
        d = cls(a.shape[0], a.dtype)
        d.upload(ctx, a)
        return d

    @property
    def nbytes(self) -> int:
        return self.n * self.dtype.itemsize

    def upload(self, ctx: Ctx, a: np.ndarray):
        a = np.ascontiguousarray(a, self.dtype)
        assert a.shape[0] == self.n
        check(lib().rvk_memcpy_h2d(ctx.h, self.ptr, _ptr(a), self.nbytes))
        ctx.synchronize()

    def download(self, ctx: Ctx) -> np.ndarray:
        out = np.empty(self.n, self.dtype)
        check(lib().rvk_memcpy_d2h(ctx.h, _ptr(out), self.ptr, self.nbytes))
        ctx.synchronize()
        return out

    def download_range(self, ctx: Ctx, start: int, count: int) -> np.ndarray:
        """Elements [start, start + count) to a new host array."""
        assert 0 <= start and start + count <= self.n
        out = np.empty(count, self.dtype)
        if count:
            check(lib().rvk_memcpy_d2h(ctx.h, _ptr(out), self.ptr + start * self.dtype.itemsize,
                                       count * self.dtype.itemsize))
            ctx.synchronize()
        return out

    def free(self):
        if self.ptr:
            lib().rvk_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def scalar_const(c: float) -> Scalar:
    return Scalar(SCALAR_CONST, c, None, None)


def scalar_ptr(p: int, kind: int = SCALAR_PTR, p1: int | None = None) -> Scalar:
    return Scalar(kind, 0.0, p, p1)


class DeviceCsr:
    """CSR on device (int64 offsets, int32 columns, float64 values)."""

    def __init__(self, n_rows, n_cols, off: DeviceArray, cols: DeviceArray, vals: DeviceArray):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.off, self.cols, self.vals = off, cols, vals
        self.nnz = cols.n
        self.c = Csr(self.n_rows, self.n_cols, self.nnz, off.ptr, cols.ptr, vals.ptr)

    @classmethod
    def from_host(cls, ctx: Ctx, n_rows, n_cols, off, cols, vals):
        return cls(n_rows, n_cols, DeviceArray.from_host(ctx, np.asarray(off, np.int64)),
                   DeviceArray.from_host(ctx, np.asarray(cols, np.int32)),
                   DeviceArray.from_host(ctx, np.asarray(vals, np.float64)))

    @classmethod
    def laplacian(cls, ctx: Ctx, dim: int, points: int, grid):
        """Device-side assembly (rvk_build_laplacian)."""
        nx, ny, nz = (list(grid) + [1, 1])[:3]
        n, nnz = C.c_int64(), C.c_int64()
        check(lib().rvk_laplacian_size(dim, points, nx, ny, nz, C.byref(n), C.byref(nnz)))
        off = DeviceArray(n.value + 1, np.int64)
        cols = DeviceArray(nnz.value, np.int32)
        vals = DeviceArray(nnz.value, np.float64)
        check(lib().rvk_build_laplacian(ctx.h, dim, points, nx, ny, nz, off.ptr, cols.ptr,
                                        vals.ptr))
        return cls(n.value, n.value, off, cols, vals)

    def validate(self, ctx: Ctx) -> int:
        ml = C.c_int64()
        check(lib().rvk_csr_validate(ctx.h, C.byref(self.c), C.byref(ml)))
        return ml.value

    def spmv(self, ctx: Ctx, x: DeviceArray, y: DeviceArray):
        check(lib().rvk_csr_spmv(ctx.h, C.byref(self.c), x.ptr, y.ptr))


@dataclass
class CgResult:
    hist: np.ndarray
    state: int
    iterations: int
    breakdown_iter: int


class CgPlan:
    """KSPSetUp + KSPSolve for Jacobi-PCG (rvk_cg_plan_*).  A is a DeviceCsr,
    or a stencil spec (dim, points, grid) for the matrix-free operator."""

    def __init__(self, ctx: Ctx, A, max_it: int = 20, pc: str = "jacobi",
                 rtol: float = 0.0, atol: float = 0.0, mode: str = "fused",
                 use_graph: bool = True, opts: int = 0):
        self.ctx, self.A = ctx, A
        self.max_it = max_it
        graph = 2 if use_graph == "while" else (1 if use_graph else 0)
        cfg = CgConfig(max_it, PC_JACOBI if pc == "jacobi" else PC_NONE, rtol, atol,
                       MODES[mode], graph, opts)
        h = C.c_void_p()
        if isinstance(A, DeviceCsr):
            self.n = A.n_rows
            check(lib().rvk_cg_plan_create(ctx.h, C.byref(A.c), cfg, C.byref(h)))
        else:
            dim, points, grid = A
            nx, ny, nz = (list(grid) + [1, 1])[:3]
            self.n = nx * ny * (nz if dim == 3 else 1)
            check(lib().rvk_cg_plan_create_stencil(ctx.h, dim, points, nx, ny, nz, cfg,
                                                   C.byref(h)))
        self.h = h
        ctx._deps.add(self)

    def close(self):
        if self.h:
            lib().rvk_cg_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def solve_dev(self, b: DeviceArray, x: DeviceArray):
        check(lib().rvk_cg_solve_dev(self.h, b.ptr, x.ptr))

    def result(self, raise_breakdown: bool = True) -> CgResult:
        hist = np.full(self.max_it + 1, np.nan)
        info = CgInfo()
        st = lib().rvk_cg_result(self.h, _ptr(hist), C.byref(info))
        res = CgResult(hist[: info.iterations + 1].copy(), info.state, info.iterations,
                       info.breakdown_iter)
        if st == RVK_ERR_BREAKDOWN:
            if raise_breakdown:
                raise BreakdownError(st, lib().rvk_last_error().decode(), info.breakdown_iter)
            return res
        check(st)
        return res

    def solve_host(self, b: np.ndarray, x_out: np.ndarray | None = None, hist_out=None):
        b = np.ascontiguousarray(b, np.float64)
        x = x_out if x_out is not None else np.empty_like(b)
        hist = hist_out if hist_out is not None else np.full(self.max_it + 1, np.nan)
        info = CgInfo()
        st = lib().rvk_cg_solve_host(self.h, _ptr(b), _ptr(x), _ptr(hist), C.byref(info))
        if st not in (RVK_OK, RVK_ERR_BREAKDOWN):
            check(st)
        return x, CgResult(hist[: info.iterations + 1].copy(), info.state, info.iterations,
                           info.breakdown_iter)

    def solve_host_many(self, bs: list, xs: list):
        """Pipelined solves of several host right-hand sides (rvk_cg_solve_host_many).
        bs / xs: float64 arrays (pinned -- e.g. torch pin_memory -- for overlap).
        Returns the per-RHS CgResults."""
        n = len(bs)
        B = (C.c_void_p * n)(*[_ptr(b) for b in bs])
        X = (C.c_void_p * n)(*[_ptr(x) for x in xs])
        H = self.max_it + 1
        hist = np.full(n * H, np.nan)
        infos = (CgInfo * n)()
        st = lib().rvk_cg_solve_host_many(self.h, n, B, X, _ptr(hist), infos)
        if st not in (RVK_OK, RVK_ERR_BREAKDOWN):
            check(st)
        return [CgResult(hist[k * H: k * H + infos[k].iterations + 1].copy(), infos[k].state,
                         infos[k].iterations, infos[k].breakdown_iter) for k in range(n)]

    def set_profiling(self, on: bool):
        check(lib().rvk_cg_set_profiling(self.h, 1 if on else 0))

    def kernel_times(self):
        a, b, n = C.c_float(), C.c_float(), C.c_int()
        check(lib().rvk_cg_kernel_times(self.h, C.byref(a), C.byref(b), C.byref(n)))
        return a.value, b.value, n.value

    def flags(self) -> int:
        """RVK_PLAN_* bits: 1 constant diagonal folded to a scalar, 2 matrix-free,
        4 matrix-free via the TMA 2.5D kernel, 8 int32 row offsets streamed."""
        return lib().rvk_cg_plan_flags(self.h)

    VEC = {"r": 0, "z": 1, "p0": 2, "p1": 3, "w": 4}

    def work_vector(self, which: str) -> np.ndarray:
        """Test hook: a plan work vector (after a synchronised solve)."""
        ptr = lib().rvk_cg_plan_vector(self.h, self.VEC[which])
        out = np.empty(self.n, np.float64)
        check(lib().rvk_memcpy_d2h(self.ctx.h, out.ctypes.data, ptr, out.nbytes))
        check(lib().rvk_ctx_synchronize(self.ctx.h))
        return out

    def mode(self) -> str:
        m = lib().rvk_cg_plan_mode(self.h)
        return {v: k for k, v in MODES.items()}[m]

    def launches(self) -> int:
        n = C.c_int()
        lib().rvk_cg_kernel_times(self.h, None, None, C.byref(n))
        return n.value


class TfqmrPlan:
    """KSPSetUp + KSPSolve for left-Jacobi TFQMR (rvk_tfqmr_plan_*).
    result().hist = ||B r0|| then one quasi-residual estimate per half step."""

    def __init__(self, ctx: Ctx, A: DeviceCsr, max_it: int = 20, pc: str = "jacobi",
                 rtol: float = 0.0, atol: float = 0.0, use_graph: bool = True,
                 mode: str = "fused", opts: int = 0):
        self.ctx, self.A, self.max_it = ctx, A, max_it
        cfg = CgConfig(max_it, PC_JACOBI if pc == "jacobi" else PC_NONE, rtol, atol,
                       MODES[mode], 1 if use_graph else 0, opts)
        h = C.c_void_p()
        check(lib().rvk_tfqmr_plan_create(ctx.h, C.byref(A.c), cfg, C.byref(h)))
        self.h = h
        ctx._deps.add(self)

    def close(self):
        if self.h:
            lib().rvk_tfqmr_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def solve_dev(self, b: DeviceArray, x: DeviceArray):
        check(lib().rvk_tfqmr_solve_dev(self.h, b.ptr, x.ptr))

    def flags(self) -> int:
        """RVK_PLAN_* bits (CONST_DIAG = 1)."""
        return lib().rvk_tfqmr_plan_flags(self.h)

    def result(self, raise_breakdown: bool = True) -> CgResult:
        hist = np.full(2 * self.max_it + 1, np.nan)
        info, nh = CgInfo(), C.c_int()
        st = lib().rvk_tfqmr_result(self.h, _ptr(hist), C.byref(nh), C.byref(info))
        res = CgResult(hist[: nh.value].copy(), info.state, info.iterations, info.breakdown_iter)
        if st == RVK_ERR_BREAKDOWN:
            if raise_breakdown:
                raise BreakdownError(st, lib().rvk_last_error().decode(), info.breakdown_iter)
            return res
        check(st)
        return res
