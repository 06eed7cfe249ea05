"""Generate tests/golden/cg_golden.json and tfqmr_golden.json from the
REFERENCE's own kernels.

Run here (needs oracle/_ref, i.e. /root/reference at build time):
    python tests/golden/make_golden.py

Every vector/matrix operation of each solve goes through
/root/reference/proj/src/kernels_scalar.cpp (oracle/_ref/librivulet_ref.so,
backend 0 = the documented reference summation order, kernels_scalar.cpp:8-9).
The CG loop order is SPEC.md:458-466 / PAPER.md:104-150 (restated in
oracle/ref_shim.cpp because solvers.cpp is absent from the reference tree).
The CSR comes from the restated SPEC.md:526-550 builder; its bytes are hashed
so any drift in assembly is caught.  Values are stored as float.hex() strings
so the fixture is bit-exact.
"""
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import oracle as O  # noqa: E402

CASES = [
    # (name, dim, points, grid, pc)  -- SPEC.md:626 grids 16^2, 32^2, 8^3 x 4 stencils
    ("5pt_16x16", 2, 5, (16, 16), "jacobi"),
    ("5pt_32x32", 2, 5, (32, 32), "jacobi"),
    ("9pt_16x16", 2, 9, (16, 16), "jacobi"),
    ("9pt_32x32", 2, 9, (32, 32), "jacobi"),
    ("7pt_8x8x8", 3, 7, (8, 8, 8), "jacobi"),
    ("27pt_8x8x8", 3, 27, (8, 8, 8), "jacobi"),
    # ragged / non-cubic grids and the no-preconditioner path
    ("5pt_7x5", 2, 5, (7, 5), "jacobi"),
    ("7pt_5x4x3", 3, 7, (5, 4, 3), "jacobi"),
    ("27pt_6x5x4", 3, 27, (6, 5, 4), "jacobi"),
    ("9pt_16x16_nopc", 2, 9, (16, 16), "none"),
]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def hexs(a):
    return [float(v).hex() for v in np.asarray(a, np.float64)]


def main():
    out = {"generator": "oracle/_ref (reference kernels_scalar.cpp) via tests/golden/make_golden.py",
           "seed": hex(O.DEFAULT_SEED), "max_it": 20, "cases": []}
    for name, dim, pts, grid, pc in CASES:
        A = O.build_laplacian(dim, pts, grid)
        b = O.rhs(A.n_rows)
        r = O.ref_cg_solve(A, b, max_it=20, pc=pc, backend=0)
        out["cases"].append({
            "name": name, "dim": dim, "points": pts, "grid": list(grid), "pc": pc,
            "n": A.n_rows, "nnz": A.nnz,
            "sha_off": sha(A.off), "sha_cols": sha(A.cols), "sha_vals": sha(A.vals),
            "sha_b": sha(b), "status": r.status, "iterations": r.iterations,
            "hist": hexs(r.hist), "x": hexs(r.x),
            # SpMV of the RHS through the reference kernel: bit-exact target
            "spmv_b": hexs(O.ref_spmv(A, b, backend=0)),
        })
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cg_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=0)
    print("wrote", path, os.path.getsize(path), "bytes")
    tfqmr()


TFQMR_CASES = [
    # (name, dim, points, grid, pc, max_it, rtol)  -- SPEC.md:467-475 left-Jacobi TFQMR
    ("5pt_16x16", 2, 5, (16, 16), "jacobi", 20, 0.0),
    ("5pt_32x32", 2, 5, (32, 32), "jacobi", 20, 0.0),
    ("9pt_32x32", 2, 9, (32, 32), "jacobi", 20, 0.0),
    ("7pt_8x8x8", 3, 7, (8, 8, 8), "jacobi", 20, 0.0),
    ("27pt_8x8x8", 3, 27, (8, 8, 8), "jacobi", 20, 0.0),
    ("7pt_5x4x3", 3, 7, (5, 4, 3), "jacobi", 20, 0.0),
    ("9pt_16x16_nopc", 2, 9, (16, 16), "none", 20, 0.0),
    # device-side exit inside an outer iteration (rtol on the residual bound)
    ("5pt_24x20_rtol", 2, 5, (24, 20), "jacobi", 200, 1e-6),
]


def tfqmr():
    """The TFQMR loop of oracle/ref_shim.cpp:ref_tfqmr_solve: every vector and
    matrix operation through kernels_scalar.cpp (backend 0)."""
    out = {"generator": "oracle/_ref (reference kernels_scalar.cpp) via ref_tfqmr_solve, "
                        "tests/golden/make_golden.py",
           "seed": hex(O.DEFAULT_SEED), "cases": []}
    for name, dim, pts, grid, pc, max_it, rtol in TFQMR_CASES:
        A = O.build_laplacian(dim, pts, grid)
        b = O.rhs(A.n_rows)
        r = O.ref_tfqmr_solve(A, b, max_it=max_it, pc=pc, rtol=rtol, backend=0)
        out["cases"].append({
            "name": name, "dim": dim, "points": pts, "grid": list(grid), "pc": pc,
            "max_it": max_it, "rtol": rtol, "n": A.n_rows, "sha_b": sha(b),
            "status": r.status, "iterations": r.iterations, "hist": hexs(r.hist), "x": hexs(r.x)})
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "tfqmr_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=0)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
