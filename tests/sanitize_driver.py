"""Small workload run under compute-sanitizer by tests/test_gpu_sanitizer.py."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from paper_2306_17801_b200 import rvk  # noqa: E402


def main(parts=("csr", "mf", "dcg", "tfqmr", "irregular")):
    ctx = rvk.Ctx()
    if "csr" not in parts:
        return _rest(ctx, parts)
    for dim, pts, g in [(2, 5, (33, 17)), (3, 7, (9, 8, 7)), (3, 27, (7, 6, 5)), (2, 9, (40, 37))]:
        A = rvk.DeviceCsr.laplacian(ctx, dim, pts, g)
        b = O.rhs(A.n_rows)
        for mode in ("fused", "unfused", "persistent"):  # persistent: the cluster kernel (27-pt: grid barriers)
            for graph in (False, True):
                plan = rvk.CgPlan(ctx, A, max_it=20, mode=mode, use_graph=graph)
                x, res = plan.solve_host(b)
                assert res.iterations == 20
                plan.close()
    return _rest(ctx, parts)


def _rest(ctx, parts):
    # matrix-free operator: the TMA 2.5D kernel (even nx, partial tiles) and
    # the row-per-thread fallback (odd nx); WHILE-loop graph
    for dim, pts, g in ([(3, 7, (34, 10, 6)), (3, 27, (36, 18, 5)), (2, 9, (132, 9)),
                         (3, 7, (9, 8, 7))] if "mf" in parts else []):
        b = O.rhs(int(np.prod(g)))
        for graph in (True, False):
            plan = rvk.CgPlan(ctx, (dim, pts, g), max_it=20, use_graph=graph)
            x, res = plan.solve_host(b)
            assert res.iterations == 20
            plan.close()
    # row-sharded PEER kernels (in-kernel halo pushes, flag protocol) on one GPU
    from paper_2306_17801_b200.sharded import loopback_solve
    for backend in (("gather", "peer") if "dcg" in parts else ()):
        Ah = O.build_laplacian(3, 7, (12, 10, 9))
        x, res, _ = loopback_solve(ctx, 3, 7, (12, 10, 9), 3, O.rhs(Ah.n_rows), max_it=20,
                                   backend=backend, repeats=2)
        assert res.iterations == 20
    if "tfqmr" in parts:
        A = rvk.DeviceCsr.laplacian(ctx, 2, 5, (24, 20))
        tp = rvk.TfqmrPlan(ctx, A, max_it=10)
        db, dx = rvk.DeviceArray.from_host(ctx, O.rhs(A.n_rows)), rvk.DeviceArray(A.n_rows)
        tp.solve_dev(db, dx)
        tp.result()
        tp.close()
    if "irregular" not in parts:
        print("sanitize driver ok")
        return
    # irregular CSR with empty rows, a long row and odd nnz
    rng = np.random.default_rng(0)
    n = 3001
    lens = rng.integers(0, 9, n)
    lens[::7] = 0
    lens[100] = 2500
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum(lens)
    cols = np.concatenate([np.sort(rng.choice(n, L, replace=False)) for L in lens]).astype(np.int32)
    vals = rng.standard_normal(int(off[-1]))
    A = rvk.DeviceCsr.from_host(ctx, n, n, off, cols, vals)
    x = rvk.DeviceArray.from_host(ctx, rng.standard_normal(n))
    y = rvk.DeviceArray(n)
    A.spmv(ctx, x, y)
    ctx.synchronize()
    print("sanitize driver ok")


if __name__ == "__main__":
    main(tuple(sys.argv[1].split(",")) if len(sys.argv) > 1 else
         ("csr", "mf", "dcg", "tfqmr", "irregular"))
