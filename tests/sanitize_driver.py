"""Small workload run under compute-sanitizer by tests/test_gpu_sanitizer.py."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from paper_2306_17801_b200 import rvk  # noqa: E402


def main():
    ctx = rvk.Ctx()
    for dim, pts, g in [(2, 5, (33, 17)), (3, 7, (9, 8, 7)), (3, 27, (7, 6, 5)), (2, 9, (40, 37))]:
        A = rvk.DeviceCsr.laplacian(ctx, dim, pts, g)
        b = O.rhs(A.n_rows)
        for mode in ("fused", "unfused"):
            for graph in (False, True):
                plan = rvk.CgPlan(ctx, A, max_it=20, mode=mode, use_graph=graph)
                x, res = plan.solve_host(b)
                assert res.iterations == 20
                plan.close()
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
    main()
