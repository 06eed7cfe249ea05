"""GPU parity of the one-launch grid solve (k_cg_grid, rvk_cg_small.cu;
RVK_PLAN_GRID): PERSISTENT / AUTO plans for 16 K < n <= ~450 K rows with
rows of <= 9 entries.  CSR in shared memory, row vectors in registers, two
grid barriers per iteration fused with the reductions (every CTA folds the
partials in the same order).  Bar: hist and x within 1e-10 of the oracle
(SPEC.md:466), repeatable bit for bit, early exits at the oracle's
iteration, the eligibility boundaries."""
import numpy as np
import pytest

import oracle as O
from paper_2306_17801_b200 import rvk
from test_gpu_parity import check_cg_floor

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("spec", [(2, 5, (129, 128)), (2, 5, (256, 256)), (2, 9, (300, 200)),
                                  (2, 5, (512, 512)), (3, 7, (40, 40, 40)), (3, 7, (64, 64, 32)),
                                  (2, 9, (512, 511)), (2, 5, (660, 660))],
                         ids=["5pt129x128", "5pt256", "9pt300x200", "5pt512", "7pt40", "7pt64x64x32",
                              "9pt512x511", "5pt660"])
@pytest.mark.parametrize("pc", ["jacobi", "none"])
def test_grid_solve_vs_oracle(ctx, spec, pc):
    dim, pts, g = spec
    Ah = O.build_laplacian(dim, pts, g)
    b = O.rhs(Ah.n_rows)
    A = rvk.DeviceCsr.laplacian(ctx, dim, pts, g)
    for max_it, rtol in ((20, 0.0), (300, 1e-6)):
        ref = O.cg_solve(Ah, b, max_it=max_it, rtol=rtol, pc=pc)
        for mode in ("auto", "persistent"):
            plan = rvk.CgPlan(ctx, A, max_it=max_it, rtol=rtol, pc=pc, mode=mode)
            assert plan.flags() & rvk.PLAN_GRID, plan.flags()
            x, res = plan.solve_host(b)
            check_cg_floor(res, x, ref)
            x2, res2 = plan.solve_host(b)
            assert np.array_equal(x, x2) and np.array_equal(res.hist, res2.hist)
            plan.close()


def test_grid_solve_eligibility(ctx):
    for dim, pts, g, want in [(2, 5, (64, 64), False),     # 4096 rows: the cluster solve
                              (2, 5, (128, 128), True),     # 16384: grid (cluster only <= 8 K rows)
                              (3, 27, (30, 30, 30), False),  # rows of 27 entries
                              (2, 5, (129, 128), True),
                              (2, 5, (660, 660), True),
                              (2, 5, (700, 700), True),    # > 148 x 3 x 1024 rows: the L2 variant
                              (2, 5, (778, 778), True),    # 4096 rows per CTA
                              (2, 5, (780, 780), False),   # AUTO: fused above 4 K rows per CTA
                              (2, 5, (1024, 1024), False)]:
        A = rvk.DeviceCsr.laplacian(ctx, dim, pts, g)
        plan = rvk.CgPlan(ctx, A, max_it=2, mode="auto")
        assert bool(plan.flags() & rvk.PLAN_GRID) == want, g
        l2 = g[0] * g[1] > 148 * 3072
        assert bool(plan.flags() & rvk.PLAN_GRID_L2) == (want and l2), g
        plan.close()
    # explicit PERSISTENT: the L2 grid solve up to 148 x 8 K rows
    for g, want in [((780, 780), True), ((1024, 1024), True), ((1110, 1100), False)]:
        A = rvk.DeviceCsr.laplacian(ctx, 2, 5, g)
        plan = rvk.CgPlan(ctx, A, max_it=2, mode="persistent")
        assert bool(plan.flags() & rvk.PLAN_GRID_L2) == want, g
        plan.close()
    A = rvk.DeviceCsr.laplacian(ctx, 2, 5, (700, 700))
    plan = rvk.CgPlan(ctx, A, max_it=2, mode="auto", opts=rvk.OPT_NO_GRID_L2)
    assert not plan.flags() & (rvk.PLAN_GRID | rvk.PLAN_GRID_L2)
    plan.close()
    A = rvk.DeviceCsr.laplacian(ctx, 2, 5, (256, 256))
    plan = rvk.CgPlan(ctx, A, max_it=2, mode="persistent", opts=rvk.OPT_NO_GRID)
    assert not plan.flags() & rvk.PLAN_GRID
    plan.close()


def permuted_spd(rng, grid):
    """P (L + D) P^T: a 2D 5-point Laplacian plus a random positive diagonal,
    symmetrically permuted -- rows of 3..5 entries, no band structure, a
    non-constant Jacobi diagonal."""
    L = O.build_laplacian(2, 5, grid)
    n = L.n_rows
    perm = rng.permutation(n)
    inv = np.empty(n, np.int64)
    inv[perm] = np.arange(n)
    rows = np.repeat(np.arange(n), np.diff(L.off))
    vals = L.vals.copy()
    vals[L.cols == rows] += rng.uniform(0.5, 2.0, n)[rows[L.cols == rows]]
    ii, jj = inv[rows], inv[L.cols.astype(np.int64)]
    order = np.lexsort((jj, ii))
    ii, jj, vv = ii[order], jj[order], vals[order]
    off = np.zeros(n + 1, np.int64)
    np.add.at(off, ii + 1, 1)
    return O.Csr(n, n, np.cumsum(off), jj.astype(np.int32), vv)


@pytest.mark.parametrize("spec", [(2, 5, (700, 700)), (2, 5, (1024, 1024)), (2, 9, (1024, 1000)),
                                  (3, 7, (100, 100, 100)), (3, 7, (80, 80, 80)), (3, 27, (40, 40, 40))],
                         ids=["5pt700", "5pt1024", "9pt1024x1000", "7pt100", "7pt80", "27pt40"])
def test_grid_solve_l2_vs_oracle(ctx, spec):
    """k_cg_grid_l2 (RVK_PLAN_GRID_L2): the matrix from the plan's global
    k-major ELL copy, x / r / p in shared memory -- 3 K .. 8 K rows per CTA
    (27-point rows exceed 9 entries: not eligible, the fused graph runs)."""
    dim, pts, g = spec
    Ah = O.build_laplacian(dim, pts, g)
    b = O.rhs(Ah.n_rows)
    A = rvk.DeviceCsr.laplacian(ctx, dim, pts, g)
    for pc in ("jacobi", "none"):
        for max_it, rtol in ((20, 0.0), (400, 1e-5)):
            ref = O.cg_solve(Ah, b, max_it=max_it, rtol=rtol, pc=pc)
            plan = rvk.CgPlan(ctx, A, max_it=max_it, rtol=rtol, pc=pc, mode="persistent")
            assert bool(plan.flags() & rvk.PLAN_GRID_L2) == (pts != 27), plan.flags()
            x, res = plan.solve_host(b)
            check_cg_floor(res, x, ref)
            x2, res2 = plan.solve_host(b)
            assert np.array_equal(x, x2) and np.array_equal(res.hist, res2.hist)
            plan.close()


@pytest.mark.parametrize("seed,grid", [(0, (200, 200)), (1, (450, 440)), (2, (800, 790))])
def test_grid_solve_irregular(ctx, seed, grid):
    rng = np.random.default_rng(seed)
    Ah = permuted_spd(rng, grid)
    n = Ah.n_rows
    A = rvk.DeviceCsr.from_host(ctx, n, n, Ah.off, Ah.cols, Ah.vals)
    b = O.rhs(n)
    ref = O.cg_solve(Ah, b, max_it=20)
    plan = rvk.CgPlan(ctx, A, max_it=20, mode="persistent")
    assert plan.flags() & rvk.PLAN_GRID
    assert bool(plan.flags() & rvk.PLAN_GRID_L2) == (n > 148 * 3072)
    x, res = plan.solve_host(b)
    check_cg_floor(res, x, ref)


@pytest.mark.parametrize("g", [(256, 256), (1024, 1024)])
def test_grid_solve_zero_rhs_and_host_syncs(ctx, g):
    A = rvk.DeviceCsr.laplacian(ctx, 2, 5, g)
    plan = rvk.CgPlan(ctx, A, max_it=20, mode="persistent")
    assert plan.flags() & rvk.PLAN_GRID
    x0, r0 = plan.solve_host(np.zeros(A.n_rows))
    assert r0.iterations == 0 and not np.any(x0)
    b = rvk.DeviceArray.from_host(ctx, O.rhs(A.n_rows))
    x = rvk.DeviceArray(A.n_rows)
    ctx.synchronize()
    before = rvk.host_syncs()
    plan.solve_dev(b, x)
    plan.solve_dev(b, x)
    assert rvk.host_syncs() == before   # one launch per solve, no host sync
    assert plan.result().iterations == 20
