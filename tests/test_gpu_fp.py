"""GPU parity of the fused persistent solve (k_cg_fp, rvk_cg_fp.cu;
RVK_PLAN_FPERSIST): each iteration's SpMV phase (the fused K1's TMA ring,
kept alive across iterations) and update phase in ONE cooperative launch,
grid barriers fused with the reductions.  AUTO runs it for fixed-iteration
solves past the grid solves when RVK_OPT_FPERSIST asks (measured level with
or slower than the fused graph, so opt-in); explicit PERSISTENT plans (with
RVK_OPT_NO_GRID) run it with tolerances too, draining the ring after the
exit.  Bar: hist and x within 1e-10 of the oracle, repeatable
bit for bit, the oracle's exit iteration, zero host syncs."""
import numpy as np
import pytest

import oracle as O
from paper_2306_17801_b200 import rvk
from test_gpu_grid_solve import permuted_spd
from test_gpu_parity import check_cg, check_cg_floor

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("spec", [(2, 5, (1024, 1024)), (2, 9, (1024, 1000)), (3, 7, (100, 100, 100)),
                                  (3, 7, (128, 128, 128)), (2, 5, (2048, 2048)), (3, 7, (160, 150, 140))],
                         ids=["5pt1024", "9pt1024x1000", "7pt100", "7pt128", "5pt2048", "7pt160x150x140"])
def test_fp_auto_fixed_iterations_vs_oracle(ctx, spec):
    dim, pts, g = spec
    Ah = O.build_laplacian(dim, pts, g)
    b = O.rhs(Ah.n_rows)
    ref = O.cg_solve(Ah, b, max_it=20)
    A = rvk.DeviceCsr.laplacian(ctx, dim, pts, g)
    plan = rvk.CgPlan(ctx, A, max_it=20, mode="auto", opts=rvk.OPT_FPERSIST)
    assert plan.flags() & rvk.PLAN_FPERSIST, plan.flags()
    assert plan.mode() == "persistent"
    x, res = plan.solve_host(b)
    check_cg(res, x, ref)
    x2, res2 = plan.solve_host(b)
    assert np.array_equal(x, x2) and np.array_equal(res.hist, res2.hist)
    plan.close()


@pytest.mark.parametrize("spec", [(2, 5, (700, 640)), (3, 7, (90, 90, 90)), (2, 9, (900, 900))])
@pytest.mark.parametrize("pc", ["jacobi", "none"])
def test_fp_tolerance_exit_drains_ring(ctx, spec, pc):
    """Explicit PERSISTENT without the grid solves: early exit at the
    oracle's iteration, the remaining iterations' stages drained."""
    dim, pts, g = spec
    Ah = O.build_laplacian(dim, pts, g)
    b = O.rhs(Ah.n_rows)
    A = rvk.DeviceCsr.laplacian(ctx, dim, pts, g)
    for max_it, rtol in ((400, 1e-6), (30, 0.0)):
        ref = O.cg_solve(Ah, b, max_it=max_it, rtol=rtol, pc=pc)
        plan = rvk.CgPlan(ctx, A, max_it=max_it, rtol=rtol, pc=pc, mode="persistent", opts=rvk.OPT_NO_GRID)
        assert plan.flags() & rvk.PLAN_FPERSIST
        x, res = plan.solve_host(b)
        check_cg_floor(res, x, ref)
        # the plan is reusable after a drained exit
        x2, res2 = plan.solve_host(b)
        assert np.array_equal(x, x2) and res2.iterations == res.iterations
        plan.close()


@pytest.mark.parametrize("seed,grid", [(3, (800, 790)), (4, (1100, 1000))])
def test_fp_irregular_nonconstant_diagonal(ctx, seed, grid):
    rng = np.random.default_rng(seed)
    Ah = permuted_spd(rng, grid)
    n = Ah.n_rows
    A = rvk.DeviceCsr.from_host(ctx, n, n, Ah.off, Ah.cols, Ah.vals)
    b = O.rhs(n)
    ref = O.cg_solve(Ah, b, max_it=20)
    plan = rvk.CgPlan(ctx, A, max_it=20, mode="persistent", opts=rvk.OPT_NO_GRID)
    assert plan.flags() & rvk.PLAN_FPERSIST
    assert not plan.flags() & 1   # RVK_PLAN_CONST_DIAG: the diagonal streams
    x, res = plan.solve_host(b)
    check_cg_floor(res, x, ref)


def test_fp_eligibility(ctx):
    for dim, pts, g, opts, want in [
            (2, 5, (1024, 1024), 0, False),                      # opt-in only
            (2, 5, (1024, 1024), rvk.OPT_FPERSIST, True),
            (2, 5, (700, 700), rvk.OPT_FPERSIST, False),         # the L2 grid solve first
            (2, 5, (700, 700), rvk.OPT_FPERSIST | rvk.OPT_NO_GRID_L2, True),
            (2, 5, (2048, 2049), rvk.OPT_FPERSIST, True),
            (3, 27, (60, 60, 60), rvk.OPT_FPERSIST, False),      # 27-entry rows: 4 consumer groups
            (2, 5, (1024, 1024), rvk.OPT_FPERSIST | rvk.OPT_NO_FPERSIST, False)]:
        A = rvk.DeviceCsr.laplacian(ctx, dim, pts, g)
        plan = rvk.CgPlan(ctx, A, max_it=20, mode="auto", opts=opts)
        assert bool(plan.flags() & rvk.PLAN_FPERSIST) == want, (g, opts)
        plan.close()
    # a tolerance solve stays on the fused graph in AUTO
    A = rvk.DeviceCsr.laplacian(ctx, 2, 5, (1024, 1024))
    plan = rvk.CgPlan(ctx, A, max_it=20, rtol=1e-8, mode="auto", opts=rvk.OPT_FPERSIST)
    assert not plan.flags() & rvk.PLAN_FPERSIST and plan.mode() == "fused"
    plan.close()


def test_fp_headline_size_forced(ctx):
    """RVK_OPT_FPERSIST at the 256^3 headline size (16.8 M rows)."""
    Ah = O.build_laplacian(3, 7, (256, 256, 256))
    b = O.rhs(Ah.n_rows)
    ref = O.cg_solve(Ah, b, max_it=20)
    A = rvk.DeviceCsr.laplacian(ctx, 3, 7, (256, 256, 256))
    plan = rvk.CgPlan(ctx, A, max_it=20, mode="auto", opts=rvk.OPT_FPERSIST)
    assert plan.flags() & rvk.PLAN_FPERSIST
    x, res = plan.solve_host(b)
    check_cg(res, x, ref)


def test_fp_zero_rhs_and_host_syncs(ctx):
    A = rvk.DeviceCsr.laplacian(ctx, 2, 5, (1024, 1024))
    plan = rvk.CgPlan(ctx, A, max_it=20, mode="auto", opts=rvk.OPT_FPERSIST)
    assert plan.flags() & rvk.PLAN_FPERSIST
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
