"""GPU parity of the plane-marching K1 (csrc/rvk_spmv_march.cuh,
RVK_PLAN_MARCH): each SM walks an in-plane row range through the planes
with the formed gathered operand of planes k-1, k, k+1 cached in shared
memory.  Row sums keep the reference's order (kernels_scalar.cpp:53-63), so
w and p_new are BIT-identical to the row-order TMA kernel; the solve agrees
with the oracle within 1e-10 (the p.w reduction groups rows per SM range, a
different -- still fixed -- order).  Grids: plane sizes Q = nx ny that are
multiples of 32 with Q / 32 >= 148 ranges (the kernel's precondition), range
halos (in-plane +-1 / +-nx / 27-point corners crossing a range boundary are
global gathers), ranges shorter than one tile, the minimum of 3 planes."""
import numpy as np
import pytest

import oracle as O
from paper_2306_17801_b200 import rvk

pytestmark = pytest.mark.gpu

SPECS = [(3, 7, (96, 64, 12)), (3, 27, (96, 64, 9)), (3, 7, (160, 96, 5)), (3, 7, (128, 48, 3)),
         (3, 27, (80, 64, 6)), (3, 7, (256, 256, 24))]
IDS = ["7pt96x64x12", "27pt96x64x9", "7pt160x96x5", "7pt128x48x3", "27pt80x64x6", "7pt256x256x24"]


@pytest.mark.parametrize("spec", SPECS, ids=IDS)
@pytest.mark.parametrize("zv", [False, True])
def test_march_w_p_bitexact_vs_row_order(ctx, spec, zv):
    dim, pts, g = spec
    A = rvk.DeviceCsr.laplacian(ctx, dim, pts, g)
    b = O.rhs(A.n_rows)
    zopt = rvk.OPT_Z_VIRTUAL if zv else rvk.OPT_Z_STORED
    out = {}
    for name, opt in (("march", rvk.OPT_MARCH), ("rows", 0)):
        plan = rvk.CgPlan(ctx, A, max_it=2, opts=opt | zopt | rvk.OPT_KEEP_WORK)
        assert bool(plan.flags() & rvk.PLAN_MARCH) == (name == "march"), plan.flags()
        plan.solve_host(b)
        out[name] = (plan.work_vector("w"), plan.work_vector("p0"))
        plan.close()
    assert np.array_equal(out["march"][0].view(np.uint64), out["rows"][0].view(np.uint64))
    assert np.array_equal(out["march"][1].view(np.uint64), out["rows"][1].view(np.uint64))


@pytest.mark.parametrize("spec", SPECS, ids=IDS)
@pytest.mark.parametrize("pc", ["jacobi", "none"])
def test_march_solve_vs_oracle(ctx, spec, pc):
    dim, pts, g = spec
    Ah = O.build_laplacian(dim, pts, g)
    b = O.rhs(Ah.n_rows)
    ref = O.cg_solve(Ah, b, max_it=20, pc=pc)
    A = rvk.DeviceCsr.laplacian(ctx, dim, pts, g)
    plan = rvk.CgPlan(ctx, A, max_it=20, pc=pc, opts=rvk.OPT_MARCH)
    assert plan.flags() & rvk.PLAN_MARCH
    x, res = plan.solve_host(b)
    assert res.iterations == 20
    eh = np.max(np.abs(res.hist - ref.hist) / ref.hist)
    ex = np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x)
    assert eh < 1e-10 and ex < 1e-10, (eh, ex)
    # replay is bit-reproducible
    x2, res2 = plan.solve_host(b)
    assert np.array_equal(x, x2) and np.array_equal(res.hist, res2.hist)
    plan.close()


@pytest.mark.parametrize("use_graph", [True, False, "while"])
def test_march_early_exit_and_graph_modes(ctx, use_graph):
    dim, pts, g = 3, 7, (96, 64, 12)
    Ah = O.build_laplacian(dim, pts, g)
    b = O.rhs(Ah.n_rows)
    ref = O.cg_solve(Ah, b, max_it=200, rtol=1e-6)
    assert 3 < ref.iterations < 200
    A = rvk.DeviceCsr.laplacian(ctx, dim, pts, g)
    plan = rvk.CgPlan(ctx, A, max_it=200, rtol=1e-6, opts=rvk.OPT_MARCH, use_graph=use_graph)
    x, res = plan.solve_host(b)
    assert res.iterations == ref.iterations and res.state == ref.status
    assert np.max(np.abs(res.hist - ref.hist) / ref.hist) < 1e-9
    assert np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x) < 1e-9
    plan.close()


def test_march_selection_rules(ctx):
    # opt-in only; 2D grids, small planes, < 3 planes never
    for dim, pts, g, opts, want in [(3, 7, (96, 64, 12), 0, False),
                                    (3, 7, (768, 768, 3), 0, False),
                                    (3, 7, (96, 64, 12), rvk.OPT_MARCH, True),
                                    (2, 5, (4096, 64), rvk.OPT_MARCH, False),   # Q = 4096 < 148 x 32
                                    (3, 7, (90, 64, 12), rvk.OPT_MARCH, True),  # Q = 5760
                                    (3, 7, (95, 64, 12), rvk.OPT_MARCH, True),  # Q = 6080
                                    (3, 7, (95, 63, 12), rvk.OPT_MARCH, False),  # Q % 32 != 0
                                    (3, 7, (96, 64, 2), rvk.OPT_MARCH, False)]:  # < 3 planes
        A = rvk.DeviceCsr.laplacian(ctx, dim, pts, g)
        plan = rvk.CgPlan(ctx, A, max_it=2, opts=opts)
        assert bool(plan.flags() & rvk.PLAN_MARCH) == want, (g, opts)
        plan.close()


@pytest.mark.parametrize("nranks,backend", [(1, "gather"), (2, "peer"), (3, "peer"), (2, "gather"),
                                            (3, "gather"), (4, "peer")])
@pytest.mark.parametrize("pts", [7, 27])
def test_march_row_sharded(ctx, nranks, backend, pts):
    """Row-sharded plans (z-slabs with one halo plane): the march K1 on the
    local CSR (columns shifted by the lower halo), the lower halo plane read
    as global gathers, the boundary planes' p pushed to the neighbours."""
    from paper_2306_17801_b200.sharded import loopback_solve
    g = (96, 64, 3 * nranks + 6)
    Ah = O.build_laplacian(3, pts, g)
    b = O.rhs(Ah.n_rows)
    ref = O.cg_solve(Ah, b, max_it=20)
    flags = []
    x, res, per = loopback_solve(ctx, 3, pts, g, nranks, b, max_it=20, backend=backend,
                                 opts=rvk.OPT_MARCH, flags_out=flags)
    assert all(f & rvk.PLAN_MARCH for f in flags), flags
    x0, res0, _ = loopback_solve(ctx, 3, pts, g, nranks, b, max_it=20, backend=backend,
                                 opts=0)
    assert res.iterations == 20
    eh = np.abs(res.hist - ref.hist) / ref.hist
    ex = np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x)
    assert eh.max() < 1e-10 and ex < 1e-10, (np.argmax(eh > 1e-10), eh.max(), ex,
                                             [np.linalg.norm(x[s] - ref.x[s]) for s in
                                              np.array_split(np.arange(x.size), nranks)])
    assert np.max(np.abs(res.hist - res0.hist) / res0.hist) < 1e-12
