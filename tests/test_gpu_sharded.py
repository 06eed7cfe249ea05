"""Row-sharded CG kernels (rvk_dcg.cu) on one B200 via the LOOPBACK backend:
all P shards live on the device, halos are D2D copies and the dot partials
share one gather buffer -- the same kernels and phase order the NCCL path
runs with one shard per GPU.  Parity vs the CPU oracle at 1e-10."""
import numpy as np
import pytest

import oracle as O
from paper_2306_17801_b200 import rvk
from paper_2306_17801_b200.sharded import loopback_solve, partition, local_laplacian

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dim,pts,grid", [(3, 7, (16, 12, 10)), (3, 27, (9, 8, 12)),
                                          (2, 5, (40, 33)), (2, 9, (17, 24))])
def test_local_csr_matches_global_rows_bitexact(ctx, dim, pts, grid):
    A = O.build_laplacian(dim, pts, grid)
    for sh in partition(dim, grid, 3):
        L = local_laplacian(ctx, dim, pts, grid, sh)
        k0, k1 = A.off[sh.row_begin], A.off[sh.row_end]
        assert np.array_equal(L.off.download(ctx), A.off[sh.row_begin:sh.row_end + 1] - k0)
        assert np.array_equal(L.cols.download(ctx), (A.cols[k0:k1] - sh.col_shift).astype(np.int32))
        assert np.array_equal(L.vals.download(ctx), A.vals[k0:k1])


@pytest.mark.parametrize("backend", ["gather", "peer"])
@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("dim,pts,grid", [(3, 7, (32, 32, 40)), (3, 27, (16, 16, 24)),
                                          (2, 5, (128, 96)), (2, 9, (64, 80))])
def test_loopback_sharded_cg_vs_oracle(ctx, P, dim, pts, grid, backend):
    A = O.build_laplacian(dim, pts, grid)
    b = O.rhs(A.n_rows)
    ref = O.cg_solve(A, b, max_it=20)
    x, res, per = loopback_solve(ctx, dim, pts, grid, P, b, max_it=20, backend=backend)
    assert res.iterations == 20
    for r in per:  # every shard holds the identical scalar history
        assert np.array_equal(r.hist, res.hist)
    assert np.max(np.abs(res.hist - ref.hist) / ref.hist) < 1e-10
    assert np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x) < 1e-10


@pytest.mark.parametrize("backend", ["gather", "peer"])
def test_loopback_rtol_exit_and_single_shard(ctx, backend):
    dim, pts, grid = 2, 5, (48, 48)
    A = O.build_laplacian(dim, pts, grid)
    b = O.rhs(A.n_rows)
    ref = O.cg_solve(A, b, max_it=300, rtol=1e-7)
    for P in (1, 3):
        x, res, _ = loopback_solve(ctx, dim, pts, grid, P, b, max_it=300, rtol=1e-7,
                                   backend=backend)
        assert res.state == rvk.CG_CONVERGED and res.iterations == ref.iterations
        assert np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x) < 1e-10


@pytest.mark.parametrize("P", [2, 5])
def test_peer_loopback_bitwise_equals_gather_backend_and_resolves(ctx, P):
    """The PEER kernels (in-kernel halo pushes, partial broadcast, flag
    waits) produce exactly the gather backend's numbers -- same reduction
    order -- and stay correct over repeated solves on the same plans (solve
    counter + finish->setup barrier of the flag protocol)."""
    dim, pts, grid = 3, 7, (24, 20, 30)
    A = O.build_laplacian(dim, pts, grid)
    b = O.rhs(A.n_rows)
    xg, rg, _ = loopback_solve(ctx, dim, pts, grid, P, b, max_it=20, backend="gather")
    xp, rp, per = loopback_solve(ctx, dim, pts, grid, P, b, max_it=20, backend="peer", repeats=3)
    assert np.array_equal(rp.hist, rg.hist)
    assert np.array_equal(xp, xg)
    assert all(r.state == rvk.CG_RUNNING and r.iterations == 20 for r in per)


def test_peer_loopback_early_exit_then_resolve(ctx):
    """Converged early (kernels skip their signals), then solved again: the
    finish kernel still releases every rank, so the next setup proceeds."""
    dim, pts, grid = 2, 5, (40, 36)
    A = O.build_laplacian(dim, pts, grid)
    b = O.rhs(A.n_rows)
    ref = O.cg_solve(A, b, max_it=400, rtol=1e-6)
    x, res, per = loopback_solve(ctx, dim, pts, grid, 4, b, max_it=400, rtol=1e-6,
                                 backend="peer", repeats=2)
    assert res.state == rvk.CG_CONVERGED and res.iterations == ref.iterations
    assert all(r.iterations == res.iterations for r in per)
    assert np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x) < 1e-10


@pytest.mark.parametrize("backend", ["gather", "peer"])
def test_loopback_headline_256cubed_4_shards(ctx, backend):
    A = O.build_laplacian(3, 7, (256, 256, 256))
    b = O.rhs(A.n_rows)
    ref = O.cg_solve(A, b, max_it=20)
    x, res, _ = loopback_solve(ctx, 3, 7, (256, 256, 256), 4, b, max_it=20, backend=backend)
    assert np.max(np.abs(res.hist - ref.hist) / ref.hist) < 1e-10
    assert np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x) < 1e-10


@pytest.mark.parametrize("backend", ["gather", "peer"])
def test_loopback_zero_rhs_writes_x(ctx, backend):
    """The shard plans skip the x = 0 store of the setup (the whole-solve x
    pass starts from 0.0): a zero right-hand side converges at the setup and
    x must still come back all zeros on every shard."""
    dim, pts, grid = 3, 7, (24, 20, 30)
    n = grid[0] * grid[1] * grid[2]
    x, res, per = loopback_solve(ctx, dim, pts, grid, 2, np.zeros(n), max_it=20, backend=backend)
    assert res.iterations == 0
    assert not np.any(x) and np.all(np.isfinite(x))
