"""CPU tests of the row-sharded CG design: the partition,
the local-CSR column remap and the per-iteration dataflow of rvk_dcg.cu
(halo exchange of z and p, allgather of the dot partials, scalar tails
deferred to the next kernel's prologue) replayed in numpy over a real
world_size-2/3 torch.distributed gloo group, checked against the oracle."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2306_17801_b200.sharded import partition


def local_rows(A: O.Csr, sh):
    """Rows [row_begin, row_end) of the global CSR with columns remapped to the
    shard's extended [lo halo | owned | hi halo] index space."""
    k0, k1 = A.off[sh.row_begin], A.off[sh.row_end]
    off = A.off[sh.row_begin:sh.row_end + 1] - k0
    cols = A.cols[k0:k1].astype(np.int64) - sh.col_shift
    return O.Csr(sh.n_own, sh.n_ext, off.astype(np.int64), cols.astype(np.int32), A.vals[k0:k1].copy())


@pytest.mark.parametrize("dim,pts,grid,P", [(3, 7, (6, 5, 7), 3), (3, 27, (4, 4, 9), 4),
                                            (2, 5, (9, 11), 2), (2, 9, (7, 5), 5)])
def test_partition_covers_operator(dim, pts, grid, P):
    A = O.build_laplacian(dim, pts, grid)
    shards = partition(dim, grid, P)
    assert shards[0].row_begin == 0 and shards[-1].row_end == A.n_rows
    for a, b in zip(shards, shards[1:]):
        assert a.row_end == b.row_begin
    x = np.random.default_rng(0).standard_normal(A.n_rows)
    y = O.spmv(A, x)
    for sh in shards:
        L = local_rows(A, sh)
        assert L.cols.min() >= 0 and L.cols.max() < sh.n_ext   # one halo plane suffices
        xe = x[sh.col_shift:sh.col_shift + sh.n_ext]
        assert np.array_equal(O.spmv(L, xe), y[sh.row_begin:sh.row_end])  # bit-exact per row


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, dim, pts, grid, max_it, rtol, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    A = O.build_laplacian(dim, pts, grid)
    sh = partition(dim, grid, world)[rank]
    L = local_rows(A, sh)
    b = O.rhs(A.n_rows)[sh.row_begin:sh.row_end]
    dinv = 1.0 / O.diagonal(A)[sh.row_begin:sh.row_end]
    n, lo = sh.n_own, sh.halo_lo
    own = slice(lo, lo + n)
    z = np.zeros(sh.n_ext)
    p = [np.zeros(sh.n_ext), np.zeros(sh.n_ext)]
    x = np.zeros(n)

    def allgather(vals):
        t = torch.tensor(vals, dtype=torch.float64)
        out = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return np.array([o.numpy() for o in out])

    def halo(v):
        pl = sh.plane
        reqs = []
        if rank > 0:
            reqs.append(dist.isend(torch.from_numpy(v[lo:lo + pl].copy()), rank - 1))
        if rank < world - 1:
            reqs.append(dist.isend(torch.from_numpy(v[lo + n - pl:lo + n].copy()), rank + 1))
        if rank > 0:
            t = torch.zeros(pl, dtype=torch.float64)
            dist.recv(t, rank - 1)
            v[:lo] = t.numpy()
        if rank < world - 1:
            t = torch.zeros(pl, dtype=torch.float64)
            dist.recv(t, rank + 1)
            v[lo + n:] = t.numpy()
        for r in reqs:
            r.wait()

    # K0
    r = b.copy()
    z[own] = dinv * r
    g = allgather([z[own] @ z[own], z[own] @ r])
    hist, beta, state, its, dp0 = [], [], "running", 0, None
    for it in range(max_it + 1):
        # prologue of K1(it) (or the finish kernel): fold, hist, convergence
        zz, zr = g[:, 0].sum(), g[:, 1].sum()
        dp = np.sqrt(zz)
        dp0 = dp if it == 0 else dp0
        hist.append(dp)
        beta.append(zr)
        its = it
        if dp <= max(rtol * dp0, 0.0):
            state = "converged"
            break
        if it == max_it:
            break
        halo(z)
        if it > 0:
            halo(p[it & 1])
        bb = 0.0 if it == 0 else beta[it] / beta[it - 1]
        pe = z + bb * p[it & 1] if it > 0 else z.copy()
        pn = p[(it + 1) & 1]
        pn[own] = pe[own]
        w = O.spmv(L, pe)
        g = allgather([pn[own] @ w])
        pAp = g[:, 0].sum()
        a = beta[it] / pAp
        x += a * pn[own]
        r += -a * w
        z[own] = dinv * r
        g = allgather([z[own] @ z[own], z[own] @ r])
    q.put((rank, np.array(hist), its, state, sh.row_begin, x))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,dim,pts,grid,max_it,rtol", [
    (2, 3, 7, (8, 8, 8), 20, 0.0),
    (3, 3, 27, (6, 6, 7), 20, 0.0),
    (2, 2, 5, (16, 16), 200, 1e-6),
])
def test_sharded_dataflow_matches_oracle_gloo(world, dim, pts, grid, max_it, rtol):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dim, pts, grid, max_it, rtol, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    A = O.build_laplacian(dim, pts, grid)
    ref = O.cg_solve(A, O.rhs(A.n_rows), max_it=max_it, rtol=rtol)
    x = np.concatenate([t[5] for t in res])
    for t in res:  # every rank holds identical scalars
        assert np.array_equal(t[1], res[0][1]) and t[2] == res[0][2]
    assert res[0][2] == ref.iterations
    assert np.max(np.abs(res[0][1] - ref.hist) / ref.hist) < 1e-10
    assert np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x) < 1e-10
