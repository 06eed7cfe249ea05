"""Row-sharded Jacobi-CG across GPUs -- host-side driver.

The global stencil grid is cut into contiguous slabs of planes (z-planes in
3D, y-rows in 2D).  Shard r owns rows [row_begin, row_end); its gathered
vectors (z, p) carry one halo plane on each interior side, and its local CSR
(assembled on the device by ``rvk_build_laplacian_rows``) indexes columns in
that extended space.  The per-iteration exchange is the halo of z and p plus
an allgather of the three dot-product partials, all issued by librvk on the
solve stream (NCCL, or a single-device LOOPBACK that runs every shard on one
GPU for testing).  ``torch.distributed`` is only used to broadcast NCCL's
unique id.

Everything here is plumbing around the C ABI (include/rvk.h); no compute.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import rvk


@dataclass(frozen=True)
class ShardSpec:
    rank: int
    nranks: int
    row_begin: int
    row_end: int
    halo_lo: int      # rows in the lower halo (0 on rank 0)
    halo_hi: int      # rows in the upper halo (0 on the last rank)
    plane: int        # rows per plane (nx*ny in 3D, nx in 2D)

    @property
    def n_own(self) -> int:
        return self.row_end - self.row_begin

    @property
    def col_shift(self) -> int:
        """global column - col_shift = local (extended) column."""
        return self.row_begin - self.halo_lo

    @property
    def n_ext(self) -> int:
        return self.halo_lo + self.n_own + self.halo_hi


def partition(dim: int, grid, nranks: int) -> list[ShardSpec]:
    """Balanced contiguous plane slabs; every shard at least one plane thick
    (a 5/7/9/27-point stencil couples only adjacent planes)."""
    nx, ny, nz = (list(grid) + [1, 1])[:3]
    if dim == 2:
        plane, nplanes = nx, ny
    else:
        plane, nplanes = nx * ny, nz
    if nranks < 1 or nranks > nplanes:
        raise ValueError(f"cannot split {nplanes} planes over {nranks} ranks")
    base, extra = divmod(nplanes, nranks)
    out, p0 = [], 0
    for r in range(nranks):
        cnt = base + (1 if r < extra else 0)
        out.append(ShardSpec(r, nranks, p0 * plane, (p0 + cnt) * plane,
                             plane if r > 0 else 0, plane if r < nranks - 1 else 0, plane))
        p0 += cnt
    return out


def local_laplacian(ctx: "rvk.Ctx", dim: int, points: int, grid, sh: ShardSpec) -> "rvk.DeviceCsr":
    """The shard's rows of the global operator, columns in the extended space."""
    nx, ny, nz = (list(grid) + [1, 1])[:3]
    L = rvk.lib()
    nnz = C.c_int64()
    rvk.check(L.rvk_laplacian_rows_nnz(dim, points, nx, ny, nz, sh.row_begin, sh.row_end,
                                       C.byref(nnz)))
    off = rvk.DeviceArray(sh.n_own + 1, np.int64)
    cols = rvk.DeviceArray(nnz.value, np.int32)
    vals = rvk.DeviceArray(nnz.value, np.float64)
    rvk.check(L.rvk_build_laplacian_rows(ctx.h, dim, points, nx, ny, nz, sh.row_begin, sh.row_end,
                                         sh.col_shift, off.ptr, cols.ptr, vals.ptr))
    return rvk.DeviceCsr(sh.n_own, sh.n_ext, off, cols, vals)


def _cfg(max_it, pc, rtol, atol):
    return rvk.CgConfig(max_it, rvk.PC_JACOBI if pc == "jacobi" else rvk.PC_NONE, rtol, atol,
                        rvk.MODE_FUSED, 0)


class ShardPlan:
    """One shard's distributed CG plan (rvk_dcg_plan)."""

    def __init__(self, ctx, A: "rvk.DeviceCsr", sh: ShardSpec, max_it=20, pc="jacobi", rtol=0.0,
                 atol=0.0, comm=None, shared_gather: int | None = None):
        self.ctx, self.A, self.sh, self.max_it = ctx, A, sh, max_it
        shard = rvk.Shard(sh.n_own, sh.halo_lo, sh.halo_hi, sh.rank, sh.nranks)
        h = C.c_void_p()
        rvk.check(rvk.lib().rvk_dcg_plan_create(ctx.h, C.byref(A.c), shard,
                                                _cfg(max_it, pc, rtol, atol), comm, shared_gather,
                                                C.byref(h)))
        self.h = h
        ctx._deps.add(self)

    def solve_dev(self, b: "rvk.DeviceArray", x: "rvk.DeviceArray"):
        rvk.check(rvk.lib().rvk_dcg_solve_dev(self.h, b.ptr, x.ptr))

    def result(self, raise_breakdown=True) -> "rvk.CgResult":
        hist = np.full(self.max_it + 1, np.nan)
        info = rvk.CgInfo()
        st = rvk.lib().rvk_dcg_result(self.h, hist.ctypes.data, C.byref(info))
        res = rvk.CgResult(hist[: info.iterations + 1].copy(), info.state, info.iterations,
                           info.breakdown_iter)
        if st == rvk.RVK_ERR_BREAKDOWN and not raise_breakdown:
            return res
        if st == rvk.RVK_ERR_BREAKDOWN:
            raise rvk.BreakdownError(st, rvk.lib().rvk_last_error().decode(), info.breakdown_iter)
        rvk.check(st)
        return res

    def close(self):
        if self.h:
            rvk.lib().rvk_dcg_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def loopback_solve(ctx, dim, points, grid, nranks, b_host: np.ndarray, max_it=20, pc="jacobi",
                   rtol=0.0, atol=0.0):
    """All shards on one device (test path): returns (x, CgResult of shard 0,
    per-shard results)."""
    shards = partition(dim, grid, nranks)
    gather = rvk.DeviceArray(4 * nranks)
    rvk.check(rvk.lib().rvk_set(ctx.h, 4 * nranks, 0.0, gather.ptr))
    mats = [local_laplacian(ctx, dim, points, grid, s) for s in shards]
    plans = [ShardPlan(ctx, mats[i], s, max_it, pc, rtol, atol, None,
                       gather.ptr if nranks > 1 else None) for i, s in enumerate(shards)]
    bs = [rvk.DeviceArray.from_host(ctx, b_host[s.row_begin:s.row_end]) for s in shards]
    xs = [rvk.DeviceArray(s.n_own) for s in shards]
    P = (C.c_void_p * nranks)(*[p.h.value for p in plans])
    B = (C.c_void_p * nranks)(*[b.ptr for b in bs])
    X = (C.c_void_p * nranks)(*[x.ptr for x in xs])
    rvk.check(rvk.lib().rvk_dcg_loopback_solve(P, nranks, B, X))
    results = [p.result(raise_breakdown=False) for p in plans]
    x = np.concatenate([xx.download(ctx) for xx in xs])
    for p in plans:
        p.close()
    return x, results[0], results


# ---------------------------------------------------------------------------
# one process per GPU (torchrun)
# ---------------------------------------------------------------------------
def init_comm(rank: int, world: int):
    """NCCL communicator: rank 0 makes the unique id, torch.distributed
    broadcasts it (the only thing torch does on this path)."""
    import torch
    import torch.distributed as dist

    idbuf = (C.c_char * 128)()
    if rank == 0:
        rvk.check(rvk.lib().rvk_comm_unique_id(idbuf, 128))
    t = torch.tensor(list(bytes(idbuf)), dtype=torch.uint8)
    if dist.get_backend() == "nccl":
        t = t.cuda()
    dist.broadcast(t, 0)
    raw = bytes(t.cpu().tolist())
    comm = C.c_void_p()
    rvk.check(rvk.lib().rvk_comm_init(raw, world, rank, C.byref(comm)))
    return comm


def bench_main(args, cfg):
    """bench.py under torchrun: one shard per rank, NCCL halo + allgather."""
    import json
    import statistics
    import sys
    import time

    import torch
    import torch.distributed as dist

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dim, pts, grid, desc = cfg
    weak = args.config != "7pt768"
    if weak:  # every GPU keeps the single-GPU workload: stack slabs along the slowest axis
        grid = tuple(grid[:-1]) + (grid[-1] * world,)
    shards = partition(dim, grid, world)
    sh = shards[rank]
    stream = torch.cuda.Stream()
    ctx = rvk.Ctx(stream.cuda_stream)
    comm = init_comm(rank, world)
    A = local_laplacian(ctx, dim, pts, grid, sh)
    b = rvk.DeviceArray(sh.n_own)
    x = rvk.DeviceArray(sh.n_own)
    # the slice of the global RHS this shard owns
    full_seed = 0x9E3779B97F4A7C15
    rvk.check(rvk.lib().rvk_fill_rhs(ctx.h, (full_seed + sh.row_begin) & (2 ** 64 - 1), sh.n_own,
                                     b.ptr))
    plan = ShardPlan(ctx, A, sh, 20, comm=comm)
    for _ in range(args.warmup):
        plan.solve_dev(b, x)
    plan.result()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    dist.barrier()
    torch.cuda.synchronize()
    syncs0 = rvk.host_syncs()
    for k in range(args.steps):
        ev0[k].record(stream)
        plan.solve_dev(b, x)
        ev1[k].record(stream)
    stream.synchronize()
    syncs = rvk.host_syncs() - syncs0
    dist.barrier()
    ms_local = sum(ev0[k].elapsed_time(ev1[k]) for k in range(args.steps)) / args.steps
    t = torch.tensor([ms_local], device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    res = plan.result()
    n_glob = int(np.prod(grid))
    nnz_glob = _global_nnz(dim, pts, grid)
    b_min = 20 * (12 * nnz_glob + 8 * (n_glob + 1) + 96 * n_glob) + 64 * n_glob
    if rank == 0:
        out = {
            "metric": "20-iter Jacobi-CG solve time, achieved HBM GB/s vs peak, host syncs/iter",
            "value": round(ms, 4), "unit": "ms/solve", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": False,
            "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{desc} row-sharded over {world} GPUs"
                                   + (f" (weak: global grid {grid})" if weak else ""),
                       "n": n_glob, "nnz": nnz_glob, "parallelism": f"rows{world}",
                       "comm": "NCCL halo (1 plane/neighbour, z and p) + allgather of dot partials"},
            "solve_roofline": {"alg_bytes_per_solve": b_min,
                               "achieved_aggregate_gbs": round(b_min / (ms * 1e-3) / 1e9, 1)},
            "host_syncs_per_iter": syncs / (args.steps * 20),
            "iterations": res.iterations,
            "gpu_launches": None,
        }
        print(json.dumps(out), flush=True)
    plan.close()
    rvk.lib().rvk_comm_destroy(comm)
    dist.destroy_process_group()


def _global_nnz(dim, pts, grid):
    nx, ny, nz = (list(grid) + [1, 1])[:3]
    n = C.c_int64()
    nnz = C.c_int64()
    rvk.check(rvk.lib().rvk_laplacian_size(dim, pts, nx, ny, nz, C.byref(n), C.byref(nnz)))
    return nnz.value
