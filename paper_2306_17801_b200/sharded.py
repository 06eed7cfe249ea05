"""Row-sharded Jacobi-CG across GPUs -- host-side driver.

The global stencil grid is cut into contiguous slabs of planes (z-planes in
3D, y-rows in 2D).  Shard r owns rows [row_begin, row_end); its gathered
vectors (z, p) carry one halo plane on each interior side, and its local CSR
(assembled on the device by ``rvk_build_laplacian_rows``) indexes columns in
that extended space.  The per-iteration exchange is the halo of z and p plus
the three dot-product partials, all on the solve stream:

* ``peer`` (default across GPUs): the kernels themselves store the halo
  planes and partials into the neighbours' windows over NVLink and sync on
  device flags (rvk_dcg_attach_peers) -- windows are shared with cudaIpc;
* ``nccl``: ncclSend/Recv halos + ncclAllGather of partials between kernels;
* loopback variants of both run every shard on ONE GPU for testing.

``torch.distributed`` only moves setup bytes (NCCL id, cudaIpc handles).

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


def _cfg(max_it, pc, rtol, atol, opts=0):
    return rvk.CgConfig(max_it, rvk.PC_JACOBI if pc == "jacobi" else rvk.PC_NONE, rtol, atol,
                        rvk.MODE_FUSED, 0, opts)


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

    def window(self) -> tuple[int, int]:
        base, nbytes = C.c_void_p(), C.c_size_t()
        rvk.check(rvk.lib().rvk_dcg_window(self.h, C.byref(base), C.byref(nbytes)))
        return base.value, nbytes.value

    def attach_peers(self, windows: list[int], shards: list[ShardSpec]):
        """PEER backend: windows[q] = rank q's window as mapped on this device."""
        n = len(shards)
        W = (C.c_void_p * n)(*windows)
        S = (rvk.Shard * n)(*[rvk.Shard(s.n_own, s.halo_lo, s.halo_hi, s.rank, s.nranks)
                              for s in shards])
        rvk.check(rvk.lib().rvk_dcg_attach_peers(self.h, W, S))

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
                   rtol=0.0, atol=0.0, backend="gather", repeats=1):
    """All shards on one device (test path): returns (x, CgResult of shard 0,
    per-shard results).  backend "gather": D2D halo copies + one shared
    gather buffer between kernels; "peer": the PEER kernels (in-kernel halo
    pushes, partial broadcast, flag protocol) with every window on this GPU.
    `repeats` > 1 re-solves on the same plans (exercises the solve counter
    and the finish -> setup barrier of the flag protocol)."""
    shards = partition(dim, grid, nranks)
    peer = backend == "peer"
    gather = None
    if not peer:
        gather = rvk.DeviceArray(4 * nranks)
        rvk.check(rvk.lib().rvk_set(ctx.h, 4 * nranks, 0.0, gather.ptr))
    mats = [local_laplacian(ctx, dim, points, grid, s) for s in shards]
    plans = [ShardPlan(ctx, mats[i], s, max_it, pc, rtol, atol, None,
                       gather.ptr if (gather is not None and nranks > 1) else None)
             for i, s in enumerate(shards)]
    if peer:
        windows = [p.window()[0] for p in plans]
        for p in plans:
            p.attach_peers(windows, shards)
    bs = [rvk.DeviceArray.from_host(ctx, b_host[s.row_begin:s.row_end]) for s in shards]
    xs = [rvk.DeviceArray(s.n_own) for s in shards]
    P = (C.c_void_p * nranks)(*[p.h.value for p in plans])
    B = (C.c_void_p * nranks)(*[b.ptr for b in bs])
    X = (C.c_void_p * nranks)(*[x.ptr for x in xs])
    for _ in range(repeats):
        rvk.check(rvk.lib().rvk_dcg_loopback_solve(P, nranks, B, X))
    results = [p.result(raise_breakdown=False) for p in plans]
    x = np.concatenate([xx.download(ctx) for xx in xs])
    for p in plans:
        p.close()
    return x, results[0], results


# ---------------------------------------------------------------------------
# one process per GPU (torchrun)
# ---------------------------------------------------------------------------
def connect_peers(plan: ShardPlan, shards: list[ShardSpec], rank: int, world: int) -> list[int]:
    """PEER backend across processes: exchange cudaIpc handles of every
    rank's window (torch.distributed all_gather_object), map the peers'
    windows on this device, attach.  Returns the mapped pointers (close with
    disconnect_peers after a barrier)."""
    import torch.distributed as dist

    base, _ = plan.window()
    h = (C.c_char * 64)()
    rvk.check(rvk.lib().rvk_ipc_get_handle(base, h, 64))
    handles = [None] * world
    dist.all_gather_object(handles, bytes(h))
    windows, opened = [], []
    for q in range(world):
        if q == rank:
            windows.append(base)
            continue
        p = C.c_void_p()
        rvk.check(rvk.lib().rvk_ipc_open_handle(handles[q], C.byref(p)))
        windows.append(p.value)
        opened.append(p.value)
    plan.attach_peers(windows, shards)
    dist.barrier()  # every rank attached (flags zeroed) before anyone solves
    return opened


def disconnect_peers(opened: list[int]):
    for p in opened:
        rvk.lib().rvk_ipc_close_handle(p)


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
    """bench.py under torchrun: one shard per rank.  Backend PEER (in-kernel
    NVLink halo pushes + partial broadcast, no NCCL on the data path) unless
    --comm nccl, or unless the PEER setup fails / its first solve differs
    from the NCCL solve bit for bit (then NCCL, with the reason in the JSON)."""
    import json
    import sys

    import torch
    import torch.distributed as dist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import ClockSampler, peaks  # noqa: E402  (bench.py is the caller)

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    # RVK_SHARED_GPU=1 (functional check on a 1-GPU box): every rank on GPU 0,
    # gloo bootstrap, PEER only (NCCL refuses two ranks on one device);
    # contexts time-slice, so the timings are meaningless -- the JSON says so
    shared = os.environ.get("RVK_SHARED_GPU") == "1"
    if shared or torch.cuda.device_count() == 1:
        local = 0  # (a launcher that pins one visible GPU per process)
    torch.cuda.set_device(local)
    if shared:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    tdev = "cpu" if shared else f"cuda:{local}"
    dim, pts, grid, desc = cfg
    weak = args.config != "7pt768"
    if weak:  # every GPU keeps the single-GPU workload: stack slabs along the slowest axis
        grid = tuple(grid[:-1]) + (grid[-1] * world,)
    shards = partition(dim, grid, world)
    sh = shards[rank]
    stream = torch.cuda.Stream()
    ctx = rvk.Ctx(stream.cuda_stream)
    comm, comm_err = None, None
    if not shared:
        try:
            comm = init_comm(rank, world)
        except Exception as e:  # noqa: BLE001 -- PEER needs no NCCL; report it
            comm_err = f"NCCL unavailable: {e}".splitlines()[0][:200]
    A = local_laplacian(ctx, dim, pts, grid, sh)
    b = rvk.DeviceArray(sh.n_own)
    x = rvk.DeviceArray(sh.n_own)
    # the slice of the global RHS this shard owns
    full_seed = 0x9E3779B97F4A7C15
    rvk.check(rvk.lib().rvk_fill_rhs(ctx.h, (full_seed + sh.row_begin) & (2 ** 64 - 1), sh.n_own,
                                     b.ptr))
    nccl_plan = ref_hist = ref_x = None
    if comm is not None:
        nccl_plan = ShardPlan(ctx, A, sh, 20, comm=comm)
        nccl_plan.solve_dev(b, x)
        ref_hist = nccl_plan.result().hist
        ref_x = x.download(ctx)

    backend, fallback, opened, plan = "nccl", comm_err, [], nccl_plan
    if comm is None or getattr(args, "comm", "peer") == "peer":
        try:
            peer_plan = ShardPlan(ctx, A, sh, 20)
            opened = connect_peers(peer_plan, shards, rank, world)
            peer_plan.solve_dev(b, x)
            ph = peer_plan.result().hist
            ok = nccl_plan is None or (np.array_equal(ph, ref_hist) and
                                       np.array_equal(x.download(ctx), ref_x))
            err = None if ok else "PEER solve differs from the NCCL solve"
        except Exception as e:  # noqa: BLE001 -- report and fall back, never hang
            err, peer_plan = f"PEER setup failed: {e}".splitlines()[0][:200], None
        if nccl_plan is None and err is not None:
            raise RuntimeError(err)  # no backend left
        flags = torch.tensor([0 if err is None else 1], device=tdev)
        dist.all_reduce(flags)  # every rank takes the same backend
        if int(flags.item()) == 0:
            backend, plan = "peer", peer_plan
        else:
            fallback = err or "another rank's PEER check failed"
    for _ in range(args.warmup):
        plan.solve_dev(b, x)
    plan.result()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    dist.barrier()
    torch.cuda.synchronize()
    syncs0 = rvk.host_syncs()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            ev0[k].record(stream)
            plan.solve_dev(b, x)
            ev1[k].record(stream)
        stream.synchronize()
    syncs = rvk.host_syncs() - syncs0
    dist.barrier()
    ms_local = sum(ev0[k].elapsed_time(ev1[k]) for k in range(args.steps)) / args.steps
    t = torch.tensor([ms_local], device=tdev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    res = plan.result()

    # ---- e2e: pinned host b shard -> device, solve, x shard -> host (events) --
    bh = torch.empty(sh.n_own, dtype=torch.float64, pin_memory=True)
    xh = torch.empty(sh.n_own, dtype=torch.float64, pin_memory=True)
    bh.numpy()[:] = b.download(ctx)
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    L = rvk.lib()
    dist.barrier()
    for k in range(args.steps):
        e0[k].record(stream)
        rvk.check(L.rvk_memcpy_h2d(ctx.h, b.ptr, bh.data_ptr(), 8 * sh.n_own))
        plan.solve_dev(b, x)
        rvk.check(L.rvk_memcpy_d2h(ctx.h, xh.data_ptr(), x.ptr, 8 * sh.n_own))
        e1[k].record(stream)
    stream.synchronize()
    e2e_local = sum(e0[k].elapsed_time(e1[k]) for k in range(args.steps)) / args.steps
    t = torch.tensor([e2e_local], device=tdev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())
    plan.result()

    n_glob = int(np.prod(grid))
    nnz_glob = _global_nnz(dim, pts, grid)
    fl = rvk.lib().rvk_dcg_plan_flags(plan.h)
    ob = 4 if fl & 8 else 8               # int32 row offsets streamed
    # per-iteration vector bytes: 96 n, x traffic 24 n -> 8 n + 16 n / group
    # (pairs: 16 n; whole solve, RVK_PLAN_X_SOLVE: 8.8 n), constant
    # Jacobi diagonal (RVK_PLAN_CONST_DIAG) -8 n per iteration and setup
    grp = 20 if fl & 128 else (2 if fl & 16 else 1)
    vb = 96 - (16 - 16 / grp) - (8 if fl & 1 else 0)
    b_min = int(20 * (12 * nnz_glob + ob * (n_glob + 1) + vb * n_glob) + (56 if fl & 1 else 64) * n_glob)
    hbm_peak, peak_src = peaks()
    per_gpu = b_min / world / (ms * 1e-3) / 1e9
    launches = 3 + 2 * 20 + (1 if fl & 16 else 0)  # reset, setup, 20 x (K1, K2), finish, x-fix
    if rank == 0:
        comm_desc = {"peer": "PEER: K1/K2 store halo planes + dot partials into the neighbours' "
                             "windows over NVLink (cudaIpc), device flag sync; no NCCL on the "
                             "data path",
                     "nccl": "NCCL halo (ncclSend/Recv, 1 plane/neighbour, z and p) + "
                             "ncclAllGather of dot partials between kernels"}[backend]
        out = {
            "metric": "20-iter Jacobi-CG solve time, achieved HBM GB/s vs peak, host syncs/iter",
            "value": round(ms, 4), "unit": "ms/solve", "n_gpus": 1 if shared else world,
            "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": False,
            "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{desc} row-sharded over {world} GPUs"
                                   + (f" (weak: global grid {grid})" if weak else ""),
                       "n": n_glob, "nnz": nnz_glob, "parallelism": f"rows{world}",
                       "comm": comm_desc, "comm_fallback": fallback,
                       "shared_gpu_functional_check": shared,
                       "l2": "no flush: per-GPU working set >> 126 MB L2"},
            "roofline": {"bound": "hbm", "kernel": "whole sharded solve, per GPU (K1+K2+comm)",
                         "achieved": round(per_gpu, 1), "peak": hbm_peak, "unit": "GB/s",
                         "frac": round(per_gpu / hbm_peak, 4), "traffic": None,
                         "peak_source": peak_src},
            "solve_roofline": {"alg_bytes_per_solve": b_min,
                               "achieved_aggregate_gbs": round(b_min / (ms * 1e-3) / 1e9, 1)},
            "host_syncs_per_iter": syncs / (args.steps * 20),
            "iterations": res.iterations,
            "iters_per_s": round(res.iterations / (ms * 1e-3), 1),
            "e2e": {"value": round(e2e_ms, 4), "unit": "ms/solve",
                    "h2d_bytes_per_step": 8 * n_glob, "d2h_bytes_per_step": 8 * n_glob},
            "gpu_launches": launches * args.steps * world,
            "cpu_baseline": None,
            "clocks": clk.summary(),
        }
        print(json.dumps(out), flush=True)
    dist.barrier()  # no rank frees a window a peer may still store into
    plan.close()
    if nccl_plan is not None and plan is not nccl_plan:
        nccl_plan.close()
    disconnect_peers(opened)
    if comm is not None:
        rvk.lib().rvk_comm_destroy(comm)
    dist.destroy_process_group()


def _global_nnz(dim, pts, grid):
    nx, ny, nz = (list(grid) + [1, 1])[:3]
    n = C.c_int64()
    nnz = C.c_int64()
    rvk.check(rvk.lib().rvk_laplacian_size(dim, pts, nx, ny, nz, C.byref(n), C.byref(nnz)))
    return nnz.value
