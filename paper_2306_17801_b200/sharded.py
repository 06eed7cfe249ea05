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
    """One shard's distributed CG plan (rvk_dcg_plan).  use_graph: the solve
    is captured into a CUDA graph on first use (per b / x pair) and replayed
    (rvk_dcg_solve_dev; loopback plans are solved phase by phase instead)."""

    def __init__(self, ctx, A: "rvk.DeviceCsr", sh: ShardSpec, max_it=20, pc="jacobi", rtol=0.0,
                 atol=0.0, comm=None, shared_gather: int | None = None, use_graph: bool = False,
                 opts: int = 0):
        self.ctx, self.A, self.sh, self.max_it = ctx, A, sh, max_it
        shard = rvk.Shard(sh.n_own, sh.halo_lo, sh.halo_hi, sh.rank, sh.nranks)
        cfg = _cfg(max_it, pc, rtol, atol, opts)
        cfg.use_graph = 1 if use_graph else 0
        h = C.c_void_p()
        rvk.check(rvk.lib().rvk_dcg_plan_create(ctx.h, C.byref(A.c), shard, cfg, comm,
                                                shared_gather, C.byref(h)))
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
                   rtol=0.0, atol=0.0, backend="gather", repeats=1, opts=0, flags_out=None):
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
                       gather.ptr if (gather is not None and nranks > 1) else None, opts=opts)
             for i, s in enumerate(shards)]
    if flags_out is not None:
        flags_out.extend(int(rvk.lib().rvk_dcg_plan_flags(p.h)) for p in plans)
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
    broadcasts it (the only thing torch does on this path).  The
    communicator's own view (ncclCommCount / ncclCommUserRank) is logged and
    checked against the launcher's."""
    import sys

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
    nr, rk = C.c_int(), C.c_int()
    rvk.check(rvk.lib().rvk_comm_size(comm, C.byref(nr), C.byref(rk)))
    print(f"[rvk] NCCL communicator: rank {rk.value} of {nr.value} (launcher: {rank} of {world})",
          file=sys.stderr, flush=True)
    if (nr.value, rk.value) != (world, rank):
        raise RuntimeError(f"NCCL communicator reports rank {rk.value}/{nr.value}, "
                           f"launcher {rank}/{world}")
    return comm


def _build_shard(ctx, dim, pts, grid, shards, rank, seed=0x9E3779B97F4A7C15):
    """The shard's local CSR (device assembly) and its slice of the global RHS."""
    sh = shards[rank]
    A = local_laplacian(ctx, dim, pts, grid, sh)
    b = rvk.DeviceArray(sh.n_own)
    x = rvk.DeviceArray(sh.n_own)
    rvk.check(rvk.lib().rvk_fill_rhs(ctx.h, (seed + sh.row_begin) & (2 ** 64 - 1), sh.n_own, b.ptr))
    return sh, A, b, x


def _time_sharded(plan, b, x, stream, steps, warmup, tdev, local):
    """K solves timed by CUDA events on every rank's solve stream, a barrier
    and a device sync on both sides; returns (max-over-ranks ms, clocks,
    host syncs on this rank)."""
    import torch
    import torch.distributed as dist

    import bench
    for _ in range(warmup):
        plan.solve_dev(b, x)
    plan.result()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    dist.barrier()
    torch.cuda.synchronize()
    syncs0 = rvk.host_syncs()
    with bench.ClockSampler(local) as clk:
        for k in range(steps):
            ev0[k].record(stream)
            plan.solve_dev(b, x)
            ev1[k].record(stream)
        stream.synchronize()
    syncs = rvk.host_syncs() - syncs0
    dist.barrier()
    ms_local = sum(ev0[k].elapsed_time(ev1[k]) for k in range(steps)) / steps
    t = torch.tensor([ms_local], device=tdev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()), clk.summary(), syncs


def _peer_or_nccl(args, ctx, A, sh, shards, b, x, comm, rank, world, tdev):
    """The product backend is PEER (in-kernel NVLink halo / partial stores);
    it is used only if its first solve equals the NCCL solve bit for bit on
    every rank (same arithmetic and fold order by construction).  Returns
    (backend, plan, other_plan, opened handles, fallback reason)."""
    import numpy as _np
    import torch
    import torch.distributed as dist

    nccl_plan = ref_hist = ref_x = None
    if comm is not None:
        nccl_plan = ShardPlan(ctx, A, sh, 20, comm=comm, use_graph=True)
        nccl_plan.solve_dev(b, x)
        ref_hist = nccl_plan.result().hist
        ref_x = x.download(ctx)
    backend, fallback, opened, plan = "nccl", None, [], nccl_plan
    if comm is None or getattr(args, "comm", "peer") == "peer":
        peer_plan = None
        try:
            peer_plan = ShardPlan(ctx, A, sh, 20, use_graph=True)
            opened = connect_peers(peer_plan, shards, rank, world)
            peer_plan.solve_dev(b, x)
            ph = peer_plan.result().hist
            ok = nccl_plan is None or (_np.array_equal(ph, ref_hist) and
                                       _np.array_equal(x.download(ctx), ref_x))
            err = None if ok else "PEER solve differs from the NCCL solve"
        except Exception as e:  # noqa: BLE001 -- report and fall back, never hang
            err, peer_plan = f"PEER setup failed: {e}".splitlines()[0][:200], None
        if nccl_plan is None and err is not None:
            raise RuntimeError(err)  # no backend left
        flags = torch.tensor([0 if err is None else 1], device=tdev)
        dist.all_reduce(flags)  # every rank takes the same backend
        if int(flags.item()) == 0:
            backend, plan = "peer", peer_plan
            if nccl_plan is not None:
                nccl_plan.close()
                nccl_plan = None
        else:
            fallback = err or "another rank's PEER check failed"
            if peer_plan is not None:
                peer_plan.close()
    return backend, plan, opened, fallback, nccl_plan is not None or backend == "nccl"


def _check_vs_single_gpu(ctx, dim, pts, grid, hist, x_shard, sh, rank, tdev):
    """Rank 0 solves the same GLOBAL system with the single-GPU plan (when it
    fits) and every rank compares: the history (identical on all ranks) and
    ||x||^2 summed over the shards, within 1e-10 (reduction trees differ
    between the 1-GPU and the P-shard solve, so not bitwise)."""
    import numpy as _np
    import torch
    import torch.distributed as dist

    n_glob = int(_np.prod(grid))
    res = torch.zeros(3, dtype=torch.float64, device=tdev)  # ok, hist err, x err
    xx = torch.tensor([float(_np.dot(x_shard, x_shard))], dtype=torch.float64, device=tdev)
    dist.all_reduce(xx)
    if rank == 0:
        if n_glob <= (1 << 28):
            A = rvk.DeviceCsr.laplacian(ctx, dim, pts, grid)
            b = rvk.DeviceArray(n_glob)
            x = rvk.DeviceArray(n_glob)
            rvk.check(rvk.lib().rvk_fill_rhs(ctx.h, 0x9E3779B97F4A7C15, n_glob, b.ptr))
            p1 = rvk.CgPlan(ctx, A, max_it=20)
            p1.solve_dev(b, x)
            r1 = p1.result()
            x1 = x.download(ctx)
            p1.close()
            del A, b, x
            eh = float(_np.max(_np.abs(r1.hist - hist) / _np.abs(r1.hist)))
            ex = abs(float(_np.dot(x1, x1)) - float(xx.item())) / float(_np.dot(x1, x1))
            res[:] = torch.tensor([1.0, eh, ex], dtype=torch.float64)
    dist.broadcast(res, 0)
    if res[0].item() == 0.0:
        return {"checked": False, "reason": f"global system of {n_glob} rows not solved on one GPU"}
    eh, ex = float(res[1].item()), float(res[2].item())
    return {"checked": True, "vs": "single-GPU plan, same global system", "hist_rel_err": eh,
            "x_norm2_rel_err": ex, "ok": bool(eh < 1e-10 and ex < 1e-10)}


def bench_main(args, cfg):
    """bench.py under torchrun: one shard per rank.

    value: the weak-scaled workload (each GPU keeps one config-sized slab, the
    global grid grows along the slowest axis), so it stays comparable with
    the N = 1 line.  strong_768: BASELINE.json configs[4] -- the fixed 768^3
    grid row-sharded over the N GPUs -- measured in the same invocation.
    Backend PEER (in-kernel NVLink halo pushes + partial broadcast, no NCCL
    on the data path) unless --comm nccl, or unless the PEER setup fails / its
    first solve differs from the NCCL solve bit for bit (then NCCL, with the
    reason in the JSON).  Every solve is one replayed CUDA graph."""
    import json
    import sys

    import torch
    import torch.distributed as dist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench  # noqa: E402  (bench.py is the caller)

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
    dim, pts, grid, desc, strong_cfg = bench.workload(args, world)
    shards = partition(dim, grid, world)
    stream = torch.cuda.Stream()
    ctx = rvk.Ctx(stream.cuda_stream)
    comm, comm_err = None, None
    if not shared:
        try:
            comm = init_comm(rank, world)
        except Exception as e:  # noqa: BLE001 -- PEER needs no NCCL; report it
            comm_err = f"NCCL unavailable: {e}".splitlines()[0][:200]
    sh, A, b, x = _build_shard(ctx, dim, pts, grid, shards, rank)
    backend, plan, opened, fallback, _ = _peer_or_nccl(args, ctx, A, sh, shards, b, x, comm, rank,
                                                        world, tdev)
    fallback = fallback or comm_err
    ms, clocks, syncs = _time_sharded(plan, b, x, stream, args.steps, args.warmup, tdev, local)
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
    res = plan.result()
    x_own = x.download(ctx)
    fl = rvk.lib().rvk_dcg_plan_flags(plan.h)
    dist.barrier()  # no rank frees a window a peer may still store into
    plan.close()
    disconnect_peers(opened)
    del A, b, x

    # ---- correctness of this run: vs the single-GPU solve of the same system --
    check = _check_vs_single_gpu(ctx, dim, pts, grid, res.hist, x_own, sh, rank, tdev)

    # ---- BASELINE configs[4]: 768^3 row-sharded over the N GPUs ---------------
    strong = None
    if not strong_cfg and not getattr(args, "no_strong", False):
        strong = _strong_768(args, ctx, stream, comm, rank, world, tdev, local)

    n_glob = int(np.prod(grid))
    nnz_glob = _global_nnz(dim, pts, grid)
    b_min = _shard_bytes(n_glob, nnz_glob, fl)
    hbm_peak, peak_src = bench.peaks()
    per_gpu = b_min / world / (ms * 1e-3) / 1e9
    launches = 3 + 2 * 20 + (1 if fl & 16 else 0)  # reset, setup, 20 x (K1, K2), finish, x-fix
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = bench.cpu_baseline_entry(dim, pts, grid)
    traffic, traffic_src = bench.ncu_traffic(args.config + "_shard", "solve")
    if rank == 0:
        comm_desc = {"peer": "PEER: K1/K2 store halo planes + dot partials into the neighbours' "
                             "windows over NVLink (cudaIpc), device flag sync; no NCCL on the "
                             "data path",
                     "nccl": "NCCL halo (ncclSend/Recv, 1 plane/neighbour, z and p) + "
                             "ncclAllGather of dot partials between kernels"}[backend]
        out = {
            "metric": bench.METRIC,
            "value": round(ms, 4), "unit": "ms/solve", "n_gpus": 1 if shared else world,
            "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": False,
            "scaling": bench.scaling_label(args), "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": bench.bench_config(args, world),
            "run": {"comm": comm_desc, "comm_fallback": fallback, "graph": True,
                    "shared_gpu_functional_check": shared,
                    "l2": "no flush: per-GPU working set >> 126 MB L2"},
            "roofline": {"bound": "hbm", "kernel": "whole sharded solve, per GPU (K1+K2+comm)",
                         "achieved": round(per_gpu, 1), "peak": hbm_peak, "unit": "GB/s",
                         "frac": round(per_gpu / hbm_peak, 4), "traffic": traffic,
                         "traffic_source": traffic_src, "peak_source": peak_src,
                         "alg_bytes_per_solve_per_gpu": b_min // world},
            "solve_roofline": {"alg_bytes_per_solve": b_min,
                               "achieved_aggregate_gbs": round(b_min / (ms * 1e-3) / 1e9, 1)},
            "host_syncs_per_iter": syncs / (args.steps * 20),
            "iterations": res.iterations,
            "iters_per_s": round(res.iterations / (ms * 1e-3), 1),
            "e2e": {"value": round(e2e_ms, 4), "unit": "ms/solve",
                    "h2d_bytes_per_step": 8 * n_glob, "d2h_bytes_per_step": 8 * n_glob},
            "gpu_launches": launches * args.steps * world,
            "check": check,
            "strong_768": strong,
            "cpu_baseline": cpu,
            "clocks": clocks,
        }
        print(json.dumps(out), flush=True)
    dist.barrier()
    if comm is not None:
        rvk.lib().rvk_comm_destroy(comm)
    dist.destroy_process_group()


def _shard_bytes(n_glob, nnz_glob, fl):
    """Algorithmic bytes of one sharded solve (all ranks): per iteration
    12 nnz + 8 (n+1) + 96 n with the x traffic cut by the x group (whole
    solve, RVK_PLAN_X_SOLVE: 8.4 n; pairs: 16 n) and the constant Jacobi
    diagonal (RVK_PLAN_CONST_DIAG: -8 n per iteration and in the setup)."""
    grp = 20 if fl & 128 else (2 if fl & 16 else 1)
    vb = 96 - (16 - 16 / grp) - (8 if fl & 1 else 0)
    return int(20 * (12 * nnz_glob + 8 * (n_glob + 1) + vb * n_glob) + (56 if fl & 1 else 64) * n_glob)


def _strong_768(args, ctx, stream, comm, rank, world, tdev, local):
    """768^3 7-point row-sharded over the N GPUs, same backend selection as
    the main run; ms/solve max over ranks, iterations/s, per-GPU GB/s."""
    import bench
    g = bench.CONFIGS["7pt768"][2]
    shards = partition(3, g, world)
    sh, A, b, x = _build_shard(ctx, 3, 7, g, shards, rank)
    backend, plan, opened, fallback, _ = _peer_or_nccl(args, ctx, A, sh, shards, b, x, comm, rank,
                                                        world, tdev)
    steps = max(3, min(args.steps, 10))
    ms, clocks, syncs = _time_sharded(plan, b, x, stream, steps, 3, tdev, local)
    res = plan.result()
    fl = rvk.lib().rvk_dcg_plan_flags(plan.h)
    import torch.distributed as dist
    dist.barrier()
    plan.close()
    disconnect_peers(opened)
    n, nnz = bench._laplacian_size(3, 7, g)
    b_min = _shard_bytes(n, nnz, fl)
    hbm_peak, _ = bench.peaks()
    per_gpu = b_min / world / (ms * 1e-3) / 1e9
    if rank == 0:
        print(f"strong_768 N={world}: {ms:.2f} ms/solve ({backend}), {per_gpu:.0f} GB/s per GPU",
              file=__import__("sys").stderr, flush=True)
    return {"workload": "3D 7-point Laplacian 768^3, Jacobi-CG 20 iterations (BASELINE configs[4])",
            "n_gpus": world, "backend": backend, "comm_fallback": fallback,
            "ms_per_solve": round(ms, 3), "steps": steps,
            "iters_per_s": round(res.iterations / (ms * 1e-3), 1),
            "per_gpu_gbs": round(per_gpu, 1), "frac": round(per_gpu / hbm_peak, 4),
            "alg_bytes_per_solve": b_min, "host_syncs_per_iter": syncs / (steps * 20),
            "clocks": clocks}
def _global_nnz(dim, pts, grid):
    nx, ny, nz = (list(grid) + [1, 1])[:3]
    n = C.c_int64()
    nnz = C.c_int64()
    rvk.check(rvk.lib().rvk_laplacian_size(dim, pts, nx, ny, nz, C.byref(n), C.byref(nnz)))
    return nnz.value
