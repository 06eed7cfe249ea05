#!/usr/bin/env python3
"""Benchmark: 20-iteration Jacobi-CG solve on a constant-coefficient Laplacian.

Metric (BASELINE.json): "20-iter Jacobi-CG solve time, achieved HBM GB/s vs
peak, host syncs/iter".  One STEP = one full solve (setup residual + 20 CG
iterations, PAPER.md:46-65 timing loop; assembly and the Jacobi setup are
outside, as in the reference's KSPSolve timing).  Headline workload: 3D
7-point 256^3 (BASELINE.json north_star target) on one B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 7pt256]
  python bench.py --impl reference ...   # the reference CPU solver (oracle/_ref)

Prints ONE JSON line on rank 0.  Diagnostics go to stderr.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (dim, points, grid, description)
    "5pt1024": (2, 5, (1024, 1024), "2D 5-point Laplacian 1024x1024"),
    "9pt4096": (2, 9, (4096, 4096), "2D 9-point Laplacian 4096x4096"),
    "7pt256": (3, 7, (256, 256, 256), "3D 7-point Laplacian 256^3"),
    "27pt256": (3, 27, (256, 256, 256), "3D 27-point Laplacian 256^3"),
    "7pt768": (3, 7, (768, 768, 768), "3D 7-point Laplacian 768^3"),
    "7pt384": (3, 7, (384, 384, 384), "3D 7-point Laplacian 384^3 (plane-size study)"),
    "7pt512": (3, 7, (512, 512, 512), "3D 7-point Laplacian 512^3 (plane-size study)"),
    "5pt64": (2, 5, (64, 64), "2D 5-point Laplacian 64x64 (latency sweep)"),
    "5pt128": (2, 5, (128, 128), "2D 5-point Laplacian 128x128 (latency sweep)"),
    "5pt256": (2, 5, (256, 256), "2D 5-point Laplacian 256x256 (latency sweep)"),
    "5pt512": (2, 5, (512, 512), "2D 5-point Laplacian 512x512 (latency sweep)"),
}
METRIC = "20-iter Jacobi-CG solve time, achieved HBM GB/s vs peak, host syncs/iter"
MAX_IT = 20
L2_BYTES = 126 * 2 ** 20


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy kernel)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def bytes_model(n: int, nnz: int, mode: str = "fused", const_diag: bool = False,
                off32: bool = False, x_defer: bool = False, z_virtual: bool = False,
                x_group: int = 2, fold_setup: bool = False):
    """Algorithmic HBM bytes.  All FP64 + int64 offsets + int32 cols.
    k1 = the SpMV launch (fused: + on-the-fly AYPX), k2 = the rest of an iteration.
    const_diag: the plan folded a constant Jacobi diagonal into a scalar
    (RVK_PLAN_CONST_DIAG), so the dinv stream (8n per iteration and in the
    setup) is not part of the algorithm's traffic any more.  off32: the SpMV
    streams the plan's int32 copy of the row offsets (RVK_PLAN_OFF32): 4 instead
    of 8 bytes per row.  x_defer: x += a p applied once per GROUP of x_group
    iterations (RVK_PLAN_X_DEFER / _X_GROUP4 / _X_SOLVE = the whole solve):
    the x traffic per iteration drops from 24 n (p read, x read + write) to
    8 n + 16 n / x_group.
    z_virtual: z = d r is never stored (RVK_PLAN_Z_VIRTUAL): K2 and the setup
    write 8 n less; K1 gathers r instead of z (same bytes)."""
    ob = 4 if off32 else 8
    # x_group > 4 (the whole solve): K2 never touches x; one k_cg_xfix pass at
    # the end reads the x_group p's and writes x (starting from 0.0: the setup
    # does not store x = 0 either) -- counted per solve
    x_pass = (8 * n + 8 * n * x_group) if (x_defer and x_group > 4) else 0
    x_cut = (24 * n if x_pass else 16 * n - 16 * n // x_group) if x_defer else 0
    if mode == "stencil":                        # matrix-free: no CSR, constant dinv
        k1 = 32 * n                              # z, p_old -> p_new, w
        k2 = 56 * n - x_cut - (8 * n if z_virtual else 0)
        b_min = k1 + k2 + x_pass // MAX_IT
        st = (24 if z_virtual else 32) * n - (8 * n if x_pass else 0) - (8 * n if z_virtual else 16 * n)
        return {"k1": k1, "k2": k2, "b_min_iter": b_min, "b_ref_iter": b_min,
                "b_min_solve": MAX_IT * b_min + st,
                "b_ref_solve": MAX_IT * b_min + st,
                "b_min_survey_solve": MAX_IT * (12 * nnz + 8 * (n + 1) + 96 * n) + 64 * n,
                "flops_iter": 2 * nnz + 13 * n}
    if mode == "fused":
        k1 = 12 * nnz + ob * (n + 1) + 32 * n   # off, cols, vals, z, p_old -> p_new, w
        k2 = (56 if const_diag else 64) * n      # x, p, r, w, (dinv) -> x, r, z
        k2 -= x_cut
        if z_virtual:
            k2 -= 8 * n
    else:
        k1 = 12 * nnz + ob * (n + 1) + 16 * n   # off, cols, vals, p -> w
        k2 = 136 * n                             # aypx 24, dot 16, 2 axpy 48, jacobi 24, norm 8, dot 16
    b_min = k1 + k2 + (x_pass // MAX_IT if mode == "fused" else 0)  # 12 nnz + 8 (n+1) + 96 n plain
    b_ref = 12 * nnz + 8 * (n + 1) + 152 * n     # reference's unfused sequence
    setup = (56 if (const_diag and mode == "fused") else 64) * n - (8 * n if z_virtual else 0) \
        - (8 * n if x_pass else 0)
    if fold_setup and mode == "fused":  # setup inside K1(0): only its r = b store is extra
        setup = 8 * n
    survey = MAX_IT * (12 * nnz + 8 * (n + 1) + 96 * n) + 64 * n  # SURVEY.md 8d B_min as stated
    # fused fixed-iteration solve: the last K2 stores neither r nor z (dead)
    last = ((8 if z_virtual else 16) * n) if mode == "fused" else 0
    return {"k1": k1, "k2": k2, "b_min_iter": b_min, "b_ref_iter": b_ref,
            "b_min_solve": MAX_IT * b_min + setup - last, "b_ref_solve": MAX_IT * b_ref + setup,
            "b_min_survey_solve": survey, "flops_iter": 2 * nnz + 13 * n}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.p = None
        self.path = os.path.join("/tmp", f"rvk_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *exc):
        if self.p:
            time.sleep(0.2)
            self.p.terminate()
            self.p.wait()
            self.f.close()

    def summary(self):
        if not self.p or not os.path.exists(self.path):
            return None
        rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                smax = float(r[2])
                for name, v in zip(names, r[5:9]):
                    if v.strip() == "Active":
                        reasons.add(name)
            except (ValueError, IndexError):
                continue
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def ncu_traffic(config: str):
    """DRAM bytes per K1 launch from the committed `ncu --set full` summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    k = d.get(config, {}).get("k1")
    return k.get("dram_bytes") if k else None


def cpu_baseline(dim, pts, grid, steps=1):
    """The reference's own kernels (oracle/_ref, kernels_scalar.cpp via dispatch)
    running the restated PCG, 1 host thread (the kernels are single-threaded).
    Sample = `steps` full 20-iteration solves of the SAME workload, or, above
    ~256^3 rows, of a slab of whole planes of it (~16.8 M rows) with each
    time scaled to the workload by nnz.  Returns (kind, times_ms, sample)."""
    import oracle as O
    kind = "reference" if O.ref_available() else "port"
    nx, ny, nz = (list(grid) + [1, 1])[:3]
    plane, nplanes = (nx * ny, nz) if dim == 3 else (nx, ny)
    sgrid = tuple(grid)
    if plane * nplanes > 256 ** 3:
        k = max(1, 256 ** 3 // plane)
        sgrid = (nx, ny, k) if dim == 3 else (nx, k)
    A = O.build_laplacian(dim, pts, sgrid)
    b = O.rhs(A.n_rows)
    scale = _laplacian_size(dim, pts, grid)[1] / A.nnz
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        if kind == "reference":
            O.ref_cg_solve(A, b, max_it=MAX_IT, backend=2)   # reference auto dispatch
        else:
            O.cg_solve(A, b, max_it=MAX_IT)
        times.append((time.perf_counter() - t0) * 1e3 * scale)
    what = (f"{steps} full {MAX_IT}-iteration solve(s)" if sgrid == tuple(grid) else
            f"{steps} {MAX_IT}-iteration solve(s) of a {sgrid} slab, scaled by nnz x{scale:.3f}")
    return kind, times, what


def workload_grid(args, cfg, world: int):
    """The global grid bench.py solves at N = world GPUs (sharded.bench_main):
    weak scaling stacks one config-sized slab per GPU along the slowest axis;
    7pt768 is strong scaling of the fixed grid."""
    dim, pts, grid, desc = cfg
    if world > 1 and args.config != "7pt768":
        return tuple(grid[:-1]) + (grid[-1] * world,)
    return tuple(grid)


def run_reference(args, cfg):
    """The reference CPU solver (reference kernels from oracle/_ref driving the
    PETSc-order PCG, or the oracle port) on the host, rank 0 only.  For
    workloads above ~256^3 rows (N > 1 weak scaling, 768^3) one bounded sample
    is timed -- a slab of whole planes of the same grid holding ~16.8 M rows --
    and scaled to the whole workload by nnz (per-iteration cost is linear in
    nnz and n at fixed stencil)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    dim, pts, grid, desc = cfg
    t_all = time.perf_counter()
    import oracle as O
    kind = "reference" if O.ref_available() else "port"
    full = workload_grid(args, cfg, world)
    nx, ny, nz = (list(full) + [1, 1])[:3]
    plane = nx * ny if dim == 3 else nx
    nplanes = nz if dim == 3 else ny
    cap = 256 ** 3
    sample = full
    if plane * nplanes > cap:
        k = max(1, cap // plane)
        sample = (nx, ny, k) if dim == 3 else (nx, k)
    A = O.build_laplacian(dim, pts, sample)
    b = O.rhs(A.n_rows)
    n_full, nnz_full = _laplacian_size(dim, pts, full)
    scale = nnz_full / A.nnz
    solve = (lambda: O.ref_cg_solve(A, b, max_it=MAX_IT, backend=2)) if kind == "reference" \
        else (lambda: O.cg_solve(A, b, max_it=MAX_IT))
    for _ in range(args.warmup):
        solve()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        solve()
        times.append((time.perf_counter() - t0) * 1e3 * scale)
    ms = statistics.mean(times)
    # the reference's scalar and AVX2 backends, one solve each
    per_backend = {}
    if kind == "reference":
        for name, be in (("scalar", 0), ("avx2", 1)):
            t0 = time.perf_counter()
            O.ref_cg_solve(A, b, max_it=MAX_IT, backend=be)
            per_backend[name] = round((time.perf_counter() - t0) * 1e3 * scale, 3)
    bm = bytes_model(n_full, nnz_full)
    what = (f"{args.steps} full {MAX_IT}-iteration solves of {desc}" if sample == full else
            f"{args.steps} {MAX_IT}-iteration solves of a {sample} slab of the {full} workload "
            f"(whole planes, {A.n_rows} rows), each scaled by nnz x{scale:.3f}")
    wl = f"{desc}, Jacobi-CG {MAX_IT} iterations" + (f", global grid {full} (N={world})"
                                                       if full != tuple(grid) else "")
    out = {
        "metric": METRIC, "impl": "reference", "value": round(ms, 3), "unit": "ms/solve",
        "n_gpus": 0, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "min_ms": round(min(times), 3), "higher_is_better": False,
        "scaling": "strong" if args.config == "7pt768" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl, "n": n_full, "nnz": nnz_full},
        "cpu_baseline": {"value": round(ms, 3), "unit": "ms/solve", "cores": 1, "kind": kind,
                         "sample": what + " (reference kernels_*.cpp, auto AVX2/scalar dispatch, "
                                          "single-threaded like the reference's kernels)",
                         "per_backend_ms": per_backend, "host_cpu": host_cpu()},
        "e2e": {"value": round(ms, 3), "unit": "ms/solve", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "achieved_gbs_bref": round(bm["b_ref_solve"] / (ms * 1e-3) / 1e9, 2),
        "host_syncs_per_iter": 0,
    }
    log(f"reference CPU: {ms:.1f} ms/solve (min {min(times):.1f}); total {time.perf_counter()-t_all:.0f}s")
    print(json.dumps(out), flush=True)


def host_cpu() -> dict:
    """Host CPU model and logical CPU count (stated beside the
    CPU baseline)."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"model": model, "logical_cpus": os.cpu_count()}


def _laplacian_size(dim, pts, grid):
    """(n, nnz) of the stencil operator on `grid` -- closed forms."""
    nx, ny, nz = (list(grid) + [1, 1])[:3]
    if dim == 2:
        n = nx * ny
        nnz = 5 * n - 2 * nx - 2 * ny if pts == 5 else (3 * nx - 2) * (3 * ny - 2)
    else:
        n = nx * ny * nz
        nnz = (7 * n - 2 * (nx * ny + ny * nz + nx * nz) if pts == 7 else
               (3 * nx - 2) * (3 * ny - 2) * (3 * nz - 2))
    return n, nnz


def tfqmr_bytes(n: int, nnz: int, const_diag: bool = False):
    """Algorithmic HBM bytes of the fused TFQMR solve (rvk_tfqmr.cu header):
    KA = CSR + 7n doubles, KM = 11n (6n in the last iteration), KB = CSR + 4n;
    setup K0 = 8n, plus one KB; no KB after the last iteration.  const_diag
    (the plan's RVK_PLAN_CONST_DIAG): no dinv stream in K0, KA, KB (-8n each)."""
    csr = 12 * nnz + 8 * (n + 1)
    dv = 0 if const_diag else 8 * n
    ka, km, km_last, kb, k0 = csr + 48 * n + dv, 88 * n, 48 * n, csr + 24 * n + dv, 56 * n + dv
    solve = k0 + kb + MAX_IT * ka + (MAX_IT - 1) * (km + kb) + km_last
    return {"ka": ka, "km": km, "kb": kb, "b_min_solve": solve}


def run_tfqmr(args, cfg):
    """--solver tfqmr: the 20-iteration left-Jacobi TFQMR solve (SURVEY.md 8f
    row 3), same workload, timing rules and JSON shape."""
    import torch
    from paper_2306_17801_b200 import rvk

    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        raise SystemExit("--solver tfqmr is single-GPU (replicas only)")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dim, pts, grid, desc = cfg
    stream = torch.cuda.Stream()
    ctx = rvk.Ctx(stream.cuda_stream)
    A = rvk.DeviceCsr.laplacian(ctx, dim, pts, grid)
    n, nnz = A.n_rows, A.nnz
    b, x = rvk.DeviceArray(n), rvk.DeviceArray(n)
    rvk.check(rvk.lib().rvk_fill_rhs(ctx.h, 0x9E3779B97F4A7C15, n, b.ptr))
    mode = "unfused" if args.mode == "unfused" else "fused"
    plan = rvk.TfqmrPlan(ctx, A, max_it=MAX_IT, use_graph=not args.no_graph, mode=mode)
    bm = tfqmr_bytes(n, nnz, bool(plan.flags() & 1) and mode == "fused")
    hbm_peak, peak_src = peaks()
    ws_bytes = 20 * nnz + 8 * (n + 1) + 11 * 8 * n
    for _ in range(args.warmup):
        plan.solve_dev(b, x)
    res = plan.result()
    assert res.iterations == MAX_IT, res
    flush = None
    if ws_bytes < 2 * L2_BYTES:
        flush = torch.empty(512 * 2 ** 20, dtype=torch.uint8, device=f"cuda:{local}")
    syncs0 = rvk.host_syncs()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            for k in range(args.steps):
                if flush is not None:
                    flush.fill_(k & 0xFF)
                ev0[k].record(stream)
                plan.solve_dev(b, x)
                ev1[k].record(stream)
        stream.synchronize()
    syncs = rvk.host_syncs() - syncs0
    step_ms = [ev0[k].elapsed_time(ev1[k]) for k in range(args.steps)]
    ms = sum(step_ms) / args.steps
    res = plan.result()
    solve_gbs = bm["b_min_solve"] / (ms * 1e-3) / 1e9
    launches = (2 + MAX_IT * 3 - 1) if mode == "fused" else None
    # e2e: pinned host b -> device, solve, x + history back
    bh = torch.empty(n, dtype=torch.float64, pin_memory=True)
    xh = torch.empty(n, dtype=torch.float64, pin_memory=True)
    bh.numpy()[:] = b.download(ctx)
    L = rvk.lib()

    def e2e_once():
        rvk.check(L.rvk_memcpy_h2d(ctx.h, b.ptr, bh.data_ptr(), 8 * n))
        plan.solve_dev(b, x)
        rvk.check(L.rvk_memcpy_d2h(ctx.h, xh.data_ptr(), x.ptr, 8 * n))
        plan.result()

    for _ in range(max(1, args.warmup)):
        e2e_once()
    e2e = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        e2e_once()
        e2e.append((time.perf_counter() - t0) * 1e3)
    e2e_ms = statistics.mean(e2e)
    cpu = None
    if not args.no_cpu_baseline:
        import oracle as O
        Ah = O.build_laplacian(dim, pts, grid)
        bb = O.rhs(Ah.n_rows)
        t0 = time.perf_counter()
        O.tfqmr_solve(Ah, bb, max_it=MAX_IT)
        cpu = {"value": round((time.perf_counter() - t0) * 1e3, 1), "unit": "ms/solve", "cores": 1,
               "kind": "port",
               "sample": f"1 full {MAX_IT}-iteration TFQMR solve of {desc} (oracle restatement; "
                         "the reference ships no TFQMR source)"}
    out = {
        "metric": f"20-iter Jacobi-TFQMR solve time, achieved HBM GB/s vs peak, host syncs/iter",
        "value": round(ms, 4), "unit": "ms/solve", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "min_ms": round(min(step_ms), 4),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{desc}, left-Jacobi TFQMR {MAX_IT} iterations, x0=0, splitmix64 RHS",
                   "n": n, "nnz": nnz, "mode": mode, "graph": not args.no_graph,
                   "l2": "no flush: working set >> L2" if flush is None else "L2 flushed between steps"},
        "solve_roofline": {"bound": "hbm", "alg_bytes_per_solve": bm["b_min_solve"],
                           "achieved": round(solve_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                           "frac": round(solve_gbs / hbm_peak, 4), "peak_source": peak_src},
        "host_syncs_per_iter": syncs / (args.steps * MAX_IT),
        "e2e": {"value": round(e2e_ms, 4), "unit": "ms/solve", "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": 8 * n + 8 * (2 * MAX_IT + 1) + 64},
        "gpu_launches": launches * args.steps if launches else None,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
    }
    log(f"tfqmr {mode}: solve {ms:.3f} ms (min {min(step_ms):.3f}); {solve_gbs:.0f} GB/s "
        f"({solve_gbs/hbm_peak:.1%}); e2e {e2e_ms:.2f} ms; syncs {syncs}")
    print(json.dumps(out), flush=True)
    plan.close()
    ctx.close()


def run_gpu(args, cfg):
    import torch
    from paper_2306_17801_b200 import rvk

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        log(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}")
    if world > 1:
        from paper_2306_17801_b200 import sharded
        return sharded.bench_main(args, cfg)
    torch.cuda.set_device(local)
    dim, pts, grid, desc = cfg
    stream = torch.cuda.Stream()
    ctx = rvk.Ctx(stream.cuda_stream)
    if args.operator == "stencil":
        import ctypes
        nn, nz_ = ctypes.c_int64(), ctypes.c_int64()
        gx, gy, gz = (list(grid) + [1, 1])[:3]
        rvk.check(rvk.lib().rvk_laplacian_size(dim, pts, gx, gy, gz, ctypes.byref(nn), ctypes.byref(nz_)))
        n, nnz = nn.value, nz_.value
        A = (dim, pts, grid)
    else:
        A = rvk.DeviceCsr.laplacian(ctx, dim, pts, grid)
        n, nnz = A.n_rows, A.nnz
    b = rvk.DeviceArray(n)
    x = rvk.DeviceArray(n)
    rvk.check(rvk.lib().rvk_fill_rhs(ctx.h, 0x9E3779B97F4A7C15, n, b.ptr))
    plan = rvk.CgPlan(ctx, A, max_it=MAX_IT, mode=args.mode, use_graph=not args.no_graph)
    const_diag = bool(plan.flags() & 1)
    off32 = bool(plan.flags() & 8)
    x_defer = bool(plan.flags() & 16)
    x_group = MAX_IT if plan.flags() & 128 else (4 if plan.flags() & 64 else 2)
    z_virtual = bool(plan.flags() & 32)
    bm = bytes_model(n, nnz, "stencil" if args.operator == "stencil" else
                     ("unfused" if args.mode == "unfused" else "fused"), const_diag, off32, x_defer,
                     z_virtual, x_group, bool(plan.flags() & 512))
    hbm_peak, peak_src = peaks()
    ws_bytes = 20 * nnz + 8 * (n + 1) + 9 * 8 * n
    log(f"{desc}: n={n} nnz={nnz} working set {ws_bytes/1e9:.2f} GB (L2 {L2_BYTES/1e6:.0f} MB)")

    for _ in range(args.warmup):
        plan.solve_dev(b, x)
    res = plan.result()
    assert res.iterations == MAX_IT, res

    # ---- timed region: K solves, CUDA events on the solve stream --------------
    # Working sets above 2x L2 stream from HBM anyway; smaller ones get an L2
    # flush (a 512 MiB write on the same stream) between steps, outside the
    # per-step event pairs.
    flush = None
    if ws_bytes < 2 * L2_BYTES:
        flush = torch.empty(512 * 2 ** 20, dtype=torch.uint8, device=f"cuda:{local}")
    syncs0 = rvk.host_syncs()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            for k in range(args.steps):
                if flush is not None:
                    flush.fill_(k & 0xFF)
                ev0[k].record(stream)
                plan.solve_dev(b, x)
                ev1[k].record(stream)
        stream.synchronize()
    syncs = rvk.host_syncs() - syncs0
    step_ms = [ev0[k].elapsed_time(ev1[k]) for k in range(args.steps)]
    ms = sum(step_ms) / args.steps
    res = plan.result()
    assert res.iterations == MAX_IT
    launches = plan.launches()

    mode = plan.mode()
    if mode in ("fused", "unfused"):
        # ---- per-kernel durations: the same solves with event pairs captured in
        # the graph around every K1 (SpMV) and K2 (update) launch, same stream --
        plan.set_profiling(True)
        plan.solve_dev(b, x)                      # (re)capture the profiled graph
        plan.result()
        k1_ms = k2_ms = 0.0
        for _ in range(args.steps):
            plan.solve_dev(b, x)
            plan.result()
            a1, a2, _ = plan.kernel_times()
            k1_ms += a1
            k2_ms += a2
        k1_ms /= args.steps
        k2_ms /= args.steps
        plan.set_profiling(False)
        k1_avg = k1_ms / MAX_IT
        k2_avg = k2_ms / MAX_IT
        k1_gbs = bm["k1"] / (k1_avg * 1e-3) / 1e9
        k2_gbs = bm["k2"] / (k2_avg * 1e-3) / 1e9
    else:
        # one persistent kernel (or the host-sync baseline): the dominant
        # "kernel" is the whole solve
        k1_avg, k2_avg = ms, 0.0
        bm = dict(bm, k1=bm["b_min_solve"])
        k1_gbs = bm["k1"] / (ms * 1e-3) / 1e9
        k2_gbs = 0.0
    solve_gbs = bm["b_min_solve"] / (ms * 1e-3) / 1e9
    traffic = ncu_traffic(args.config) if (mode == "fused" and args.operator == "csr") else None

    # ---- e2e through the C-ABI with host buffers (pinned) ----------------------
    # (1) latency: one rvk_cg_solve_host call per step (H2D b, solve, D2H x +
    #     hist, sync), wall clock;
    # (2) headline e2e: the K steps as a stream of K right-hand sides through
    #     rvk_cg_solve_host_many -- every step still copies its b in and its x
    #     out inside the timed region, but the copies of step k+-1 overlap
    #     solve k on the copy engines (double-buffered staging).
    bh = [torch.empty(n, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    xh = [torch.empty(n, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    bh[0].numpy()[:] = b.download(ctx)
    bh[1].numpy()[:] = bh[0].numpy()
    hist = np.empty(MAX_IT + 1)
    for _ in range(max(1, args.warmup)):
        plan.solve_host(bh[0].numpy(), xh[0].numpy(), hist)
    lat = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        _, r = plan.solve_host(bh[0].numpy(), xh[0].numpy(), hist)
        lat.append((time.perf_counter() - t0) * 1e3)
    lat_ms = statistics.mean(lat)
    bs = [bh[k & 1].numpy() for k in range(args.steps)]
    xs = [xh[k & 1].numpy() for k in range(args.steps)]
    plan.solve_host_many(bs[:2], xs[:2])  # warm: captures the second staging pair's graph
    t0 = time.perf_counter()
    many = plan.solve_host_many(bs, xs)
    e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    assert all(m.iterations == MAX_IT for m in many)

    cpu = None
    if not args.no_cpu_baseline:
        kind, ctimes, what = cpu_baseline(dim, pts, grid, steps=1)
        cpu = {"value": round(statistics.mean(ctimes), 1), "unit": "ms/solve", "cores": 1,
               "kind": kind,
               "sample": f"{what} of {desc} on the GPU box host "
                         "(reference kernels_*.cpp from oracle/_ref, auto dispatch, 1 thread)",
               "host_cpu": host_cpu()}

    out = {
        "metric": METRIC, "value": round(ms, 4), "unit": "ms/solve", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "min_ms": round(min(step_ms), 4), "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{desc}, Jacobi-CG {MAX_IT} iterations, x0=0, splitmix64 RHS",
                   "n": n, "nnz": nnz, "mode": mode, "graph": not args.no_graph,
                   "operator": args.operator,
                   "l2": (f"no flush: working set {ws_bytes/1e9:.2f} GB >> 126 MB L2 "
                          "(every operand streams from HBM each step)") if flush is None else
                         (f"L2 flushed between steps (512 MiB write); working set "
                          f"{ws_bytes/1e6:.1f} MB")},
        "roofline": {"bound": "hbm",
                     "kernel": {"fused": ("k_mf_cg (matrix-free stencil + on-the-fly AYPX + p.w)"
                                          if args.operator == "stencil" else
                                          "k_spmv_tma<CgSpmvOp> (SpMV + on-the-fly AYPX + p.w)"),
                                "unfused": "k_spmv_tma<SpmvGuardedOp> (SpMV)",
                                "persistent": "k_cg_persistent (whole solve, one launch)",
                                "hostsync": "whole solve (host-sync baseline)"}[mode],
                     "achieved": round(k1_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                     "frac": round(k1_gbs / hbm_peak, 4), "traffic": traffic,
                     "alg_bytes_per_launch": bm["k1"], "avg_launch_ms": round(k1_avg, 5),
                     "peak_source": peak_src},
        "solve_roofline": {"alg_bytes_per_solve": bm["b_min_solve"],
                           "achieved": round(solve_gbs, 1), "frac": round(solve_gbs / hbm_peak, 4),
                           "update_kernel_gbs": round(k2_gbs, 1),
                           "const_diag_folded": const_diag,
                           "int32_row_offsets": off32,
                           "x_update_group": x_group if x_defer else 1,
                           "z_virtual": z_virtual,
                           "survey_b_min_gbs": round(bm["b_min_survey_solve"] / (ms * 1e-3) / 1e9, 1),
                           "b_ref_gbs": round(bm["b_ref_solve"] / (ms * 1e-3) / 1e9, 1)},
        "host_syncs_per_iter": syncs / (args.steps * MAX_IT),
        "iters_per_s": round(MAX_IT / (ms * 1e-3), 1),
        "e2e": {"value": round(e2e_ms, 4), "unit": "ms/solve", "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": 8 * n + 8 * (MAX_IT + 1) + 64,
                "api": "rvk_cg_solve_host_many: K right-hand sides from pinned host memory, "
                       "H2D/D2H of neighbouring steps overlapped with the solve (wall clock)",
                "latency_ms": round(lat_ms, 4),
                "latency_api": "rvk_cg_solve_host: one RHS per call, H2D + solve + D2H "
                               "serial, synchronised (wall clock)"},
        "gpu_launches": launches * args.steps,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
    }
    log(f"solve {ms:.3f} ms (min {min(step_ms):.3f}); K1 {k1_avg*1e3:.1f} us = {k1_gbs:.0f} GB/s; "
        f"K2 {k2_avg*1e3:.1f} us = {k2_gbs:.0f} GB/s; solve {solve_gbs:.0f} GB/s "
        f"({solve_gbs/hbm_peak:.1%}); e2e {e2e_ms:.2f} ms (latency {lat_ms:.2f}); syncs {syncs}")
    print(json.dumps(out), flush=True)
    plan.close()
    ctx.close()


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawTextHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["rvk", "reference"], default="rvk")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="7pt256")
    ap.add_argument("--mode", choices=["fused", "unfused", "persistent", "auto", "hostsync"],
                    default="auto", help="auto: one persistent kernel for L2-sized grids, "
                                         "else the fused 2-kernel/iteration graph")
    ap.add_argument("--operator", choices=["csr", "stencil"], default="csr",
                    help="csr: the AIJ/CSR operator (headline); stencil: matrix-free (SURVEY 8f)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--comm", choices=["peer", "nccl"], default="peer",
                    help="N>1: peer = in-kernel NVLink halo/partial pushes (fused); nccl = "
                         "library collectives between kernels (baseline)")
    ap.add_argument("--solver", choices=["cg", "tfqmr"], default="cg",
                    help="cg: the headline Jacobi-PCG; tfqmr: left-Jacobi TFQMR (SURVEY 8f)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "rvk":
        log("note: raising --warmup to 3 (timing rule)")
        args.warmup = 3
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    elif args.solver == "tfqmr":
        run_tfqmr(args, cfg)
    else:
        run_gpu(args, cfg)


if __name__ == "__main__":
    main()
