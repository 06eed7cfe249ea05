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
    "5pt768": (2, 5, (768, 768), "2D 5-point Laplacian 768x768 (latency sweep)"),
    "9pt1024": (2, 9, (1024, 1024), "2D 9-point Laplacian 1024x1024 (grid-solve study)"),
    "7pt100": (3, 7, (100, 100, 100), "3D 7-point Laplacian 100^3 (grid-solve study)"),
    "7pt128": (3, 7, (128, 128, 128), "3D 7-point Laplacian 128^3 (fused persistent study)"),
    "9pt2048": (2, 9, (2048, 2048), "2D 9-point Laplacian 2048x2048 (fused persistent study)"),
    "5pt2048": (2, 5, (2048, 2048), "2D 5-point Laplacian 2048x2048 (fused persistent study)"),
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
                x_defer: bool = False, z_virtual: bool = False,
                x_group: int = 2, fold_setup: bool = False):
    """Algorithmic HBM bytes.  All FP64 + int64 offsets + int32 cols.
    k1 = the SpMV launch (fused: + on-the-fly AYPX), k2 = the rest of an iteration.
    const_diag: the plan folded a constant Jacobi diagonal into a scalar
    (RVK_PLAN_CONST_DIAG), so the dinv stream (8n per iteration and in the
    setup) is not part of the algorithm's traffic any more.  x_defer: x += a p
    applied once per GROUP of x_group
    iterations (RVK_PLAN_X_DEFER / _X_GROUP4 / _X_SOLVE = the whole solve):
    the x traffic per iteration drops from 24 n (p read, x read + write) to
    8 n + 16 n / x_group.
    z_virtual: z = d r is never stored (RVK_PLAN_Z_VIRTUAL): K2 and the setup
    write 8 n less; K1 gathers r instead of z (same bytes)."""
    ob = 8  # int64 row offsets
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


def _file_sha16(path: str) -> str | None:
    import hashlib
    try:
        with open(path, "rb") as f:
            return hashlib.sha256(f.read()).hexdigest()[:16]
    except OSError:
        return None


def ncu_traffic(config: str, kernel: str = "k1"):
    """DRAM bytes per launch of `kernel` from the committed `ncu --set full`
    summary (profiles/ncu_summary.json), with where it came from: the capture
    records the sha of the librvk.so it profiled, compared here with the
    library this run loaded (a kernel change without a profile refresh shows
    up as build_match = false)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None, None
    with open(p) as f:
        d = json.load(f)
    k = d.get(config, {}).get(kernel)
    if not k:
        return None, None
    from paper_2306_17801_b200 import rvk
    lib = os.path.join(ROOT, "paper_2306_17801_b200", "lib", "librvk.so")
    src = {"file": "profiles/ncu_summary.json", "capture": d.get("_note"),
           "captured_build_id": d.get("build_id"), "loaded_build_id": rvk.lib().rvk_build_id().decode(),
           "captured_lib_sha16": d.get("lib_sha16"), "loaded_lib_sha16": _file_sha16(lib)}
    # build ids hash the library's sources (stable across rebuilds)
    src["build_match"] = bool(src["captured_build_id"]) and \
        src["captured_build_id"] == src["loaded_build_id"]
    return k.get("dram_bytes"), src


# ---- workload and config (identical for the GPU arm and the reference arm) ----
STRONG = {"7pt768"}   # configs whose total work is fixed as N grows


def workload(args, world: int):
    """(dim, pts, global grid, desc, strong): weak scaling stacks one
    config-sized slab per GPU along the slowest axis; 7pt768 is the fixed
    (strong-scaling) grid of BASELINE.json configs[4]."""
    dim, pts, grid, desc = CONFIGS[args.config]
    strong = args.config in STRONG
    if world > 1 and not strong:
        return dim, pts, tuple(grid[:-1]) + (grid[-1] * world,), desc, False
    return dim, pts, tuple(grid), desc, strong


def bench_config(args, world: int) -> dict:
    dim, pts, g, desc, strong = workload(args, world)
    n, nnz = _laplacian_size(dim, pts, g)
    wl = f"{desc}, Jacobi-CG {MAX_IT} iterations, x0=0, splitmix64 RHS"
    if g != tuple(CONFIGS[args.config][2]):
        wl += f"; global grid {'x'.join(map(str, g))} ({world} row slabs)"
    cfg = {"workload": wl, "n": n, "nnz": nnz}
    if world > 1:
        cfg["parallelism"] = f"rows{world}"
    return cfg


def scaling_label(args) -> str:
    return "strong" if args.config in STRONG else "weak"


# ---- the reference CPU solver (oracle/_ref), bounded sample ------------------
SAMPLE_ROWS = 1 << 22


def sample_grid(dim, grid):
    """The CPU sample: whole planes (slowest axis) of the workload grid, at most
    SAMPLE_ROWS rows (~1.5 s per 20-iteration solve on one core)."""
    nx, ny, nz = (list(grid) + [1, 1])[:3]
    plane, nplanes = (nx * ny, nz) if dim == 3 else (nx, ny)
    k = max(2, min(nplanes, SAMPLE_ROWS // plane))
    return ((nx, ny, k) if dim == 3 else (nx, k)) if k < nplanes else tuple(grid)


def time_reference(dim, pts, grid, steps: int, warmup: int, solver: str = "cg") -> dict:
    """The reference's own kernels (oracle/_ref, kernels_{scalar,avx2}.cpp)
    driving the PETSc-order PCG on this host, 1 thread (the reference's
    kernels are single-threaded), on a bounded sample of the workload, each
    time scaled to the whole workload by nnz (per-iteration cost is linear in
    nnz and n at a fixed stencil).  Both backends are timed once; the FASTEST
    is the baseline (the reference's auto dispatch picks AVX2 when present,
    kernels_dispatch.cpp:76-89, which is not always the faster one).  The
    oracle port stands in when oracle/_ref is absent (kind "port")."""
    import oracle as O
    kind = "reference" if O.ref_available() else "port"
    sg = sample_grid(dim, grid)
    A = O.build_laplacian(dim, pts, sg)
    b = O.rhs(A.n_rows)
    scale = _laplacian_size(dim, pts, grid)[1] / A.nnz
    if kind == "reference":
        backends = {"scalar": 0}
        if O.ref_lib().ref_avx2_supported():
            backends["avx2"] = 1
        ref = O.ref_tfqmr_solve if solver == "tfqmr" else O.ref_cg_solve
        solvers = {k: (lambda be=be: ref(A, b, max_it=MAX_IT, backend=be))
                   for k, be in backends.items()}
    else:
        port = O.tfqmr_solve if solver == "tfqmr" else O.cg_solve
        solvers = {"port": lambda: port(A, b, max_it=MAX_IT)}
    solvers[next(iter(solvers))]()  # first touch of the work arrays (page faults), untimed
    per = {}
    for name, f in solvers.items():
        t0 = time.perf_counter()
        f()
        per[name] = (time.perf_counter() - t0) * 1e3 * scale
    best = min(per, key=per.get)
    for _ in range(warmup):
        solvers[best]()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        solvers[best]()
        times.append((time.perf_counter() - t0) * 1e3 * scale)
    if not times:
        times = [per[best]]
    what = (f"full {MAX_IT}-iteration solves" if sg == tuple(grid) else
            f"{MAX_IT}-iteration solves of a {'x'.join(map(str, sg))} slab (whole planes, "
            f"{A.n_rows} rows) of the {'x'.join(map(str, grid))} workload, each scaled by nnz "
            f"x{scale:.3f}")
    return {"kind": kind, "best": best, "per_backend_ms": {k: round(v, 1) for k, v in per.items()},
            "times_ms": times, "sample": what, "cores": 1}


def run_reference(args, cfg):
    """--impl reference: the reference CPU solver on this host, rank 0 only
    (other ranks exit without work), on the GPU arm's workload / config /
    metric.  Each step is one bounded sample solve with the reference's
    fastest backend (time_reference)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    t_all = time.perf_counter()
    dim, pts, g, desc, _ = workload(args, world)
    ref = time_reference(dim, pts, g, args.steps, args.warmup)
    ms = statistics.mean(ref["times_ms"])
    n, nnz = _laplacian_size(dim, pts, g)
    bm = bytes_model(n, nnz)
    out = {
        "metric": METRIC, "impl": "reference", "value": round(ms, 3), "unit": "ms/solve",
        "n_gpus": 0, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "min_ms": round(min(ref["times_ms"]), 3), "higher_is_better": False,
        "scaling": scaling_label(args), "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args, world),
        "cpu_baseline": {"value": round(ms, 3), "unit": "ms/solve", "cores": ref["cores"],
                         "kind": ref["kind"],
                         "sample": ref["sample"] + f" ({ref['best']} backend: the fastest of "
                                   + ", ".join(ref["per_backend_ms"]) + ")",
                         "per_backend_ms": ref["per_backend_ms"], "host_cpu": host_cpu()},
        "e2e": {"value": round(ms, 3), "unit": "ms/solve", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "achieved_gbs_bref": round(bm["b_ref_solve"] / (ms * 1e-3) / 1e9, 2),
        "host_syncs_per_iter": 0,
    }
    log(f"reference CPU ({ref['best']}): {ms:.1f} ms/solve (min {min(ref['times_ms']):.1f}); "
        f"per backend {ref['per_backend_ms']}; total {time.perf_counter()-t_all:.0f}s")
    print(json.dumps(out), flush=True)


def cpu_baseline_entry(dim, pts, grid, solver: str = "cg") -> dict:
    """cpu_baseline of a GPU line: one sample solve per reference backend, the
    fastest reported (time_reference)."""
    ref = time_reference(dim, pts, grid, steps=0, warmup=0, solver=solver)
    return {"value": round(ref["per_backend_ms"][ref["best"]], 1), "unit": "ms/solve",
            "cores": ref["cores"], "kind": ref["kind"],
            "sample": "1 " + ref["sample"] + f" on the GPU box host per backend; value = the "
                      f"fastest ({ref['best']})",
            "per_backend_ms": ref["per_backend_ms"], "host_cpu": host_cpu()}


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
    # the TFQMR loop over the reference's own kernels (oracle/ref_shim.cpp:
    # ref_tfqmr_solve; the reference ships no TFQMR driver), fastest backend
    cpu = None if args.no_cpu_baseline else cpu_baseline_entry(dim, pts, grid, solver="tfqmr")
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


def time_solves(plan, b, x, stream, steps, warmup, flush=None):
    """K solves bracketed by CUDA events on the solve stream (device time),
    after `warmup` untimed ones; nvidia-smi clocks sampled during the timed
    region.  Returns (per-step ms, clock summary, host syncs counted)."""
    import torch
    from paper_2306_17801_b200 import rvk
    for _ in range(warmup):
        plan.solve_dev(b, x)
    plan.result()
    syncs0 = rvk.host_syncs()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    with ClockSampler(torch.cuda.current_device()) as clk:
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            for k in range(steps):
                if flush is not None:
                    flush.fill_(k & 0xFF)
                ev0[k].record(stream)
                plan.solve_dev(b, x)
                ev1[k].record(stream)
        stream.synchronize()
    syncs = rvk.host_syncs() - syncs0
    return [ev0[k].elapsed_time(ev1[k]) for k in range(steps)], clk.summary(), syncs


def strong768_single(args, stream, ctx) -> dict:
    """BASELINE.json configs[4] anchor at N = 1: the 768^3 7-point solve on
    this GPU (the single-GPU plan), reported beside the headline so the
    driver's N = 1, 2, 4, 8 runs give one strong-scaling curve under the same
    key (sharded.bench_main measures it at N > 1)."""
    from paper_2306_17801_b200 import rvk
    g = CONFIGS["7pt768"][2]
    A = rvk.DeviceCsr.laplacian(ctx, 3, 7, g)
    n, nnz = A.n_rows, A.nnz
    b, x = rvk.DeviceArray(n), rvk.DeviceArray(n)
    rvk.check(rvk.lib().rvk_fill_rhs(ctx.h, 0x9E3779B97F4A7C15, n, b.ptr))
    plan = rvk.CgPlan(ctx, A, max_it=MAX_IT, mode="fused", opts=args.opts)
    fl = plan.flags()
    bm = bytes_model(n, nnz, "fused", bool(fl & 1), bool(fl & 16), bool(fl & 32),
                     MAX_IT if fl & 128 else (4 if fl & 64 else 2), bool(fl & 512))
    steps = max(3, min(args.steps, 10))
    ms_list, clk, syncs = time_solves(plan, b, x, stream, steps, 3)
    res = plan.result()
    ms = statistics.mean(ms_list)
    hbm_peak, _ = peaks()
    gbs = bm["b_min_solve"] / (ms * 1e-3) / 1e9
    plan.close()
    log(f"strong_768 N=1: {ms:.2f} ms/solve, {gbs:.0f} GB/s ({gbs/hbm_peak:.1%})")
    return {"workload": "3D 7-point Laplacian 768^3, Jacobi-CG 20 iterations (BASELINE configs[4])",
            "n_gpus": 1, "plan": "single-GPU CSR plan", "ms_per_solve": round(ms, 3),
            "steps": steps, "iters_per_s": round(res.iterations / (ms * 1e-3), 1),
            "per_gpu_gbs": round(gbs, 1), "frac": round(gbs / hbm_peak, 4),
            "alg_bytes_per_solve": bm["b_min_solve"], "host_syncs_per_iter": syncs / (steps * MAX_IT),
            "clocks": clk}


def run_gpu(args, cfg):
    import torch
    from paper_2306_17801_b200 import rvk

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
        n, nnz = _laplacian_size(dim, pts, grid)
        A = (dim, pts, grid)
    else:
        A = rvk.DeviceCsr.laplacian(ctx, dim, pts, grid)
        n, nnz = A.n_rows, A.nnz
    b = rvk.DeviceArray(n)
    x = rvk.DeviceArray(n)
    rvk.check(rvk.lib().rvk_fill_rhs(ctx.h, 0x9E3779B97F4A7C15, n, b.ptr))
    plan = rvk.CgPlan(ctx, A, max_it=MAX_IT, mode=args.mode, use_graph=not args.no_graph,
                      opts=args.opts)
    fl = plan.flags()
    const_diag, x_defer, z_virtual = bool(fl & 1), bool(fl & 16), bool(fl & 32)
    x_group = MAX_IT if fl & 128 else (4 if fl & 64 else 2)
    bm = bytes_model(n, nnz, "stencil" if args.operator == "stencil" else
                     ("unfused" if args.mode == "unfused" else "fused"), const_diag, x_defer,
                     z_virtual, x_group, bool(fl & 512))
    hbm_peak, peak_src = peaks()
    ws_bytes = 20 * nnz + 8 * (n + 1) + 9 * 8 * n
    log(f"{desc}: n={n} nnz={nnz} working set {ws_bytes/1e9:.2f} GB (L2 {L2_BYTES/1e6:.0f} MB)")

    # ---- timed region: K solves, CUDA events on the solve stream --------------
    # Working sets above 2x L2 stream from HBM anyway; smaller ones get an L2
    # flush (a 512 MiB write on the same stream) between steps, outside the
    # per-step event pairs.
    flush = None
    if ws_bytes < 2 * L2_BYTES:
        flush = torch.empty(512 * 2 ** 20, dtype=torch.uint8, device=f"cuda:{local}")
    step_ms, clocks, syncs = time_solves(plan, b, x, stream, args.steps, args.warmup, flush)
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
    traffic, traffic_src = (None, None)
    if mode == "fused":
        traffic, traffic_src = ncu_traffic(args.config + ("_matrix_free" if args.operator == "stencil"
                                                          else ""))

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
    plan.close()
    del A, b, x, plan

    # ---- BASELINE configs[4] at N = 1 (the strong-scaling anchor) --------------
    strong = None
    if not args.no_strong and args.config != "7pt768" and args.operator == "csr":
        torch.cuda.synchronize()
        strong = strong768_single(args, stream, ctx)

    cpu = None if args.no_cpu_baseline else cpu_baseline_entry(dim, pts, grid)

    out = {
        "metric": METRIC, "value": round(ms, 4), "unit": "ms/solve", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "min_ms": round(min(step_ms), 4), "higher_is_better": False,
        "scaling": scaling_label(args), "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args, 1),
        "run": {"mode": mode, "graph": not args.no_graph, "operator": args.operator,
                "l2": (f"no flush: working set {ws_bytes/1e9:.2f} GB >> 126 MB L2 "
                       "(every operand streams from HBM each step)") if flush is None else
                      (f"L2 flushed between steps (512 MiB write); working set "
                       f"{ws_bytes/1e6:.1f} MB")},
        "roofline": {"bound": "hbm",
                     "kernel": {"fused": ("k_mf_tma (matrix-free stencil + on-the-fly AYPX + p.w)"
                                          if args.operator == "stencil" else
                                          ("k_spmv_march<CgSpmvOp> (plane-marching SpMV, smem plane "
                                           "cache + on-the-fly AYPX + p.w; K1(0): k_spmv_tma)"
                                           if fl & 1024 else
                                           "k_spmv_tma<CgSpmvOp> (SpMV + on-the-fly AYPX + p.w)")),
                                "unfused": "k_spmv_tma<SpmvGuardedOp> (SpMV)",
                                "persistent": "k_cg_persistent / k_cg_cluster (whole solve, one launch)",
                                "hostsync": "whole solve (host-sync baseline)"}[mode],
                     "achieved": round(k1_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                     "frac": round(k1_gbs / hbm_peak, 4), "traffic": traffic,
                     "traffic_source": traffic_src,
                     "alg_bytes_per_launch": bm["k1"], "avg_launch_ms": round(k1_avg, 5),
                     "peak_source": peak_src},
        "solve_roofline": {"alg_bytes_per_solve": bm["b_min_solve"],
                           "achieved": round(solve_gbs, 1), "frac": round(solve_gbs / hbm_peak, 4),
                           "bytes_model": "the bytes this plan's kernels need (plan flags below)",
                           "update_kernel_gbs": round(k2_gbs, 1),
                           "const_diag_folded": const_diag,
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
        "strong_768": strong,
        "cpu_baseline": cpu,
        "clocks": clocks,
    }
    log(f"solve {ms:.3f} ms (min {min(step_ms):.3f}); K1 {k1_avg*1e3:.1f} us = {k1_gbs:.0f} GB/s; "
        f"K2 {k2_avg*1e3:.1f} us = {k2_gbs:.0f} GB/s; solve {solve_gbs:.0f} GB/s "
        f"({solve_gbs/hbm_peak:.1%}); e2e {e2e_ms:.2f} ms (latency {lat_ms:.2f}); syncs {syncs}")
    print(json.dumps(out), flush=True)
    ctx.close()


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawTextHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["rvk", "reference"], default="rvk")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="7pt256")
    ap.add_argument("--mode", choices=["fused", "unfused", "persistent", "auto", "hostsync"],
                    default="auto", help="auto: the one-cluster solve for <= 8 K rows, the one-launch "
                                         "grid solve up to 148 x 8 K rows, else the fused "
                                         "2-kernel/iteration graph")
    ap.add_argument("--operator", choices=["csr", "stencil"], default="csr",
                    help="csr: the AIJ/CSR operator (headline); stencil: matrix-free (SURVEY 8f)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--opts", type=int, default=0,
                    help="rvk_cg_config.opts bits (include/rvk.h RVK_OPT_*), for A/B runs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-strong", action="store_true",
                    help="skip the 768^3 strong-scaling section (BASELINE configs[4])")
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
