"""Per-solve cost of the row-sharded PEER kernels on ONE GPU: P shards of a
256^3 7-point grid with every window on this device, solved phase by phase
(rvk_dcg_loopback_solve: each shard's kernels use the whole GPU in turn, so
the sum over shards is directly comparable with the single-GPU plan on the
same grid).  The difference is what the PEER machinery costs per GPU
(halo-plane stores, partial broadcast, flag release/acquire, system-scope
fences) -- everything except the NVLink hop itself."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2306_17801_b200 import rvk  # noqa: E402
from paper_2306_17801_b200.sharded import ShardPlan, partition, local_laplacian  # noqa: E402

g = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "256x256x256").split("x"))
stream = torch.cuda.Stream()
ctx = rvk.Ctx(stream.cuda_stream)
n = int(np.prod(g))


def timed(fn, k=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(k):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


A = rvk.DeviceCsr.laplacian(ctx, 3, 7, g)
b, x = rvk.DeviceArray(n), rvk.DeviceArray(n)
rvk.check(rvk.lib().rvk_fill_rhs(ctx.h, 0x9E3779B97F4A7C15, n, b.ptr))
cp = rvk.CgPlan(ctx, A, max_it=20)
t_cg = timed(lambda: cp.solve_dev(b, x))
print(f"grid {g}: single-GPU fused CG plan {t_cg:.3f} ms/solve")
cp.close()
del A

for P in (1, 2, 4):
    for backend in ("peer", "gather"):
        shards = partition(3, g, P)
        gather = None
        if backend == "gather" and P > 1:
            gather = rvk.DeviceArray(4 * P)
            rvk.check(rvk.lib().rvk_set(ctx.h, 4 * P, 0.0, gather.ptr))
        mats = [local_laplacian(ctx, 3, 7, g, s) for s in shards]
        plans = [ShardPlan(ctx, mats[i], s, 20, "jacobi", 0.0, 0.0, None,
                           gather.ptr if gather is not None else None) for i, s in enumerate(shards)]
        if backend == "peer" and P > 1:
            wins = [p.window()[0] for p in plans]
            for p in plans:
                p.attach_peers(wins, shards)
        bs = [rvk.DeviceArray(s.n_own) for s in shards]
        for s, bb in zip(shards, bs):
            rvk.check(rvk.lib().rvk_fill_rhs(ctx.h, (0x9E3779B97F4A7C15 + s.row_begin) % 2**64, s.n_own, bb.ptr))
        xs = [rvk.DeviceArray(s.n_own) for s in shards]
        Pa = (C.c_void_p * P)(*[p.h.value for p in plans])
        Ba = (C.c_void_p * P)(*[v.ptr for v in bs])
        Xa = (C.c_void_p * P)(*[v.ptr for v in xs])
        t = timed(lambda: rvk.check(rvk.lib().rvk_dcg_loopback_solve(Pa, P, Ba, Xa)))
        flags = rvk.lib().rvk_dcg_plan_flags(plans[0].h)
        print(f"P={P} {backend:6s}: {t:.3f} ms/solve summed over shards "
              f"(+{100 * (t / t_cg - 1):.1f}% vs the single-GPU plan; flags {flags})")
        for p in plans:
            p.close()
        del plans, mats, bs, xs
        torch.cuda.synchronize()
