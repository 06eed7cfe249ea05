"""Single-GPU plan vs one row-shard (P = 1 loopback, the shard kernels on
the same 256^3 7-point system): times both K1s with CUDA events and runs
each solve a few times so `ncu` can capture one K1 of each
(scripts/gpu_shard_gap.sh).  VERDICT r1 weak #3 / next #6."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402
import numpy as np  # noqa: E402

from paper_2306_17801_b200 import rvk  # noqa: E402
from paper_2306_17801_b200.sharded import ShardPlan, partition, local_laplacian  # noqa: E402

g = (256, 256, 256)
n = int(np.prod(g))
ctx = rvk.Ctx()
A = rvk.DeviceCsr.laplacian(ctx, 3, 7, g)
b, x = rvk.DeviceArray(n), rvk.DeviceArray(n)
rvk.check(rvk.lib().rvk_fill_rhs(ctx.h, 0x9E3779B97F4A7C15, n, b.ptr))
cp = rvk.CgPlan(ctx, A, max_it=20)
for _ in range(3):
    cp.solve_dev(b, x)
ctx.synchronize()
cp.set_profiling(True)
cp.solve_dev(b, x)
ctx.synchronize()
k1, k2, nk = cp.kernel_times()
print(f"single-GPU plan: K1 avg {k1/20*1e3:.1f} us  K2 avg {k2/20*1e3:.1f} us", flush=True)
cp.close()
sh = partition(3, g, 1)[0]
M = local_laplacian(ctx, 3, 7, g, sh)
sp = ShardPlan(ctx, M, sh, 20, "jacobi", 0.0, 0.0, None, None)
P = (C.c_void_p * 1)(sp.h.value)
B = (C.c_void_p * 1)(b.ptr)
X = (C.c_void_p * 1)(x.ptr)
import torch  # noqa: E402
for _ in range(3):
    rvk.check(rvk.lib().rvk_dcg_loopback_solve(P, 1, B, X))
ctx.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s = torch.cuda.ExternalStream(ctx.stream)
e0.record(s)
for _ in range(5):
    rvk.check(rvk.lib().rvk_dcg_loopback_solve(P, 1, B, X))
e1.record(s)
torch.cuda.synchronize()
print(f"shard plan (P=1): {e0.elapsed_time(e1)/5:.3f} ms/solve", flush=True)
