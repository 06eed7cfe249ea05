"""Time the row-sharded kernels (rvk_dcg) as a single shard on one GPU, next to
the single-GPU fused CG plan, on the same 3D 7-point grid: the per-GPU cost of
the N>1 path without communication."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2306_17801_b200 import rvk
from paper_2306_17801_b200.sharded import ShardPlan, partition, local_laplacian

g = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "256x256x256").split("x"))
stream = torch.cuda.Stream()
ctx = rvk.Ctx(stream.cuda_stream)
sh = partition(3, g, 1)[0]
A = local_laplacian(ctx, 3, 7, g, sh)
b, x = rvk.DeviceArray(sh.n_own), rvk.DeviceArray(sh.n_own)
rvk.check(rvk.lib().rvk_fill_rhs(ctx.h, 0x9E3779B97F4A7C15, sh.n_own, b.ptr))


def timed(solve, k=10):
    for _ in range(3):
        solve()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(k):
        solve()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


if os.environ.get("CG_FIRST"):  # allocation-order control
    cp = rvk.CgPlan(ctx, A, max_it=20)
    t_cg = timed(lambda: cp.solve_dev(b, x))
dp = ShardPlan(ctx, A, sh, 20)
t_dcg = timed(lambda: dp.solve_dev(b, x))
if not os.environ.get("CG_FIRST"):
    cp = rvk.CgPlan(ctx, A, max_it=20)
    t_cg = timed(lambda: cp.solve_dev(b, x))
print(f"grid {g}: dcg single shard {t_dcg:.3f} ms/solve, fused CG plan {t_cg:.3f} ms/solve")

# the same dcg solve captured as one CUDA graph (launch overhead out of the picture)
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph, stream=stream):
    dp.solve_dev(b, x)
def replay():
    with torch.cuda.stream(stream):
        graph.replay()


t_g = timed(replay)
print(f"grid {g}: dcg single shard as a CUDA graph {t_g:.3f} ms/solve")
