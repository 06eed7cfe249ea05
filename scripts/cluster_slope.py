"""Per-iteration vs fixed cost of the one-cluster solve (latency sweep grids)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch  # noqa: E402
from paper_2306_17801_b200 import rvk  # noqa: E402
stream = torch.cuda.Stream()
ctx = rvk.Ctx(stream.cuda_stream)
for g in ((64, 64), (128, 128)):
    n = g[0] * g[1]
    A = rvk.DeviceCsr.laplacian(ctx, 2, 5, g)
    b, x = rvk.DeviceArray(n), rvk.DeviceArray(n)
    rvk.check(rvk.lib().rvk_fill_rhs(ctx.h, 0x9E3779B97F4A7C15, n, b.ptr))
    out = []
    for mi in (1, 5, 20, 80):
        for mode in ("auto",):
            p = rvk.CgPlan(ctx, A, max_it=mi, mode=mode)
            for _ in range(5):
                p.solve_dev(b, x)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(50):
                p.solve_dev(b, x)
            e1.record(stream)
            torch.cuda.synchronize()
            out.append((mi, e0.elapsed_time(e1) / 50 * 1000))
            p.close()
    print(g, " ".join(f"it={m}: {t:.1f}us" for m, t in out),
          f"slope {(out[-1][1] - out[1][1]) / 75:.2f} us/it")
