"""One plane-marching CG solve on a 3D 7-point grid (argv: nx ny nz [opts]),
checked against the row-order plan: used under compute-sanitizer."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2306_17801_b200 import rvk
import oracle as O

nx, ny, nz = (int(v) for v in sys.argv[1:4])
opts = int(sys.argv[4]) if len(sys.argv) > 4 else rvk.OPT_MARCH
ctx = rvk.Ctx()
A = rvk.DeviceCsr.laplacian(ctx, 3, 7, (nx, ny, nz))
b = O.rhs(A.n_rows)
p1 = rvk.CgPlan(ctx, A, max_it=4, opts=opts)
print("flags", p1.flags(), "march", bool(p1.flags() & rvk.PLAN_MARCH))
x1, r1 = p1.solve_host(b)
p0 = rvk.CgPlan(ctx, A, max_it=4, opts=0)
x0, r0 = p0.solve_host(b)
print("hist rel", np.max(np.abs(r1.hist - r0.hist) / r0.hist), "x rel",
      np.linalg.norm(x1 - x0) / np.linalg.norm(x0))
