import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2306_17801_b200 import rvk
import oracle as O
ctx = rvk.Ctx()
for dim, pts, g in [(3, 7, (64, 24, 10)), (2, 5, (300, 37))]:
    Ah = O.build_laplacian(dim, pts, g); b = O.rhs(Ah.n_rows)
    p = rvk.CgPlan(ctx, (dim, pts, g), max_it=2)
    print("flags", p.flags())
    x, r = p.solve_host(b)
    print(dim, pts, g, r.hist)
