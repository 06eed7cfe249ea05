"""Traced Jacobi-CG run (rvk_trace_*, reference trace.hpp:11-46): plan setup,
3 solves of the 256^3 7-point system and the result read, plus a two-context
vector pipeline with a wait edge.  Writes the JSONL event log, a Chrome
trace-event timeline (chrome://tracing / Perfetto) and the event summary to
the directory given (default profiles/r02)."""
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2306_17801_b200 import rvk  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "profiles/r02"
os.makedirs(out, exist_ok=True)
ctx = rvk.Ctx()
ctx.set_name("solver")
rvk.trace.clear()
rvk.trace.enable(True)
g = (256, 256, 256)
A = rvk.DeviceCsr.laplacian(ctx, 3, 7, g)
n = A.n_rows
b, x = rvk.DeviceArray(n), rvk.DeviceArray(n)
rvk.check(rvk.lib().rvk_fill_rhs(ctx.h, 0x9E3779B97F4A7C15, n, b.ptr))
plan = rvk.CgPlan(ctx, A, max_it=20)
rvk.trace.marker("solves")
for _ in range(3):
    plan.solve_dev(b, x)
res = plan.result()
c2 = rvk.Ctx()
c2.set_name("post")
rvk.trace.marker("two-context pipeline")
L = rvk.lib()
nrm = rvk.DeviceArray(1)
rvk.check(L.rvk_scale(ctx.h, n, rvk.scalar_const(2.0), x.ptr))
c2.wait_for(ctx)
rvk.check(L.rvk_nrm2(c2.h, n, x.ptr, nrm.ptr))
c2.synchronize()
rvk.trace.write_jsonl(os.path.join(out, "trace_7pt256.jsonl"))
rvk.trace.write_chrome(os.path.join(out, "trace_7pt256_chrome.json"))
ev = [json.loads(l) for l in open(os.path.join(out, "trace_7pt256.jsonl"))]
summ = collections.OrderedDict()
for e in ev:
    k = (e["kind"], e["label"])
    d = summ.setdefault(k, [0, 0.0, 0])
    d[0] += 1
    d[1] += (e["end"] - e["start"]) * 1e-6
    d[2] += int(e.get("device_timed", False))
with open(os.path.join(out, "trace_7pt256_summary.txt"), "w") as f:
    f.write(f"{len(ev)} events; iterations {res.iterations}; host syncs {rvk.host_syncs()}\n")
    for (kind, label), (cnt, ms, dev) in summ.items():
        f.write(f"{kind:9s} {label:28s} n={cnt:3d} total={ms:9.3f} ms device_timed={dev}\n")
print(open(os.path.join(out, "trace_7pt256_summary.txt")).read())
rvk.trace.enable(False)
