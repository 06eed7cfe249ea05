"""GPU tests of the trace (include/rvk.h rvk_trace_*; reference
trace.hpp:11-46): a traced Jacobi-CG solve records its plan setup and solve
as device-timed Task events, every counted host wait as a HostSync event
(one per rvk_host_sync_count increment), cross-context edges as Wait
events; nothing is recorded while tracing is off; the C++ API's launches
are traced by tests/cpp/test_api.cpp (run by test_gpu_api.py)."""
import json

import numpy as np
import pytest

import oracle as O
from paper_2306_17801_b200 import rvk

pytestmark = pytest.mark.gpu


@pytest.fixture
def tracing():
    rvk.trace.clear()
    rvk.trace.enable(True)
    yield rvk.trace
    rvk.trace.enable(False)
    rvk.trace.clear()


def test_traced_solve_tasks_and_host_syncs(ctx, tracing, tmp_path):
    A = rvk.DeviceCsr.laplacian(ctx, 3, 7, (64, 64, 64))
    b = rvk.DeviceArray.from_host(ctx, O.rhs(A.n_rows))
    x = rvk.DeviceArray(A.n_rows)
    ctx.synchronize()
    tracing.clear()
    s0 = rvk.host_syncs()
    plan = rvk.CgPlan(ctx, A, max_it=20)
    tracing.marker("solves")
    for _ in range(3):
        plan.solve_dev(b, x)     # first call captures the graph, then replays
    res = plan.result()
    assert res.iterations == 20
    ev = tracing.events(str(tmp_path / "solve.jsonl"))
    syncs = rvk.host_syncs() - s0
    kinds = [e["kind"] for e in ev]
    assert kinds.count("host_sync") == syncs >= 1
    assert [e["label"] for e in ev if e["kind"] == "host_sync"][-1] == "rvk_cg_result"
    solves = [e for e in ev if e["label"] == "cg.solve"]
    assert len(solves) == 3
    for e in solves:
        assert e["device_timed"] and e["end"] > e["start"] and e["ctx"] == ctx.id
    # stream order: solve k+1 starts on the GPU after solve k ended
    solves.sort(key=lambda e: e["enqueue_seq"])
    for a, c in zip(solves, solves[1:]):
        assert c["start"] >= a["end"] - 2000
    # a 64^3 20-iteration solve takes tens of microseconds to a few ms on the GPU
    d = [(e["end"] - e["start"]) * 1e-6 for e in solves[1:]]
    assert all(0.005 < t < 50 for t in d), d
    creates = [e for e in ev if e["label"] == "cg.plan_create"]
    assert len(creates) == 1 and creates[0]["device_timed"]
    # the plan's setup syncs happened inside the plan_create task (host clock)
    marker = [e for e in ev if e["kind"] == "marker"]
    assert len(marker) == 1 and marker[0]["label"] == "solves"
    plan.close()


def test_wait_edges_and_vec_tasks(ctx, tracing, tmp_path):
    c2 = rvk.Ctx()
    c2.set_name("second")
    n = 1 << 20
    v = rvk.DeviceArray.from_host(ctx, np.ones(n))
    out = rvk.DeviceArray(1)
    ctx.synchronize()
    tracing.clear()
    L = rvk.lib()
    rvk.check(L.rvk_scale(ctx.h, n, rvk.scalar_const(3.0), v.ptr))
    c2.wait_for(ctx)
    rvk.check(L.rvk_nrm2(c2.h, n, v.ptr, out.ptr))
    c2.synchronize()
    ev = tracing.events(str(tmp_path / "vec.jsonl"))
    tasks = [e for e in ev if e["kind"] == "task"]
    assert [e["label"] for e in tasks] == ["rvk_scale", "rvk_nrm2"]
    assert tasks[1]["ctx"] == c2.id and tasks[1]["ctx_name"] == "second"
    assert tasks[1]["start"] >= tasks[0]["end"] - 2000   # the wait edge ordered them
    waits = [e for e in ev if e["kind"] == "wait"]
    assert len(waits) == 1 and waits[0]["ctx"] == c2.id
    assert abs(out.download(ctx)[0] - 3.0 * np.sqrt(n)) < 1e-9
    tracing.write_chrome(str(tmp_path / "vec.json"))
    doc = json.load(open(tmp_path / "vec.json"))
    rows = {e["args"]["name"] for e in doc["traceEvents"] if e.get("ph") == "M"}
    assert f"ctx {c2.id} (second)" in rows and "host" in rows
    c2.close()


def test_trace_off_records_nothing(ctx):
    rvk.trace.enable(False)
    rvk.trace.clear()
    A = rvk.DeviceCsr.laplacian(ctx, 2, 5, (32, 32))
    plan = rvk.CgPlan(ctx, A, max_it=5)
    plan.solve_host(O.rhs(A.n_rows))
    plan.close()
    assert rvk.trace.count() == 0
