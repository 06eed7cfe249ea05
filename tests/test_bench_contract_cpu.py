"""CPU tests of bench.py's reference arm (the driver's `--impl reference`
launch): it runs the reference's own CPU kernels (oracle/_ref, test
infrastructure) on the GPU arm's workload, prints ONE JSON line with the
contract's keys, and a non-zero rank exits without work."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                          capture_output=True, text=True, env=e, timeout=600)


@pytest.fixture(scope="module")
def ref_line():
    import oracle as O
    if not O.ref_available():
        pytest.skip("oracle/_ref (the reference kernels) not built")
    p = _run(["--impl", "reference", "--config", "5pt1024", "--steps", "2", "--warmup", "0"])
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def test_reference_line_contract(ref_line):
    d = ref_line
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline",
              "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "ms/solve" and d["higher_is_better"] is False
    assert d["steps"] == 2 and d["value"] > 0
    assert d["e2e"] == {"value": d["value"], "unit": "ms/solve", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["kind"] in ("reference", "port") and cb["cores"] >= 1
    # the value is the fastest of the reference's backends
    assert min(cb["per_backend_ms"].values()) <= d["value"] * 1.5


def test_reference_config_matches_gpu_arm(ref_line):
    """Same workload keys as the GPU arm (the driver's same_config check)."""
    sys.path.insert(0, ROOT)
    import argparse

    import bench
    args = argparse.Namespace(config="5pt1024", gpus=1, impl="reference", operator="csr",
                              solver="cg", mode="auto", steps=2, warmup=0)
    assert ref_line["config"] == bench.bench_config(args, 1)
    assert ref_line["metric"] == bench.METRIC


def test_reference_nonzero_rank_exits_quietly():
    p = _run(["--impl", "reference", "--config", "5pt1024", "--steps", "1", "--warmup", "0"],
             env={"RANK": "1", "WORLD_SIZE": "2"})
    assert p.returncode == 0 and p.stdout.strip() == ""
