"""PEER backend across PROCESSES (cudaIpc windows, system-scope flags).

The round's GPU box has one B200, so the ranks share it: each rank is its
own process with its own CUDA context, and the contexts time-slice -- a
rank's kernel spinning on a flag is preempted so the peer process can run
and release it.  That exercises everything the 8-GPU path does except the
NVLink hop itself: cudaIpc export/map of the windows, remote halo-plane and
partial stores into another process's allocation, the acquire/release flag
protocol under genuine cross-process concurrency, repeated solves and the
device-side early exit.  Bars as the single-GPU parity tests (1e-10)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run(world, dim, pts, grid, max_it=20, rtol=0.0, repeats=2):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", f"--master-port={free_port()}",
           os.path.join(ROOT, "tests", "peer_ipc_worker.py"), str(dim), str(pts),
           "x".join(map(str, grid)), str(max_it), repr(rtol), str(repeats), "shared"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    line = [ln for ln in p.stdout.splitlines() if ln.startswith("{")][-1]
    return json.loads(line)


@pytest.mark.parametrize("world,dim,pts,grid", [(2, 3, 7, (24, 20, 18)), (3, 2, 9, (40, 45)),
                                                (2, 3, 27, (12, 12, 16))])
def test_peer_ipc_processes_vs_oracle(world, dim, pts, grid):
    r = run(world, dim, pts, grid)
    assert r["states"] == [0] * world and r["iterations"] == [20] * world
    assert r["all_ranks_and_repeats_identical"]
    assert r["hist_rel"] < 1e-10 and r["x_rel"] < 1e-10


def test_peer_ipc_processes_early_exit():
    r = run(2, 2, 5, (32, 30), max_it=300, rtol=1e-6)
    assert r["states"] == [1, 1] and r["iterations"][0] == r["ref_iterations"]
    assert r["x_rel"] < 1e-10
