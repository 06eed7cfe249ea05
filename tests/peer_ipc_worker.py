"""Worker for tests/test_gpu_peer_ipc.py (run under torchrun, gloo group).

Every rank is a separate PROCESS; all of them may sit on the same GPU (the
1-GPU test box: contexts time-slice, so the flag waits see real cross-process
concurrency) or on one GPU each.  Each rank builds its shard, exports its
PEER window through cudaIpc, maps the others' windows, solves `repeats`
times and rank 0 checks the gathered solution against the CPU oracle.
Prints one JSON line on rank 0.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    from paper_2306_17801_b200 import rvk
    from paper_2306_17801_b200.sharded import (ShardPlan, connect_peers, disconnect_peers,
                                               local_laplacian, partition)

    dim, pts = int(sys.argv[1]), int(sys.argv[2])
    grid = tuple(int(v) for v in sys.argv[3].split("x"))
    max_it, rtol, repeats = int(sys.argv[4]), float(sys.argv[5]), int(sys.argv[6])
    one_gpu = len(sys.argv) > 7 and sys.argv[7] == "shared"
    use_graph = len(sys.argv) > 8 and sys.argv[8] == "graph"  # the solve as one replayed CUDA graph
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = 0 if one_gpu else int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    ctx = rvk.Ctx()
    shards = partition(dim, grid, world)
    sh = shards[rank]
    A = local_laplacian(ctx, dim, pts, grid, sh)
    plan = ShardPlan(ctx, A, sh, max_it, rtol=rtol, use_graph=use_graph)
    opened = connect_peers(plan, shards, rank, world)
    b = rvk.DeviceArray(sh.n_own)
    x = rvk.DeviceArray(sh.n_own)
    seed = 0x9E3779B97F4A7C15
    rvk.check(rvk.lib().rvk_fill_rhs(ctx.h, (seed + sh.row_begin) & (2 ** 64 - 1), sh.n_own, b.ptr))
    hists = []
    for _ in range(repeats):
        plan.solve_dev(b, x)
        hists.append(plan.result().hist)
    res = plan.result()
    xs = x.download(ctx)
    out = [None] * world
    dist.all_gather_object(out, (res.state, res.iterations, [h.tolist() for h in hists], xs.tobytes()))
    dist.barrier()  # nobody frees its window while a peer may still store into it
    plan.close()
    disconnect_peers(opened)
    if rank == 0:
        import oracle as O

        Ah = O.build_laplacian(dim, pts, grid)
        ref = O.cg_solve(Ah, O.rhs(Ah.n_rows), max_it=max_it, rtol=rtol)
        xg = np.concatenate([np.frombuffer(o[3], np.float64) for o in out])
        h0 = np.array(out[0][2][-1])
        same = all(np.array_equal(np.array(h), h0) for o in out for h in o[2])
        print(json.dumps({
            "states": [o[0] for o in out], "iterations": [o[1] for o in out],
            "ref_iterations": ref.iterations,
            "hist_rel": float(np.max(np.abs(h0 - ref.hist) / ref.hist)),
            "x_rel": float(np.linalg.norm(xg - ref.x) / np.linalg.norm(ref.x)),
            "all_ranks_and_repeats_identical": bool(same)}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
