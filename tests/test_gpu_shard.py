"""The real batched solver in a 2-rank job (gloo, both ranks on cuda:0): every
rank solves its round-robin shard of the seed batch with BatchSolver and the
result gather reassembles them on rank 0 -- identical to one rank solving the
whole batch (the multi-GPU path of bench.py, without needing two
GPUs: the ranks do not wait on each other's kernels, only on the gather)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _graph():
    from paper_2410_21634_b200.metrics import sample_sources
    from paper_2410_21634_b200.synth import rmat_graph

    g = rmat_graph(20000, 150000, seed=5)
    return g, sample_sources(g, 48, seed=0)


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2410_21634_b200.batch import BatchSolver
    from paper_2410_21634_b200.shard import STAT_FIELDS, gather_results, shard_seeds

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    g, seeds = _graph()
    mine = shard_seeds(seeds, rank, world)
    os.environ["GDIFF_BATCH_MODE"] = "rounds"  # (the large-graph kernel)
    solver = BatchSolver(g, 0.1, 1e-6, slots=8)
    res = solver.solve_device(torch.as_tensor(mine, device="cuda"))
    stats = {f: res[f].cpu() for f in STAT_FIELDS}
    out = gather_results(stats, res["x_nodes"].cpu(), res["x_vals"].cpu(),
                         device=torch.device("cpu"), dst=0)
    if rank == 0:
        q.put({k: np.asarray(v).tolist() for k, v in out.items()})
    solver.close()
    dist.barrier()
    dist.destroy_process_group()


def test_real_solver_two_ranks_equals_one(gpu):
    import torch.multiprocessing as mp

    from paper_2410_21634_b200.batch import BatchSolver

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g, seeds = _graph()
    os.environ["GDIFF_BATCH_MODE"] = "rounds"
    try:
        one = BatchSolver(g, 0.1, 1e-6, slots=8).solve(seeds)
    finally:
        os.environ.pop("GDIFF_BATCH_MODE", None)
    for f in ("sweeps", "total_ops", "pushes", "x_count"):
        assert np.array_equal(np.asarray(got[f]), getattr(one, f)), f
    assert np.array_equal(np.asarray(got["converged"], bool), one.converged)
    nodes, vals = np.asarray(got["x_nodes"]), np.asarray(got["x_vals"])
    for i in range(len(seeds)):
        a, c = int(got["x_offset"][i]), int(got["x_count"][i])
        xg = np.zeros(g.n)
        xg[nodes[a:a + c]] = vals[a:a + c]
        x1 = one.x_dense(i, g.n)
        assert np.abs(xg - x1).sum() <= 1e-9 * np.abs(x1).sum()
