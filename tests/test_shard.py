"""Multi-rank host path on CPU: seed sharding + result gather over gloo,
world_size 2 (the NCCL path on GPUs runs the same code)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_21634_b200.shard import STAT_FIELDS, gather_results, shard_seeds


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _fake_solve(seeds):
    """Deterministic stand-in for a per-rank batch result."""
    k = len(seeds)
    counts = (seeds % 5) + 1
    off = np.concatenate([[0], np.cumsum(counts)[:-1]])
    nodes = np.concatenate([np.arange(c) + s for s, c in zip(seeds, counts)]) if k else np.empty(0)
    vals = np.concatenate([np.full(c, s * 0.5) for s, c in zip(seeds, counts)]) if k else np.empty(0)
    stats = {"sweeps": seeds % 7, "total_ops": seeds * 3, "pushes": seeds + 1,
             "converged": np.ones(k, np.int64), "x_offset": off, "x_count": counts}
    return stats, nodes, vals


def _worker(rank, world, port, seeds, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = shard_seeds(seeds, rank, world)
    stats, nodes, vals = _fake_solve(mine)
    args = ({f: torch.as_tensor(stats[f]) for f in STAT_FIELDS},
            torch.as_tensor(nodes, dtype=torch.int32), torch.as_tensor(vals))
    out = gather_results(*args, device=torch.device("cpu"), dst=0)
    both = gather_results(*args, device=torch.device("cpu"), dst=None)
    dev = gather_results(*args, device=torch.device("cpu"), dst=0, to_host=False)
    if rank == 0:
        assert all(np.array_equal(out[k], both[k]) for k in out)
        # the device-resident form (what bench.py keeps in rank 0's HBM) is the same data
        assert all(np.array_equal(out[k], dev[k].numpy()) for k in out)
        q.put({k: v.tolist() for k, v in out.items()})
    else:
        assert out is None and both is not None and dev is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("nseeds", [0, 7, 64])
def test_gather_world2_gloo(nseeds):
    seeds = np.arange(100, 100 + nseeds, dtype=np.int64)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, seeds, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref, rn, rv = _fake_solve(seeds)
    for f in ("sweeps", "total_ops", "pushes", "x_count"):
        assert out[f] == ref[f].tolist(), f
    for i, s in enumerate(seeds):
        a, c = out["x_offset"][i], out["x_count"][i]
        assert out["x_nodes"][a:a + c] == list(range(s, s + c))
        assert out["x_vals"][a:a + c] == [s * 0.5] * c


def test_shard_partition():
    seeds = np.arange(1000)
    parts = [shard_seeds(seeds, r, 8) for r in range(8)]
    assert sorted(np.concatenate(parts).tolist()) == seeds.tolist()
    assert max(map(len, parts)) - min(map(len, parts)) <= 1
    with pytest.raises(ValueError):
        shard_seeds(seeds, 8, 8)
