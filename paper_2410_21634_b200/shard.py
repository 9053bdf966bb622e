"""Seed sharding across GPUs and the final result gather.

Per-seed solves are independent, so the
multi-GPU layout is: the graph replicated in every GPU's HBM, the seed batch
dealt round-robin (sample_sources orders seeds by degree bucket, so dealing
balances cost), no collective during the solve, and one gather at the end.

The gather moves per-seed counters and the sparse x of every seed with two
collectives: an all_gather of per-rank sizes, then an all_gather of payloads
padded to the largest rank (NCCL over NVLink/NVSwitch on GPUs, gloo on CPU).
"""

from __future__ import annotations

import numpy as np

__all__ = ["shard_seeds", "gather_results", "STAT_FIELDS"]

STAT_FIELDS = ("sweeps", "total_ops", "pushes", "converged", "x_offset", "x_count")


def shard_seeds(seeds, rank: int, world: int) -> np.ndarray:
    """Round-robin deal of the (degree-ordered) seed list: seed i -> rank i % world."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return np.asarray(seeds, dtype=np.int64)[rank::world]


def gather_results(stats: dict, x_nodes, x_vals, group=None, device=None,
                   dst: int | None = 0, to_host: bool = True) -> dict | None:
    """Gather per-seed results of all ranks (round-robin order restored).

    stats: dict of per-seed tensors (STAT_FIELDS, int64 / int32), x_nodes
    (int32) / x_vals (float64) the rank's sparse x pool.  With dst=None every
    rank receives everything (all_gather); otherwise only rank dst does
    (gather) and the others return None.  The result is a dict of numpy
    arrays in global seed order with x_offset rebased into the concatenated
    pool.  to_host=False keeps the result on the receiving device (torch
    tensors, nothing copied to the host: the form a GPU pipeline consumes).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = device if device is not None else x_vals.device
    k = int(stats["sweeps"].numel())
    sizes = torch.tensor([k, int(x_vals.numel())], dtype=torch.int64, device=dev)
    all_sizes = [torch.empty_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    all_sizes = torch.stack(all_sizes).cpu().numpy()
    kmax, xmax = int(all_sizes[:, 0].max()), int(all_sizes[:, 1].max())

    st = torch.zeros((len(STAT_FIELDS), kmax), dtype=torch.int64, device=dev)
    for i, f in enumerate(STAT_FIELDS):
        st[i, :k] = stats[f].to(device=dev, dtype=torch.int64)
    xn = torch.zeros(xmax, dtype=torch.int32, device=dev)
    xv = torch.zeros(xmax, dtype=torch.float64, device=dev)
    xn[:x_nodes.numel()] = x_nodes.to(device=dev, dtype=torch.int32)
    xv[:x_vals.numel()] = x_vals.to(device=dev)
    me = dist.get_rank(group)
    if dst is None or me == dst:
        g_st = [torch.empty_like(st) for _ in range(world)]
        g_xn = [torch.empty_like(xn) for _ in range(world)]
        g_xv = [torch.empty_like(xv) for _ in range(world)]
    else:
        g_st = g_xn = g_xv = None
    if dst is None:
        dist.all_gather(g_st, st, group=group)
        dist.all_gather(g_xn, xn, group=group)
        dist.all_gather(g_xv, xv, group=group)
    else:
        dist.gather(st, g_st, dst=dst, group=group)
        dist.gather(xn, g_xn, dst=dst, group=group)
        dist.gather(xv, g_xv, dst=dst, group=group)
        if me != dst:
            return None

    total = int(all_sizes[:, 0].sum())
    if not to_host:  # assemble on the device
        stats_d = torch.empty((len(STAT_FIELDS), total), dtype=torch.int64, device=dev)
        nodes_d, vals_d, base = [], [], 0
        for r in range(world):
            kr, xr = int(all_sizes[r, 0]), int(all_sizes[r, 1])
            s_r = g_st[r][:, :kr].clone()
            s_r[STAT_FIELDS.index("x_offset")] += base
            stats_d[:, r::world] = s_r
            nodes_d.append(g_xn[r][:xr])
            vals_d.append(g_xv[r][:xr])
            base += xr
        out = {f: stats_d[i] for i, f in enumerate(STAT_FIELDS)}
        out["converged"] = out["converged"].to(torch.bool)
        out["x_nodes"] = torch.cat(nodes_d) if nodes_d else torch.empty(0, dtype=torch.int32, device=dev)
        out["x_vals"] = torch.cat(vals_d) if vals_d else torch.empty(0, dtype=torch.float64, device=dev)
        return out
    out = {f: np.empty(total, dtype=np.int64) for f in STAT_FIELDS}
    nodes, vals, base = [], [], 0
    for r in range(world):
        kr, xr = int(all_sizes[r, 0]), int(all_sizes[r, 1])
        s_r = g_st[r][:, :kr].cpu().numpy()
        for i, f in enumerate(STAT_FIELDS):
            out[f][r::world] = s_r[i] + (base if f == "x_offset" else 0)
        nodes.append(g_xn[r][:xr].cpu().numpy())
        vals.append(g_xv[r][:xr].cpu().numpy())
        base += xr
    out["x_nodes"] = (np.concatenate(nodes) if nodes else np.empty(0, np.int32)).astype(np.int64)
    out["x_vals"] = np.concatenate(vals) if vals else np.empty(0)
    out["converged"] = out["converged"].astype(bool)
    return out
