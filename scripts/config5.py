"""Config 5 as PAPER.md:537 / SURVEY 8(d) specify it: an arxiv-shape graph split
into snapshots -- G0 holds the first 17.9 % of the edges (R-MAT generation order),
then 16 snapshots each insert the next ~59 K edges (plus, optionally, delete a
fraction of existing ones) -- with K PPR pairs maintained by warm-started repair.

GPU: PairPool, both repair methods -- "push" (the reference's own repair,
bit-identical per pair) and "gd" (warm signed LocalGD, sweep-synchronous).
CPU: the reference loop of run_snapshots (src/dynamic.py:165-196) on the host
cores -- event_adjust per event (host, bitwise), the snapshot graph, and the
reference repair (oracle/ C port of _push_kernel) per source -- for a sample of
the sources; per-snapshot sweeps / ops of those sources are compared with the
GPU "push" pool (they must be identical).  Also the static re-solve ops (make_pair
+ repair per snapshot) for the dynamic-vs-static ratio.

usage: python scripts/config5.py [K] [cpu_sources] [delete_frac]
Prints one JSON line.  Measurement script (uses the oracle as the CPU side).
"""
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from bench import SHAPES  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2410_21634_b200 import systems as S  # noqa: E402
from paper_2410_21634_b200.dynamic import PairPool, event_adjust_many, make_pair  # noqa: E402
from paper_2410_21634_b200.graph import EdgeEvent, apply_events, csr_from_pairs  # noqa: E402
from paper_2410_21634_b200.metrics import sample_sources  # noqa: E402
from paper_2410_21634_b200.synth import rmat_edge_order  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
CPU_SOURCES = int(sys.argv[2]) if len(sys.argv) > 2 else 32
DEL = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
G0_FRAC, SNAPS = 0.179, 16
alpha, eps_target = 0.1, 1e-6
eps = alpha * eps_target  # pair eps (tests/test_acceptance.py:184)

n, m = SHAPES["arxiv"]
keys = rmat_edge_order(n, m, seed=0)  # undirected keys min*n+max, generation order
m0 = int(round(G0_FRAC * m))
g0 = csr_from_pairs(n, np.stack([keys[:m0] // n, keys[:m0] % n], axis=1))
rest = keys[m0:]
chunks = np.array_split(rest, SNAPS)
rng = np.random.default_rng(7)
batches, sim = [], g0
for c in chunks:
    b = [EdgeEvent("insert", int(k // n), int(k % n)) for k in c]
    if DEL > 0:  # delete existing edges (present before this snapshot)
        src = np.repeat(np.arange(n), sim.degrees)
        fw = src < sim.targets
        pairs = np.stack([src[fw], sim.targets[fw]], axis=1)
        pick = rng.choice(pairs.shape[0], int(DEL * len(c)), replace=False)
        b += [EdgeEvent("delete", int(u), int(v)) for u, v in pairs[pick]]
    sim = apply_events(sim, b)
    batches.append(b)
sources = sample_sources(g0, K, seed=0)
# sources must keep a neighbour in G0 (they do: sample_sources picks degree > 0)

out = {"workload": f"config 5: arxiv-shape R-MAT ({n:,} nodes, {m:,} edges), G0 = first "
                   f"{G0_FRAC:.1%} of the edges ({m0:,}), {SNAPS} snapshots of ~{len(chunks[0]):,} "
                   f"insertions" + (f" + {DEL:.0%} deletions" if DEL else "") +
                   f", {K} PPR pairs alpha={alpha} eps_pair={eps:g}",
       "pairs": K, "snapshots": SNAPS}

# ---- GPU: resident pairs, both repair methods ------------------------------
import torch  # noqa: E402

for method in ("push", "gd"):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pool = PairPool(g0, sources, alpha, eps, method=method)
    t_create = time.perf_counter() - t0
    stats, walls, kms = [], [], []
    for b in batches:
        t = time.perf_counter()
        stats.append(pool.update(b))
        walls.append(time.perf_counter() - t)
        kms.append(pool.last_kernel_ms)
    pool.close()
    ops = int(sum(int(s["total_ops"].sum()) for s in stats))
    out[f"gpu_{method}"] = {
        "pair_updates_per_s": K * SNAPS / sum(walls),
        "ms_per_snapshot": 1e3 * sum(walls) / SNAPS,
        "repair_kernel_ms_per_snapshot": sum(kms) / SNAPS,
        "initial_solve_s": t_create, "ops_total": ops,
        "timing": "host wall clock per update (device graph edit + event adjustment + repair + stats)"}
    if method == "push":
        push_stats = stats

# ---- CPU: the reference loop per source (oracle repair), host cores ----------
threads = len(os.sched_getaffinity(0))
sample = sources[:: max(1, K // CPU_SOURCES)][:CPU_SOURCES]
idx = [int(np.flatnonzero(sources == s)[0]) for s in sample]
graphs = [g0]
for b in batches:
    graphs.append(apply_events(graphs[-1], b))
arrays = [(S.arc_weights_for(g, 1.0 - alpha, "gen", 0.0), S.theta_vector(g, eps)) for g in graphs]


def repair_cpu(g, w, th, pair):
    p, r = pair.p.copy(), pair.r.copy()
    seeds = np.flatnonzero(np.abs(r) >= th)
    rep = O.push_kernel(g.offsets, g.targets, w, th, p, r, seeds, omega=1.0, x_gain=1.0,
                        signed=True)
    return p, r, rep


def one_source(s):
    pair = make_pair(g0, alpha, eps, int(s))
    p, r, rep = repair_cpu(g0, *arrays[0], pair)
    pair.p, pair.r = p, r
    res = []
    for i, b in enumerate(batches):
        pair = event_adjust_many(graphs[i], pair, b)
        p, r, rep = repair_cpu(graphs[i + 1], *arrays[i + 1], pair)
        pair.p, pair.r = p, r
        res.append((int(rep["sweeps"]), int(rep["total_ops"])))
    return res


t0 = time.perf_counter()
with ThreadPoolExecutor(threads) as ex:
    cpu = list(ex.map(one_source, sample))
wall = time.perf_counter() - t0
same = all(cpu[j][i] == (int(push_stats[i]["sweeps"][idx[j]]), int(push_stats[i]["total_ops"][idx[j]]))
           for j in range(len(sample)) for i in range(SNAPS))
# static re-solves (make_pair + repair on every snapshot graph) for the ops ratio
static_ops = 0
dyn_ops = sum(o for row in cpu for _, o in row)
for s in sample[:8]:
    for i in range(SNAPS):
        _, _, rep = repair_cpu(graphs[i + 1], *arrays[i + 1], make_pair(graphs[i + 1], alpha, eps, int(s)))
        static_ops += int(rep["total_ops"])
dyn8 = sum(o for row in cpu[:8] for _, o in row)
out["cpu_reference_loop"] = {
    "pair_updates_per_s": len(sample) * SNAPS / wall, "sources": len(sample), "threads": threads,
    "kind": "port (event_adjust host + oracle/ _push_kernel repair, one source per thread)"}
out["gpu_push_sweeps_ops_identical_to_cpu"] = bool(same)
out["dynamic_vs_static_ops"] = {"static_ops": static_ops, "dynamic_ops": dyn8,
                                "ratio": static_ops / max(dyn8, 1), "sources": min(8, len(sample))}
for mth in ("push", "gd"):
    out[f"speedup_gpu_{mth}_vs_cpu"] = out[f"gpu_{mth}"]["pair_updates_per_s"] / out["cpu_reference_loop"]["pair_updates_per_s"]
print(json.dumps(out))
