"""Config 5 batched: K resident PPR pairs maintained over a stream of
edge-insertion snapshots (PairPool: event adjustment + warm-started signed
LocalGD repair of every pair per snapshot) vs the reference's per-source
loop (event_adjust + signed FIFO repair, src/dynamic.py:110-196) on all
host cores.  Sweeps / ops of the GPU pairs are checked against the oracle's
warm LocalGD on the first snapshot for a sample of pairs.

usage: python scripts/pool_config.py [shape] [pairs] [snapshots] [events] [cpu_pairs]"""
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from bench import SHAPES
from oracle import oracle as O
from paper_2410_21634_b200 import systems as S
from paper_2410_21634_b200.dynamic import PairPool, event_adjust_many, make_pair
from paper_2410_21634_b200.gen import rmat_csr_device
from paper_2410_21634_b200.graph import CsrGraph, EdgeEvent, apply_events
from paper_2410_21634_b200.metrics import sample_sources

shape = sys.argv[1] if len(sys.argv) > 1 else "arxiv"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
snaps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
n_ev = int(sys.argv[4]) if len(sys.argv) > 4 else 1000
cpu_pairs = int(sys.argv[5]) if len(sys.argv) > 5 else 64
alpha, eps = 0.15, 0.15 * 1e-6
n, m = SHAPES[shape]
row, col = rmat_csr_device(n, m, seed=0)
g0 = CsrGraph(n=n, offsets=row.cpu().numpy(), targets=col.cpu().numpy().astype(np.int64))
rng = np.random.default_rng(1)
batches, sim, sims = [], g0, [g0]
for _ in range(snaps + 1):  # insertion snapshots (the first is a warm-up)
    b, seen = [], set()
    while len(b) < n_ev:
        u, v = sorted(rng.integers(0, n, 2).tolist())
        if u == v or (u, v) in seen or sim.has_edge(u, v):
            continue
        seen.add((u, v))
        b.append(EdgeEvent("insert", u, v))
    sim = apply_events(sim, b)
    batches.append(b)
    sims.append(sim)
sources = sample_sources(g0, K, seed=0)
threads = os.cpu_count() or 1

torch.cuda.synchronize()
t0 = time.perf_counter()
pool = PairPool(g0, sources, alpha, eps)
t_create = time.perf_counter() - t0
cold_ops = int(pool.last["total_ops"].sum())
warm = batches.pop(0)  # warm-up snapshot: the second device graph gets allocated here
pool.update(warm)
graphs = sims[1:]  # host copies of the snapshots (built with graph.apply_events above)
g0 = graphs[0]
walls, kms, ops = [], [], []
first_state = [pool.pair(i) for i in range(min(cpu_pairs, K))]
import gc

gc.collect()
gc.disable()  # (a collection of the batch generator's objects is not update work)
for b in batches:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = pool.update(b)
    walls.append(time.perf_counter() - t0)
    kms.append(pool.last_kernel_ms)
    ops.append(int(st["total_ops"].sum()))
    if len(walls) == 1:
        first_stats = {k: v.copy() for k, v in st.items()}

gc.enable()
# parity on snapshot 1 for the CPU sample: oracle warm LocalGD from the same state
k = len(first_state)
g1 = graphs[1]
w1 = S.arc_weights_for(g1, 1.0 - alpha, "gen", 0.0)
th1 = S.theta_vector(g1, eps)
same = True
for i in range(k):
    adj = event_adjust_many(g0, first_state[i], batches[0])
    ref = O.local_gd_warm(g1.offsets, g1.targets, w1, th1, adj.p.copy(), adj.r.copy(), signed=True,
                          record_trace=False)
    same &= bool(ref["sweeps"] == first_stats["sweeps"][i] and ref["total_ops"] == first_stats["total_ops"][i])

# CPU: the reference's per-source loop (event_adjust + signed FIFO repair)
w0 = S.arc_weights_for(g0, 1.0 - alpha, "gen", 0.0)


def cpu_source(i):
    pair = make_pair(g0, alpha, eps, int(sources[i]))
    th = S.theta_vector(g0, eps)
    O.push_kernel(g0.offsets, g0.targets, w0, th, pair.p, pair.r, np.flatnonzero(np.abs(pair.r) >= th),
                  signed=True)
    t0 = time.perf_counter()
    ops = 0
    for j, b in enumerate(batches):
        pair = event_adjust_many(graphs[j], pair, b)
        gj = graphs[j + 1]
        wj = S.arc_weights_for(gj, 1.0 - alpha, "gen", 0.0)
        thj = S.theta_vector(gj, eps)
        out = O.push_kernel(gj.offsets, gj.targets, wj, thj, pair.p, pair.r,
                            np.flatnonzero(np.abs(pair.r) >= thj), signed=True)
        ops += out["total_ops"]
    return time.perf_counter() - t0, ops


t0 = time.perf_counter()
with ThreadPoolExecutor(threads) as ex:
    res = list(ex.map(cpu_source, range(k)))
t_cpu = time.perf_counter() - t0
pair_updates_gpu = K * snaps / sum(walls)
pair_updates_cpu = k * snaps / t_cpu
print(json.dumps({
    "case": f"{shape} pair pool K={K} snapshots={snaps} x {n_ev} insertions alpha={alpha} eps={eps:g}",
    "create_s": round(t_create, 3), "cold_ops": cold_ops,
    "update_wall_ms": [round(w * 1e3, 2) for w in walls], "update_kernel_ms": [round(x, 2) for x in kms],
    "repair_ops": ops, "ops_ratio_static_over_dynamic": round(cold_ops / max(np.mean(ops), 1), 2),
    "gpu_pair_updates_per_s": round(pair_updates_gpu, 1),
    "gpu_pair_updates_per_s_kernel_only": round(K * snaps / (sum(kms) / 1e3), 1),
    "cpu_pair_updates_per_s": round(pair_updates_cpu, 2), "cpu_threads": threads, "cpu_sample": k,
    "cpu_note": "reference loop: event_adjust + signed FIFO push (oracle port), includes host graph rebuild per source",
    "speedup": round(pair_updates_gpu / pair_updates_cpu, 1),
    "snapshot1_sweeps_ops_identical_to_oracle_warm_gd": same,
}), flush=True)
