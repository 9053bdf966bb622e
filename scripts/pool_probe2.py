import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from bench import SHAPES
from paper_2410_21634_b200.dynamic import PairPool
from paper_2410_21634_b200.gen import rmat_csr_device
from paper_2410_21634_b200.graph import CsrGraph, EdgeEvent, apply_events
from paper_2410_21634_b200.metrics import sample_sources
n, m = SHAPES["arxiv"]
row, col = rmat_csr_device(n, m, seed=0)
g0 = CsrGraph(n=n, offsets=row.cpu().numpy(), targets=col.cpu().numpy().astype(np.int64))
rng = np.random.default_rng(1)
batches, sim = [], g0
for _ in range(6):
    b, seen = [], set()
    while len(b) < 1000:
        u, v = sorted(rng.integers(0, n, 2).tolist())
        if u == v or (u, v) in seen or sim.has_edge(u, v):
            continue
        seen.add((u, v)); b.append(EdgeEvent("insert", u, v))
    sim = apply_events(sim, b); batches.append(b)
pool = PairPool(g0, sample_sources(g0, 1024, seed=0), 0.15, 0.15e-6)
for mode in ("plain", "with_graph_export"):
    for b in batches[:3] if mode == "plain" else batches[3:]:
        torch.cuda.synchronize(); t0 = time.perf_counter()
        st = pool.update(b)
        t1 = time.perf_counter()
        if mode != "plain":
            _ = pool.graph
        print(mode, f"update {1e3*(t1-t0):.2f} ms", flush=True)
