"""Where the wall time of PairPool.update goes."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from bench import SHAPES
from paper_2410_21634_b200 import _lib as gdl
from paper_2410_21634_b200.dynamic import PairPool
from paper_2410_21634_b200.gen import rmat_csr_device
from paper_2410_21634_b200.graph import CsrGraph, EdgeEvent
from paper_2410_21634_b200.metrics import sample_sources

shape = sys.argv[1] if len(sys.argv) > 1 else "arxiv"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
n, m = SHAPES[shape]
row, col = rmat_csr_device(n, m, seed=0)
g0 = CsrGraph(n=n, offsets=row.cpu().numpy(), targets=col.cpu().numpy().astype(np.int64))
rng = np.random.default_rng(1)
pool = PairPool(g0, sample_sources(g0, K, seed=0), 0.15, 0.15e-6)
lib = gdl.load()
for it in range(6):
    b, seen = [], set()
    while len(b) < 1000:
        u, v = sorted(rng.integers(0, n, 2).tolist())
        if u == v or (u, v) in seen or g0.has_edge(u, v):
            continue
        seen.add((u, v))
        b.append(EdgeEvent("insert", u, v))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dg = pool.dgraph.apply_events(b, out=pool._spare)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    kinds = np.ones(len(b), np.int32)
    us = np.array([e.u for e in b], np.int64)
    vs = np.array([e.v for e in b], np.int64)
    st = pool._stats()
    t2 = time.perf_counter()
    gdl.check(lib.gd_pairs_update(pool.handle, dg.handle, gdl.ptr(kinds, C.c_int32),
                                  gdl.ptr(us, C.c_int64), gdl.ptr(vs, C.c_int64), len(b), 0,
                                  *pool._stat_ptrs(st)))
    t3 = time.perf_counter()
    if pool._own:
        pool._spare = pool.dgraph
    pool.dgraph, pool._host, pool._own = dg, None, True
    g0 = pool.graph
    print(f"edit {1e3*(t1-t0):.2f} ms  arrays {1e3*(t2-t1):.2f} ms  gd_pairs_update {1e3*(t3-t2):.2f} ms"
          f"  (repair kernel {pool.last_kernel_ms:.2f} ms)", flush=True)
