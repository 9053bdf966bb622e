"""Rounds 0-1 of one 64-seed products wave only (max_sweeps=2), for an ncu capture
of the first (hub) round in isolation."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import make_graph, _HostGraph, SHAPES
from paper_2410_21634_b200.batch import BatchSolver
from paper_2410_21634_b200.metrics import sample_sources
off = int(sys.argv[1]) if len(sys.argv) > 1 else 512
n, m = SHAPES["products"]
dg, row, col, row_h = make_graph("products", 0, 0)
seeds = sample_sources(_HostGraph(n, row_h), 1024, seed=0)[off:off + 64]
s = BatchSolver(dg, 0.1, 1e-7, slots=64, max_sweeps=2)
for i in range(3):
    s.solve_device(torch.as_tensor(seeds, device="cuda")); torch.cuda.synchronize()
lg = s.round_log()
print("kernel_ms", s.last_kernel_ms, [(int(r[0]), int(r[1])) for r in lg[:3]])
