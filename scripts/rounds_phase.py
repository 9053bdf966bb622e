"""Per-round phase times (push phase A / scatter phase B) of one 64-seed wave."""
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
s = BatchSolver(dg, 0.1, 1e-7, slots=64)
for i in range(3):
    s.solve_device(torch.as_tensor(seeds, device="cuda")); torch.cuda.synchronize()
lg = s.round_log()
print("kernel_ms", s.last_kernel_ms, "grid rounds", len(lg))
for i in range(len(lg)):
    F, P, t0, tb = lg[i, 0], lg[i, 1], lg[i, 2], lg[i, 3]
    t1 = lg[i + 1, 2] if i + 1 < len(lg) else None
    a = (tb - t0) / 1e3
    b = (t1 - tb) / 1e3 if t1 is not None else float('nan')
    print(f"round {i:3d} F={F:8d} P={P:10d}  phaseA {a:8.1f} us  phaseB {b:8.1f} us")
