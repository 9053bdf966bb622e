"""Per-round frontier entries / arcs of one heat-kernel wave (density of the stages)."""
import os, sys, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import make_graph, _HostGraph, SHAPES, hk_config
from paper_2410_21634_b200.batch import BatchSolver
from paper_2410_21634_b200.metrics import sample_sources
shape = sys.argv[1] if len(sys.argv) > 1 else "products"
n, m = SHAPES[shape]
dg, row, col, row_h = make_graph(shape, 0, 0)
hg = _HostGraph(n, row_h)
hk = hk_config(argparse.Namespace(tau=10.0, eps=1e-7), hg)
seeds = sample_sources(hg, 1024, seed=0)[:64]
s = BatchSolver(dg, 1.0, 1e-7, method="local-hk", hk=hk)
r = s.solve_device(torch.as_tensor(seeds[:s.slots], device="cuda")); torch.cuda.synchronize()
lg = s.round_log()
print("slots", s.slots, "kernel_ms", s.last_kernel_ms, "2E", 2 * m)
for i in range(len(lg)):
    dt = (lg[i + 1, 2] - lg[i, 2]) / 1e3 if i + 1 < len(lg) else float('nan')
    da = (lg[i, 3] - lg[i, 2]) / 1e3
    print(f"round {i:3d} F={lg[i,0]:10d} P={lg[i,1]:12d} density={lg[i,1]/(s.slots*2*m):6.3f} "
          f"{dt:9.1f} us (phase A {da:9.1f} us)")
