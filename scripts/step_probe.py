"""Where does a bench step spend time outside the sweep kernel?"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import make_graph, _HostGraph, SHAPES
from paper_2410_21634_b200.batch import BatchSolver
from paper_2410_21634_b200.metrics import sample_sources
n, m = SHAPES["products"]
dg, row, col, row_h = make_graph("products", 0, 0)
seeds = sample_sources(_HostGraph(n, row_h), 1024 * 4, seed=0)
s = BatchSolver(dg, 0.1, 1e-7, slots=int(sys.argv[1]) if len(sys.argv) > 1 else 64)
ds = [torch.as_tensor(seeds[i * 1024:(i + 1) * 1024], device="cuda") for i in range(4)]
s.solve_device(ds[0]); torch.cuda.synchronize()
for i in range(1, 4):
    t0 = time.perf_counter()
    res = s.solve_device(ds[i])
    t1 = time.perf_counter()
    a = int(res["total_ops"].sum()); b = int(res["pushes"].sum())
    t2 = time.perf_counter()
    print(f"solve_device wall {1e3*(t1-t0):.2f} ms, kernel(sweep) {s.last_kernel_ms:.2f} ms, sums {1e3*(t2-t1):.2f} ms")
