"""Per-round log of ONE fresh 64-seed wave (first solve of a new solver), for A/B
probes that leave the slots dirty (GDIFF_DBG=4)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import make_graph, _HostGraph, SHAPES
from paper_2410_21634_b200.batch import BatchSolver
from paper_2410_21634_b200.metrics import sample_sources
shape = sys.argv[1] if len(sys.argv) > 1 else "products"
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-7
off = int(sys.argv[3]) if len(sys.argv) > 3 else 0
n, m = SHAPES[shape]
dg, row, col, row_h = make_graph(shape, 0, 0)
seeds = sample_sources(_HostGraph(n, row_h), 1024, seed=0)[off:off + 64]
s = BatchSolver(dg, 0.1, eps, slots=64)
s.solve_device(torch.as_tensor(seeds, device="cuda")); torch.cuda.synchronize()
lg = s.round_log()
dt = np.diff(lg[:, 2]) / 1e3
print(f"rounds={len(lg)-1} kernel_ms={s.last_kernel_ms:.3f}")
for i in range(len(lg) - 1):
    F, P = lg[i, 0], lg[i, 1]
    print(f"round {i:3d}  F={F:9d}  P={P:11d}  {dt[i]:9.1f} us  {P/max(dt[i],1e-9)/1e3:8.2f} G arcs/s")
