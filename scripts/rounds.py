"""Per-round profile of one batched wave (frontier entries, arcs, time)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import make_graph, _HostGraph, SHAPES
from paper_2410_21634_b200.batch import BatchSolver
from paper_2410_21634_b200.metrics import sample_sources
shape = sys.argv[1] if len(sys.argv) > 1 else "products"
slots = int(sys.argv[2]) if len(sys.argv) > 2 else 128
eps = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-7
n, m = SHAPES[shape]
dg, row, col, row_h = make_graph(shape, 0, 0)
seeds = sample_sources(_HostGraph(n, row_h), slots, seed=0)
s = BatchSolver(dg, 0.1, eps, slots=slots)
d = torch.as_tensor(seeds, device="cuda")
s.solve_device(d); s.solve_device(d)
lg = s.round_log()
t = lg[:, 2] - lg[0, 2]
dt = np.diff(lg[:, 2]) / 1e3
print(f"rounds={len(lg)-1} kernel_ms={s.last_kernel_ms:.2f}")
for i in range(len(lg) - 1):
    F, P = lg[i, 0], lg[i, 1]
    print(f"round {i:3d}  F={F:9d}  P={P:11d}  {dt[i]:9.1f} us  {P/max(dt[i],1e-9)/1e3:8.2f} G arcs/s")
