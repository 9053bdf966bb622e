"""Round log summary of one refill solve: rounds, time histogram, arcs/round."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import make_graph, _HostGraph, SHAPES
from paper_2410_21634_b200.batch import BatchSolver
from paper_2410_21634_b200.metrics import sample_sources
shape, slots, nseeds = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
n, m = SHAPES[shape]
dg, row, col, row_h = make_graph(shape, 0, 0)
seeds = sample_sources(_HostGraph(n, row_h), nseeds, seed=0)
s = BatchSolver(dg, 0.1, 1e-7, slots=slots)
d = torch.as_tensor(seeds, device="cuda")
s.solve_device(d); s.solve_device(d)
lg = s.round_log()
dt = np.diff(lg[:, 2]) / 1e3
P = lg[:-1, 1]
print(f"slots={slots} seeds={nseeds} rounds={len(lg)} kernel_ms={s.last_kernel_ms:.2f} sum_round_ms={dt.sum()/1e3:.2f}")
print(f"round us: median {np.median(dt):.1f}  p10 {np.percentile(dt,10):.1f}  p90 {np.percentile(dt,90):.1f}")
print(f"arcs/round: median {np.median(P):.0f} mean {P.mean():.0f}; rate over all rounds {P.sum()/dt.sum()/1e3:.1f} G arcs/s")
small = dt[P < 100000]
print(f"rounds with <100K arcs: {len(small)} taking {small.sum()/1e3:.2f} ms (median {np.median(small) if len(small) else 0:.1f} us)")
