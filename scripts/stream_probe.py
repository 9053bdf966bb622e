"""Streaming vs wave round kernel on one graph: integer outputs and x (debug)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_21634_b200.batch import BatchSolver  # noqa: E402
from paper_2410_21634_b200.metrics import sample_sources  # noqa: E402
from paper_2410_21634_b200.synth import rmat_graph  # noqa: E402

n, m, k, slots = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
g = rmat_graph(n, m, seed=5)
seeds = sample_sources(g, k, seed=0)
os.environ["GDIFF_BATCH_MODE"] = "rounds"
outs = {}
for mode in ("0", "1"):
    os.environ["GDIFF_STREAM"] = mode
    s = BatchSolver(g, 0.1, 1e-6, slots=slots)
    o = s.solve(seeds)
    print("mode", s.mode, "ms", s.last_kernel_ms)
    outs[mode] = o
    s.close()
a, b = outs["0"], outs["1"]
for f in ("sweeps", "total_ops", "pushes", "converged", "x_count"):
    eq = np.array_equal(getattr(a, f), getattr(b, f))
    print(f, eq, getattr(a, f)[:8], getattr(b, f)[:8])
for i in range(min(3, k)):
    print(i, a.x_sparse(i)[0][:6], b.x_sparse(i)[0][:6], np.abs(a.x_dense(i, g.n) - b.x_dense(i, g.n)).sum())
