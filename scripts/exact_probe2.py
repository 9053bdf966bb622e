"""Cost of the bit-exact re-solve path on the products shape (resolve="all")."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import SHAPES, _HostGraph, make_graph  # noqa: E402
from paper_2410_21634_b200.batch import BatchSolver  # noqa: E402
from paper_2410_21634_b200.metrics import sample_sources  # noqa: E402

n, _ = SHAPES["products"]
dg, row, col, row_h = make_graph("products", 0, 0)
seeds = sample_sources(_HostGraph(n, row_h), 1024, seed=0)[::64]
for w in sys.argv[1].split(","):
    os.environ["GDIFF_RESOLVE_WORKERS"] = w
    s = BatchSolver(dg, 0.1, 1e-7, resolve="all")
    for _ in range(3):
        s.solve(seeds)
    t = time.perf_counter()
    o = s.solve(seeds)
    print(f"workers={w} seeds={len(seeds)} wall={1e3*(time.perf_counter()-t):.1f}ms "
          f"resolve={s.resolve_stats()} sweeps={o.sweeps.tolist()}")
    s.close()
