GDIFF_EXACT_TRACE=1 GDIFF_RESOLVE_WORKERS=1 timeout 300 python - <<'PY' 2>&1 | tail -40
import os, sys
sys.path.insert(0, '.')
from bench import SHAPES, _HostGraph, make_graph
from paper_2410_21634_b200.batch import BatchSolver
from paper_2410_21634_b200.metrics import sample_sources
n, _ = SHAPES["products"]
dg, row, col, row_h = make_graph("products", 0, 0)
seeds = sample_sources(_HostGraph(n, row_h), 1024, seed=0)[[100, 900]]
s = BatchSolver(dg, 0.1, 1e-7, exact_all=True)
s.solve(seeds); s.solve(seeds)
print(s.resolve_stats())
PY
