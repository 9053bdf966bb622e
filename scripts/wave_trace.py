import sys, os
sys.path.insert(0, os.getcwd())
os.environ["GDIFF_WAVE_TRACE"] = "1"
import torch
from bench import make_graph, _HostGraph, SHAPES
from paper_2410_21634_b200.batch import BatchSolver
from paper_2410_21634_b200.metrics import sample_sources
shape = sys.argv[1]; eps = float(sys.argv[2])
n, m = SHAPES[shape]
dg, row, col, row_h = make_graph(shape, 0, 0)
seeds = sample_sources(_HostGraph(n, row_h), 1024, seed=0)
s = BatchSolver(dg, 0.1, eps)
d = torch.as_tensor(seeds, device="cuda")
for i in range(3):
    print("---- solve", i, file=sys.stderr, flush=True)
    s.solve_device(d); torch.cuda.synchronize()
    print("kernel ms", s.last_kernel_ms, file=sys.stderr, flush=True)
