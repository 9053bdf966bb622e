"""In-situ kernel durations of one batched solve (torch profiler / CUPTI,
no replay): round kernel vs extract / reset / init per wave."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from bench import SHAPES, _HostGraph, make_graph
from paper_2410_21634_b200.batch import BatchSolver
from paper_2410_21634_b200.metrics import sample_sources

shape = sys.argv[1] if len(sys.argv) > 1 else "products"
seeds_n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
n, m = SHAPES[shape]
dg, row, col, row_h = make_graph(shape, 0, 0)
seeds = torch.as_tensor(sample_sources(_HostGraph(n, row_h), seeds_n, seed=0), device="cuda")
s = BatchSolver(dg, 0.1, 1e-7)
for _ in range(2):
    s.solve_device(seeds)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
s.solve_device(seeds)
e1.record()
torch.cuda.synchronize()
print(f"sets={os.environ.get('GDIFF_BATCH_SETS', 'auto')} solve_ms={e0.elapsed_time(e1):.2f} "
      f"kernel_ms={s.last_kernel_ms:.2f}")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    s.solve_device(seeds)
    torch.cuda.synchronize()
for ev in prof.key_averages():
    if ev.device_type.name == "CUDA" or True:
        t = getattr(ev, "device_time_total", 0) or getattr(ev, "cuda_time_total", 0)
        if t > 20:
            print(f"{ev.key[:70]:70s} n={ev.count:4d} total_us={t:10.1f}")
