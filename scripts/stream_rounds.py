"""Round log of one products-shape solve, streaming vs wave form (diagnostic):
rounds, entries F, arcs P and time per round from the kernel's globaltimer."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import SHAPES, _HostGraph, make_graph  # noqa: E402
from paper_2410_21634_b200.batch import BatchSolver  # noqa: E402
from paper_2410_21634_b200.metrics import sample_sources  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "products"
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-7
n, _ = SHAPES[shape]
dg, row, col, row_h = make_graph(shape, 0, 0)
hg = _HostGraph(n, row_h)
seeds = sample_sources(hg, 1024, seed=0)
for mode in (sys.argv[3].split(",") if len(sys.argv) > 3 else ("1", "0")):
    os.environ["GDIFF_STREAM"] = mode
    s = BatchSolver(dg, 0.1, eps)
    if os.environ.get("DEV"):
        import torch
        ds = torch.as_tensor(seeds, device="cuda")
        s.solve_device(ds)
        o = s.solve_device(ds)
        torch.cuda.synchronize()
    else:
        s.solve(seeds)
        o = s.solve(seeds)
    log = s.round_log()
    rs = s.resolve_stats()
    ms = s.last_kernel_ms
    dt = np.diff(log[:, 2]) / 1e3
    print(f"mode={s.mode} kernel_ms={ms:.2f} rounds_logged={len(log)} resolve={rs}")
    if len(log) > 1:
        F, P = log[:-1, 0], log[:-1, 1]
        ta = (log[:-1, 3] - log[:-1, 2]) / 1e3
        print(f"  phase A total {ta.sum()/1e3:.2f} ms")
        print(f"  sum F={F.sum()} sum P={P.sum()} median dt={np.median(dt):.1f}us "
              f"sum dt={dt.sum()/1e3:.2f}ms")
        for i in range(0, len(dt), int(os.environ.get("EVERY", max(1, len(dt) // 25)))):
            print(f"  r{i:4d} F={F[i]:9d} P={P[i]:11d} {dt[i]:8.1f}us A={ta[i]:7.1f}us fin={log[i, 4] & 0xffffffff:3d}{"R" if log[i, 4] >> 32 else " "} {P[i]/max(dt[i],1e-9)/1e3:6.2f} Garc/s")
    s.close()
