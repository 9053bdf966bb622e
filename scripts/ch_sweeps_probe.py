"""Sweeps per seed of a batched LocalCH / LocalHB wave (how many rounds a wave runs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import make_graph, _HostGraph, SHAPES, ch_params
from paper_2410_21634_b200.batch import BatchSolver
from paper_2410_21634_b200.metrics import sample_sources
import argparse
for method, prob in (("local-ch", "ppr"), ("local-hb", "ppr"), ("local-ch", "katz")):
    args = argparse.Namespace(method=method, problem=prob, alpha=0.1, eps=1e-7)
    n, m = SHAPES["products"]
    dg, row, col, row_h = make_graph("products", 0, 0)
    ch = ch_params(args, row, col, n)
    seeds = sample_sources(_HostGraph(n, row_h), 1024, seed=0)[:64]
    s = BatchSolver(dg, args.alpha, 1e-7, method=method, problem=prob, mu=ch.get("mu"), L=ch.get("L"),
                    max_sweeps=ch.get("max_sweeps", 1_000_000))
    for rep in range(2):
        r = s.solve_device(torch.as_tensor(seeds, device="cuda")); torch.cuda.synchronize()
    sw = r["sweeps"].cpu().numpy(); ops = r["total_ops"].cpu().numpy()
    print(method, prob, "slots", s.slots, "kernel_ms", round(s.last_kernel_ms, 3), "sweeps max", sw.max(),
          "mean", sw.mean(), "p50", np.median(sw), "ops/seed", ops.mean())
