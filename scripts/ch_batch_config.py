"""Config 3 batched: LocalCH (Katz and PPR) seed batches on an OGB-shape
R-MAT graph vs the reference's per-seed local_ch on all host cores.
Per-seed sweeps / operation counts are compared on the CPU sample.

usage: python scripts/ch_batch_config.py [shape] [eps] [seeds] [cpu_seeds]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from bench import SHAPES
from oracle import oracle as O
from paper_2410_21634_b200.batch import BatchSolver
from paper_2410_21634_b200.gen import rmat_csr_device
from paper_2410_21634_b200.graph import CsrGraph, spectral_norm_estimate
from paper_2410_21634_b200.metrics import sample_sources

shape = sys.argv[1] if len(sys.argv) > 1 else "products"
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-7
n_seeds = int(sys.argv[3]) if len(sys.argv) > 3 else 512
cpu_seeds = int(sys.argv[4]) if len(sys.argv) > 4 else 64
n, m = SHAPES[shape]
row, col = rmat_csr_device(n, m, seed=0)
g = CsrGraph(n=n, offsets=row.cpu().numpy(), targets=col.cpu().numpy().astype(np.int64))
seeds = sample_sources(g, n_seeds, seed=0)
threads = os.cpu_count() or 1
t0 = time.perf_counter()
lam = spectral_norm_estimate(g, iters=200, seed=0, device=True)
t_lam = time.perf_counter() - t0


def run(problem, alpha, mu, L):
    solver = BatchSolver(g, alpha, eps, method="local-ch", problem=problem, mu=mu, L=L,
                         max_sweeps=max(1000, int(10 * np.log(max(1.0 / eps, 2.0)) / max(mu, 1e-12))))
    out = solver.solve(seeds)  # warm-up (allocations, first-touch)
    torch.cuda.synchronize()
    reps = 3
    t0 = time.perf_counter()
    for _ in range(reps):
        out = solver.solve(seeds)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    kms = solver.last_kernel_ms
    k = min(cpu_seeds, n_seeds)
    t0 = time.perf_counter()
    ref = O.batch_local_ch(g, alpha, eps, seeds[:k], threads, mu, L, problem=problem,
                           max_sweeps=max(1000, int(10 * np.log(max(1.0 / eps, 2.0)) / max(mu, 1e-12))))
    tc = time.perf_counter() - t0
    same = bool(np.array_equal(ref["sweeps"], out.sweeps[:k]) and
                np.array_equal(ref["total_ops"], out.total_ops[:k]) and
                np.array_equal(ref["converged"], out.converged[:k]))
    ops = int(out.total_ops.sum())
    print(json.dumps({
        "case": f"{shape} LocalCH {problem} alpha={alpha:.6g} mu={mu:.6g} L={L:.6g} eps={eps:g}",
        "seeds": n_seeds, "gpu_solves_per_s": round(n_seeds / dt, 1),
        "gpu_kernel_ms": round(kms, 2), "gpu_wall_ms": round(dt * 1e3, 2),
        "edges_touched_per_s": round(ops / dt / 1e9, 3), "mean_sweeps": float(out.sweeps.mean()),
        "mean_ops": float(out.total_ops.mean()), "converged": int(out.converged.sum()),
        "cpu_solves_per_s": round(k / tc, 2), "cpu_threads": threads, "cpu_sample": k,
        "speedup": round((n_seeds / dt) / (k / tc), 1), "per_seed_sweeps_ops_identical": same,
    }), flush=True)
    solver.close()


ka = 1.0 / (lam + 1.0)  # default_katz_alpha (spectral regime)
lc = min(max(lam, 1e-12), float(g.d_max))
run("katz", ka, 1.0 - ka * lc, 1.0 + ka * lc)
kn = 0.9 / g.d_max      # nonneg regime
run("katz", kn, 1.0 - kn * lc, 1.0 + kn * lc)
run("ppr", 0.1, 0.1, 1.9)
print(json.dumps({"lam_hat": lam, "lam_seconds": round(t_lam, 2), "d_max": int(g.d_max)}))
