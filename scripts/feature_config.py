"""Multi-column feature push (beta_push over the columns of a sparse random
feature matrix) on the GPU vs the CPU port of beta_push per column on all
host threads.  usage: python scripts/feature_config.py [shape] [cols] [beta] [eps]"""
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from bench import SHAPES
from oracle import oracle as O
from paper_2410_21634_b200 import systems as S
from paper_2410_21634_b200.dynamic import beta_push_batch
from paper_2410_21634_b200.gen import rmat_csr_device
from paper_2410_21634_b200.graph import CsrGraph

shape = sys.argv[1] if len(sys.argv) > 1 else "arxiv"
cols = int(sys.argv[2]) if len(sys.argv) > 2 else 128
beta = float(sys.argv[3]) if len(sys.argv) > 3 else 0.5
eps = float(sys.argv[4]) if len(sys.argv) > 4 else 1e-4
alpha = 0.15
n, m = SHAPES[shape]
row, col = rmat_csr_device(n, m, seed=0)
g = CsrGraph(n=n, offsets=row.cpu().numpy(), targets=col.cpu().numpy().astype(np.int64))
rng = np.random.default_rng(0)
src = rng.standard_normal((n, cols)) * (rng.random((n, cols)) < 0.01)
beta_push_batch(g, src, alpha, beta, eps)  # warm-up (upload, allocations)
torch.cuda.synchronize()
t0 = time.perf_counter()
out = beta_push_batch(g, src, alpha, beta, eps)
tg = time.perf_counter() - t0
w = S.OperatorQ(graph=g, beta=1.0 - alpha, pkind="gen", b_exp=beta).arc_weights
th = S.theta_vector(g, eps, 1.0 - beta)
k = min(cols, 32)


def one(c):
    p, r = np.zeros(n), src[:, c].copy()
    o = O.push_kernel(g.offsets, g.targets, w, th, p, r, np.flatnonzero(np.abs(r) >= th), x_gain=alpha,
                      signed=True)
    return o["total_ops"], np.array_equal(p, out["p"][:, c])


threads = os.cpu_count() or 1
t0 = time.perf_counter()
with ThreadPoolExecutor(threads) as ex:
    res = list(ex.map(one, range(k)))
tc = time.perf_counter() - t0
print(json.dumps({"case": f"{shape} feature push beta={beta} eps={eps:g} {cols} columns (1% dense sources)",
                  "gpu_cols_per_s": round(cols / tg, 1), "gpu_s": round(tg, 3),
                  "gteps": round(float(out["total_ops"].sum()) / tg / 1e9, 2),
                  "cpu_cols_per_s": round(k / tc, 2), "cpu_threads": threads, "cpu_sample": k,
                  "speedup": round((cols / tg) / (k / tc), 1),
                  "columns_bitwise": all(b for _, b in res)}), flush=True)
