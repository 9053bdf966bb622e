"""Single-system FIFO solvers (drop-in local_gs / local_sor / repair) vs the
CPU port, per solve."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from bench import SHAPES
from oracle import oracle as O
from paper_2410_21634_b200 import local_solvers as LS, systems as S
from paper_2410_21634_b200.gen import rmat_csr_device
from paper_2410_21634_b200.graph import CsrGraph
from paper_2410_21634_b200.metrics import sample_sources

shape = sys.argv[1] if len(sys.argv) > 1 else "arxiv"
n, m = SHAPES[shape]
row, col = rmat_csr_device(n, m, seed=0)
g = CsrGraph(n=n, offsets=row.cpu().numpy(), targets=col.cpu().numpy().astype(np.int64))
for eps in (1e-6, 1e-7):
    for omega in (1.0, LS.optimal_omega(0.1)):
        s = int(sample_sources(g, 8, seed=0)[4])
        sys_ = S.make_ppr_system(g, 0.1, s, eps)
        LS.local_sor(sys_, omega=omega)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st, rep = LS.local_sor(sys_, omega=omega)
        tg = time.perf_counter() - t0
        t0 = time.perf_counter()
        ref = O.local_sor(sys_, omega)
        tc = time.perf_counter() - t0
        print(json.dumps({"case": f"{shape} local_sor omega={omega:.5f} eps={eps:g}", "gpu_ms": round(tg * 1e3, 2),
                          "cpu_ms": round(tc * 1e3, 2), "speedup": round(tc / tg, 2),
                          "bitwise": bool(np.array_equal(st.x, ref["x"])), "ops": rep.total_ops}), flush=True)
