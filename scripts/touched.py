"""How big / how concentrated is one seed's touched residual set (products, eps 1e-7)?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import SHAPES
from paper_2410_21634_b200.gen import rmat_csr_device, relabel_by_degree
from paper_2410_21634_b200.graph import CsrGraph
from paper_2410_21634_b200.systems import make_ppr_system
from paper_2410_21634_b200.local_solvers import local_gd
from paper_2410_21634_b200.metrics import sample_sources
n, m = SHAPES[sys.argv[1] if len(sys.argv) > 1 else "products"]
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-7
row, col = rmat_csr_device(n, m, seed=0)
row2, col2, perm, inv = relabel_by_degree(row, col)
g = CsrGraph(n=n, offsets=row2.cpu().numpy(), targets=col2.cpu().numpy().astype(np.int64))
print("dmax", g.d_max, "deg>0", int((g.degrees > 0).sum()))
seeds = sample_sources(g, 16, seed=0)
for s in seeds[::3]:
    st, rep = local_gd(make_ppr_system(g, 0.1, int(s), eps))
    touched = np.flatnonzero((st.r != 0) | (st.x != 0))
    sect = np.unique(touched >> 2)
    q = np.quantile(touched, [0.5, 0.9, 0.99])
    print(f"seed {s:8d} d={g.degrees[s]:6d} sweeps {rep.sweeps:3d} ops {rep.total_ops:9d} pushes {sum(rep.notes['frontier_sizes']):7d} "
          f"touched {len(touched):8d} ({len(touched)/n:.2%}) sectors {len(sect)} ({len(sect)*32/1e6:.1f} MB) "
          f"id quantiles 50/90/99% {q[0]/n:.2f} {q[1]/n:.2f} {q[2]/n:.2f}  pushed {int((st.x!=0).sum())}")
