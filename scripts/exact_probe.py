import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import SHAPES
from paper_2410_21634_b200 import local_solvers as LS, systems as S
from paper_2410_21634_b200.gen import rmat_csr_device
from paper_2410_21634_b200.graph import CsrGraph
from paper_2410_21634_b200.metrics import sample_sources
n, m = SHAPES[sys.argv[1] if len(sys.argv) > 1 else "products"]
row, col = rmat_csr_device(n, m, seed=0)
g = CsrGraph(n=n, offsets=row.cpu().numpy(), targets=col.cpu().numpy().astype(np.int64))
s = int(sample_sources(g, 8, seed=0)[4])
sys_ = S.make_ppr_system(g, 0.1, s, 1e-7)
LS.local_gd(sys_)
for i in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    st, rep = LS.local_gd(sys_)
    torch.cuda.synchronize(); print("local_gd wall ms", (time.perf_counter() - t0) * 1e3, "sweeps", rep.sweeps, flush=True)
import cProfile, pstats
cProfile.run("LS.local_gd(sys_)", "/tmp/prof")
pstats.Stats("/tmp/prof").sort_stats("cumtime").print_stats(12)
