import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import SHAPES
from paper_2410_21634_b200.gen import rmat_csr_device_big
from paper_2410_21634_b200.device import DeviceGraph
def mem(tag):
    f, t = torch.cuda.mem_get_info(); print(f"{tag}: free {f/1e9:.1f} GB, torch reserved {torch.cuda.memory_reserved()/1e9:.1f} GB", flush=True)
n, m = SHAPES["papers100M"]
t0 = time.time()
row, col = rmat_csr_device_big(n, m, seed=0)
torch.cuda.synchronize(); print(f"generated in {time.time()-t0:.1f} s, arcs {col.numel()}", flush=True)
mem("after gen")
torch.cuda.empty_cache(); mem("after empty_cache")
dg = DeviceGraph.from_device(n, row, col)
del row, col; torch.cuda.empty_cache(); mem("after DeviceGraph")
from paper_2410_21634_b200.batch import BatchSolver
s = BatchSolver(dg, 0.1, 1e-7, slots=int(sys.argv[1]) if len(sys.argv) > 1 else 8)
mem("after BatchSolver")
