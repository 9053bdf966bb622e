"""Configs 3 and 5 on one GPU: single-system solvers (bit-exact path) vs the
CPU port, per solve; prints one line per case."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import SHAPES
from oracle import oracle as O
from paper_2410_21634_b200 import local_solvers as LS, systems as S
from paper_2410_21634_b200.gen import rmat_csr_device
from paper_2410_21634_b200.graph import CsrGraph
from paper_2410_21634_b200.metrics import sample_sources
from paper_2410_21634_b200.global_solvers import gradient_descent

def graph(shape):
    n, m = SHAPES[shape]
    row, col = rmat_csr_device(n, m, seed=0)
    return CsrGraph(n=n, offsets=row.cpu().numpy(), targets=col.cpu().numpy().astype(np.int64))

def timeit(fn, reps=1):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): out = fn()
    torch.cuda.synchronize()
    return out, (time.perf_counter() - t0) / reps

def line(name, gpu_s, cpu_s, ok, extra=""):
    print(json.dumps({"case": name, "gpu_ms": round(gpu_s * 1e3, 3), "cpu_ms": round(cpu_s * 1e3, 3),
                      "speedup": round(cpu_s / gpu_s, 2), "bitwise_or_identical": ok, "note": extra}), flush=True)

shape = sys.argv[1] if len(sys.argv) > 1 else "products"
g = graph(shape)
seeds = sample_sources(g, 8, seed=0)
s = int(seeds[4])
# LocalCH PPR eps 1e-7 (mu, L = alpha, 2 - alpha)
sys_ = S.make_ppr_system(g, 0.1, s, 1e-7, symmetrized=True)
(st, rep), tg = timeit(lambda: LS.local_ch(sys_))
t0 = time.perf_counter(); ref = O.local_ch(sys_); tc = time.perf_counter() - t0
line(f"{shape} LocalCH PPR eps=1e-7 seed={s}", tg, tc, bool(np.array_equal(st.x, ref["x"]) and rep.sweeps == ref["sweeps"]),
     f"sweeps={rep.sweeps} ops={rep.total_ops}")
# LocalGD single-system (exact) for comparison
(st, rep), tg = timeit(lambda: LS.local_gd(sys_))
t0 = time.perf_counter(); ref = O.local_gd(sys_, record_trace=False); tc = time.perf_counter() - t0
line(f"{shape} LocalGD exact single PPR eps=1e-7", tg, tc, bool(np.array_equal(st.x, ref["x"])), f"ops={rep.total_ops}")
# Katz nonneg regime alpha = 0.9/d_max, LocalCH with explicit bounds (lam = d_max)
ka = 0.9 / g.d_max
ks = S.make_katz_system(g, ka, s, 1e-7, lam_hat=0.0)
mu, L = 1.0 - ka * g.d_max, 1.0 + ka * g.d_max
(st, rep), tg = timeit(lambda: LS.local_ch(ks, mu=mu, L=L))
t0 = time.perf_counter(); ref = O.local_ch(ks, mu, L); tc = time.perf_counter() - t0
line(f"{shape} LocalCH Katz a=0.9/dmax eps=1e-7", tg, tc, bool(np.array_equal(st.x, ref["x"])), f"sweeps={rep.sweeps}")
(st, rep), tg = timeit(lambda: LS.local_gd(ks))
t0 = time.perf_counter(); ref = O.local_gd(ks, record_trace=False); tc = time.perf_counter() - t0
line(f"{shape} LocalGD Katz a=0.9/dmax eps=1e-7", tg, tc, bool(np.array_equal(st.x, ref["x"])), f"sweeps={rep.sweeps}")
# heat kernel tau=10 eps=1e-7 -> N=31 stages, effectively global
eps_hk = 1e-4 if shape == "products" else 1e-7
(out, rep), tg = timeit(lambda: LS.local_hk(g, 10.0, s, eps_hk))
t0 = time.perf_counter(); ref = O.local_hk(g, 10.0, s, eps_hk); tc = time.perf_counter() - t0
line(f"{shape} HK tau=10 eps={eps_hk:g}", tg, tc, bool(np.array_equal(out, ref["f_hat"])),
     f"N={rep.notes['stage_count']} sweeps={rep.sweeps} ops={rep.total_ops}")
# global GD reference point, PPR eps=1e-6
gs = S.make_ppr_system(g, 0.1, s, 1e-6)
(st, rep), tg = timeit(lambda: gradient_descent(gs))
t0 = time.perf_counter(); ref = O.gradient_descent(gs); tc = time.perf_counter() - t0
line(f"{shape} global GD PPR eps=1e-6", tg, tc, bool(np.array_equal(st.x, ref["x"])),
     f"sweeps={rep.sweeps} GTEPS={rep.total_ops / tg / 1e9:.2f}")
