"""Config 5: arxiv-shape graph split into 16 snapshots (G0 = 17.9 % of edges),
warm-started repair (GPU, bit-exact FIFO) vs static re-solve vs the CPU port."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import oracle as O
from paper_2410_21634_b200.dynamic import make_pair, event_adjust_many, repair, repair_gd
from paper_2410_21634_b200.graph import EdgeEvent, csr_from_pairs, apply_events
from paper_2410_21634_b200.synth import rmat_graph
from paper_2410_21634_b200.systems import arc_weights_for, theta_vector

METHOD = sys.argv[1] if len(sys.argv) > 1 else "gd"
n, m = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (169_343, 1_166_243)
nsnap = 16
g_full = rmat_graph(n, m, seed=0)
src = np.repeat(np.arange(n), g_full.degrees); keep = src < g_full.targets
edges = np.stack([src[keep], g_full.targets[keep]], 1)
rng = np.random.default_rng(0); rng.shuffle(edges)
n0 = int(0.179 * len(edges))
g = csr_from_pairs(n, edges[:n0])
rest = edges[n0:]
per = (len(rest) + nsnap - 1) // nsnap
alpha, eps = 0.1, 0.1 * 1e-6
s = int(np.argmax(g.degrees))
pair, rep = (repair_gd if METHOD == "gd" else repair)(g, make_pair(g, alpha, eps, s))
tot_gpu = tot_cpu = 0.0; ops_dyn = ops_static = 0; ok = True
for k in range(nsnap):
    batch = [EdgeEvent("insert", int(a), int(b)) for a, b in rest[k * per:(k + 1) * per]]
    pair = event_adjust_many(g, pair, batch)
    g = apply_events(g, batch)
    fix = repair_gd if METHOD == "gd" else repair
    repair_gd(g, pair.copy()) if k == 0 else None  # warm the device graph upload
    torch.cuda.synchronize(); t0 = time.perf_counter()
    new, rep = fix(g, pair)
    torch.cuda.synchronize(); tg = time.perf_counter() - t0
    # CPU port of the same repair (theta = eps d)
    w = arc_weights_for(g, 1.0 - alpha, "gen", 0.0); th = theta_vector(g, eps)
    p2, r2 = pair.p.copy(), pair.r.copy()
    t0 = time.perf_counter()
    if METHOD == "gd":
        ref = O.local_gd_warm(g.offsets, g.targets, w, th, p2, r2, signed=True, record_trace=False)
    else:
        seeds = np.flatnonzero(np.abs(r2) >= th)
        ref = O.push_kernel(g.offsets, g.targets, w, th, p2, r2, seeds, omega=1.0, signed=True)
    tc = time.perf_counter() - t0
    ok &= bool(np.array_equal(new.p, p2) and rep.total_ops == ref["total_ops"])
    tot_gpu += tg; tot_cpu += tc; ops_dyn += rep.total_ops
    pair = new
    _, rs = (repair_gd if METHOD == "gd" else repair)(g, make_pair(g, alpha, eps, s))
    ops_static += rs.total_ops
print(json.dumps({"case": f"dynamic arxiv-shape {nsnap} snapshots, insert batches of {per}, repair={METHOD}",
                  "gpu_repair_ms_total": round(tot_gpu * 1e3, 2), "cpu_port_ms_total": round(tot_cpu * 1e3, 2),
                  "speedup": round(tot_cpu / tot_gpu, 2), "bitwise": ok,
                  "ops_dynamic": ops_dyn, "ops_static_resolve": ops_static,
                  "ops_ratio_static_over_dynamic": round(ops_static / max(ops_dyn, 1), 2)}))
