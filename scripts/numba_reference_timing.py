"""Time the reference's own local_gd (numba, installed in baseline/_ref) next to
the C port of oracle/ on the same seeds: the CPU baseline bench.py reports is the
port, so its speed relative to the real reference is measured here, not assumed
(VERDICT r1 "missing" 4).

    PYTHONPATH=baseline/_ref python scripts/numba_reference_timing.py SHAPE EPS SEEDS

Reference protocol (SURVEY.md 8(d) "CPU path timing"): one system per (graph,
alpha, eps), b / source swapped per seed with dataclasses.replace (the reference
CLI builds systems outside its timed region, src/cli.py:152-156), one process
per core (fork, NUMBA_NUM_THREADS=1, JIT warmed in every worker); the port runs
the same seeds on as many threads.  Integer work (sweeps, total_ops) is compared
seed by seed.  Measurement script only: not on any product or bench path.
"""
from __future__ import annotations

import dataclasses
import json
import os
import sys
import time

os.environ.setdefault("NUMBA_NUM_THREADS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))

import numpy as np  # noqa: E402

_G = {}


def _init(n, offsets, targets, alpha, eps):
    from graphdiff.graph import CsrGraph
    from graphdiff.local_solvers import local_gd
    from graphdiff.systems import make_ppr_system

    g = CsrGraph(n=n, offsets=offsets, targets=targets)
    s0 = int(np.argmax(np.diff(offsets)))
    _G["sys"] = make_ppr_system(g, alpha, s0, eps, symmetrized=True)
    _G["n"], _G["alpha"] = n, alpha
    local_gd(_G["sys"], max_sweeps=1)  # JIT warm-up


def _solve(s):
    from graphdiff.local_solvers import local_gd

    b = np.zeros(_G["n"])
    b[s] = _G["alpha"]
    sys_ = dataclasses.replace(_G["sys"], b=b, source=int(s))
    t = time.perf_counter()
    st, rep = local_gd(sys_)
    return int(st.sweeps), int(st.ops), time.perf_counter() - t


def main():
    import multiprocessing as mp

    from bench import SHAPES
    from oracle import oracle as O
    from paper_2410_21634_b200.gen import rmat_csr_device
    from paper_2410_21634_b200.metrics import sample_sources

    shape, eps, count = sys.argv[1], float(sys.argv[2]), int(sys.argv[3])
    alpha = 0.1
    n, m = SHAPES[shape]
    row, col = rmat_csr_device(n, m, seed=0, device=0, native=False)  # torch ops only
    offsets = row.cpu().numpy().astype(np.int64)
    targets = col.cpu().numpy().astype(np.int64)
    del row, col

    class _H:  # sample_sources needs degrees only
        pass
    h = _H()
    h.n, h.degrees = n, np.diff(offsets)
    batch = sample_sources(h, 1024, seed=0)
    seeds = batch[:: max(1, 1024 // count)][:count]
    P = len(os.sched_getaffinity(0))
    ctx = mp.get_context("fork")
    with ctx.Pool(P, initializer=_init, initargs=(n, offsets, targets, alpha, eps)) as pool:
        pool.map(_solve, seeds[:P])  # (every worker warm)
        t0 = time.perf_counter()
        ref = pool.map(_solve, seeds, chunksize=1)
        wall_ref = time.perf_counter() - t0

    class _Hg:
        pass
    hg = _Hg()
    hg.n, hg.offsets, hg.targets = n, offsets, targets
    hg.degrees = np.diff(offsets)
    d = np.repeat(hg.degrees.astype(np.float64), hg.degrees)
    arc_w = (1.0 / d) * (1.0 - alpha)
    from paper_2410_21634_b200.systems import theta_vector
    theta = theta_vector(hg, eps * alpha)
    O.batch_local_gd(hg, alpha, eps, seeds[:P], P, arc_w=arc_w, theta=theta, xsum=False)
    t0 = time.perf_counter()
    port = O.batch_local_gd(hg, alpha, eps, seeds, P, arc_w=arc_w, theta=theta, xsum=False)
    wall_port = time.perf_counter() - t0
    same = bool(np.array_equal([r[0] for r in ref], port["sweeps"])
                and np.array_equal([r[1] for r in ref], port["total_ops"]))
    out = {
        "shape": shape, "eps": eps, "alpha": alpha, "seeds": len(seeds),
        "sample": f"every {max(1, 1024 // count)}th seed of sample_sources(g, 1024, seed=0)",
        "cores": P, "cpu": os.uname().nodename,
        "reference_numba": {"solves_per_s": len(seeds) / wall_ref,
                            "mean_solve_s": float(np.mean([r[2] for r in ref])),
                            "protocol": "ProcessPool(fork), NUMBA_NUM_THREADS=1, system built once, "
                                        "b swapped per seed (dataclasses.replace)"},
        "port_c": {"solves_per_s": len(seeds) / wall_port, "protocol": "oracle/ threads, one seed each"},
        "port_over_reference": (len(seeds) / wall_port) / (len(seeds) / wall_ref),
        "integer_work_identical": same,
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
