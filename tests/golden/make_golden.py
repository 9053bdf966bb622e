"""Generate golden vectors by running the REFERENCE implementation.

Run in the authoring container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src:. NUMBA_CACHE_DIR=/tmp/nb \
        python tests/golden/make_golden.py

It imports the read-only reference package ``graphdiff`` and writes small
.npz fixtures next to this script.  Graphs are stored as CSR arrays inside
each fixture, so the tests need neither the reference nor its generators.
Every fixture records which reference function produced it.
"""

from __future__ import annotations

import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import graphdiff as ref  # noqa: E402  (the reference, /root/reference/pkg/src)
from graphdiff import dynamic as rdyn  # noqa: E402
from graphdiff import global_solvers as rgs  # noqa: E402
from graphdiff import local_solvers as rls  # noqa: E402
from graphdiff import synth as rsyn  # noqa: E402
from graphdiff import systems as rsys  # noqa: E402
from graphdiff.graph import CsrGraph as RefCsr  # noqa: E402
from graphdiff.graph import EdgeEvent, apply_event  # noqa: E402
from graphdiff.metrics import sample_sources  # noqa: E402

from paper_2410_21634_b200.synth import rmat_graph  # noqa: E402

warnings.simplefilter("ignore")


def put_graph(d, name, g):
    d[f"graph/{name}/n"] = np.int64(g.n)
    d[f"graph/{name}/offsets"] = np.asarray(g.offsets, dtype=np.int64)
    d[f"graph/{name}/targets"] = np.asarray(g.targets, dtype=np.int64)


def put_local(d, key, state, report, **params):
    d[f"{key}/x"] = np.asarray(state.x)
    d[f"{key}/r"] = np.asarray(state.r)
    d[f"{key}/sweeps"] = np.int64(report.sweeps)
    d[f"{key}/total_ops"] = np.int64(report.total_ops)
    d[f"{key}/converged"] = np.bool_(report.converged)
    d[f"{key}/vol_log"] = np.asarray(report.vol_log, dtype=np.int64)
    d[f"{key}/gamma_log"] = np.asarray(report.gamma_log, dtype=np.float64)
    d[f"{key}/l1_log"] = np.asarray(report.residual_l1_trace, dtype=np.float64)
    d[f"{key}/min_residual"] = np.float64(report.min_residual)
    d[f"{key}/support_size"] = np.int64(report.support_size)
    d[f"{key}/method"] = np.str_(report.method)
    if "frontier_sizes" in report.notes:
        d[f"{key}/frontier_sizes"] = np.asarray(report.notes["frontier_sizes"], dtype=np.int64)
    if "sweep_signs" in report.notes:
        d[f"{key}/sweep_signs"] = np.asarray(report.notes["sweep_signs"], dtype=np.int8)
    if "diverged" in report.notes:
        d[f"{key}/diverged"] = np.bool_(report.notes["diverged"])
    if getattr(state, "frontier_trace", None) is not None:
        tr = state.frontier_trace
        d[f"{key}/trace_flat"] = (np.concatenate(tr) if tr else np.empty(0)).astype(np.int64)
        d[f"{key}/trace_sizes"] = np.asarray([len(f) for f in tr], dtype=np.int64)
    for k, v in params.items():
        d[f"{key}/param/{k}"] = np.asarray(v)


def to_ref(g):
    return RefCsr(n=g.n, offsets=np.array(g.offsets), targets=np.array(g.targets))


def fixture_small():
    """er500 / er60 / k3 / p2: LocalGD, LocalCH, LocalGS, LocalSOR, GD, HK."""
    d = {}
    er500 = rsyn.erdos_renyi(500, 0.02, seed=21)
    er60 = rsyn.erdos_renyi(60, 0.1, seed=7)
    k3 = rsyn.complete_graph(3)
    p2 = rsyn.path_graph(2)
    for name, g in (("er500", er500), ("er60", er60), ("k3", k3), ("p2", p2)):
        put_graph(d, name, g)

    s = rsys.make_ppr_system(er500, 0.15, 0, 1e-6, symmetrized=True)
    put_local(d, "er500/ppr/local_gd", *rls.local_gd(s), graph="er500", problem="ppr",
              alpha=0.15, eps=1e-6, source=0)
    put_local(d, "er500/ppr/local_ch", *rls.local_ch(s), graph="er500", problem="ppr",
              alpha=0.15, eps=1e-6, source=0)
    put_local(d, "er500/ppr/local_gs", *rls.local_gs(s), graph="er500", problem="ppr",
              alpha=0.15, eps=1e-6, source=0)
    om = rls.optimal_omega(0.15)
    put_local(d, "er500/ppr/local_sor", *rls.local_sor(s, omega=om), graph="er500",
              problem="ppr", alpha=0.15, eps=1e-6, source=0, omega=om)
    st, rp = rgs.gradient_descent(s)
    d["er500/ppr/gd/x"], d["er500/ppr/gd/r"] = st.x, st.r
    d["er500/ppr/gd/sweeps"] = np.int64(rp.sweeps)
    d["er500/ppr/gd/total_ops"] = np.int64(rp.total_ops)
    d["er500/ppr/gd/l1_log"] = np.asarray(rp.residual_l1_trace)
    d["er500/ppr/gd/l2_log"] = np.asarray(rp.notes["l2_trace"])

    s = rsys.make_ppr_system(er60, 0.2, 0, 1e-5)
    base = dict(graph="er60", problem="ppr", alpha=0.2, eps=1e-5, source=0)
    put_local(d, "er60/ppr/local_gs", *rls.local_gs(s), **base)
    put_local(d, "er60/ppr/local_sor13", *rls.local_sor(s, omega=1.3), **base, omega=1.3)
    put_local(d, "er60/ppr/local_sor05", *rls.local_sor(s, omega=0.5), **base, omega=0.5)
    put_local(d, "er60/ppr/local_gd", *rls.local_gd(s), **base)
    put_local(d, "er60/ppr/local_gs_max2", *rls.local_gs(rsys.make_ppr_system(er60, 0.1, 0, 1e-9),
                                                          max_sweeps=2),
              graph="er60", problem="ppr", alpha=0.1, eps=1e-9, source=0, max_sweeps=2)
    s = rsys.make_ppr_system(er60, 0.2, 0, 1e-6, symmetrized=True)
    put_local(d, "er60/ppr/local_ch", *rls.local_ch(s), graph="er60", problem="ppr",
              alpha=0.2, eps=1e-6, source=0)

    ka = 0.9 / er60.d_max
    s = rsys.make_katz_system(er60, ka, 0, 1e-4)
    base = dict(graph="er60", problem="katz", alpha=ka, eps=1e-4, source=0)
    put_local(d, "er60/katz/local_gd", *rls.local_gd(s), **base)
    put_local(d, "er60/katz/local_gs", *rls.local_gs(s), **base)
    mu, L = rls._cheby_bounds(s, None, None)
    put_local(d, "er60/katz/local_ch", *rls.local_ch(s), **base, mu=mu, L=L)

    s = rsys.make_katz_system(k3, 0.25, 0, 1e-6)
    put_local(d, "k3/katz/local_gs", *rls.local_gs(s), graph="k3", problem="katz",
              alpha=0.25, eps=1e-6, source=0)

    for tau in (0.5, 1.0, 5.0):
        f, rp = rls.local_hk(er60, tau, 0, 1e-4)
        key = f"er60/hk/tau{tau}"
        d[f"{key}/f_hat"] = f
        d[f"{key}/sweeps"] = np.int64(rp.sweeps)
        d[f"{key}/total_ops"] = np.int64(rp.total_ops)
        d[f"{key}/vol_log"] = np.asarray(rp.vol_log, dtype=np.int64)
        d[f"{key}/gamma_log"] = np.asarray(rp.gamma_log)
        d[f"{key}/l1_log"] = np.asarray(rp.residual_l1_trace)
        d[f"{key}/stage_count"] = np.int64(rp.notes["stage_count"])
        d[f"{key}/residual_mass"] = np.float64(rp.notes["residual_mass"])
        d[f"{key}/series60"] = rsys.series_oracle(rsys.make_hk_system(er60, tau, 0, 1e-4), 60)
    f, rp = rls.local_hk(p2, 1e-9, 0, 1e-3)
    d["p2/hk/tiny/f_hat"] = f
    d["p2/hk/tiny/sweeps"] = np.int64(rp.sweeps)
    np.savez_compressed(os.path.join(HERE, "small.npz"), **d)


def fixture_pa():
    """Preferential attachment n=2000: 8 sampled seeds, LocalGD/GS/SOR."""
    d = {}
    g = rsyn.preferential_attachment(2000, 3, seed=1)
    put_graph(d, "pa2000", g)
    seeds = sample_sources(g, 8, seed=0)
    d["seeds"] = seeds
    om = rls.optimal_omega(0.1)
    for i, s in enumerate(seeds):
        sys_ = rsys.make_ppr_system(g, 0.1, int(s), 1e-6)
        base = dict(graph="pa2000", problem="ppr", alpha=0.1, eps=1e-6, source=int(s))
        put_local(d, f"s{i}/local_gd", *rls.local_gd(sys_), **base)
        if i < 4:
            put_local(d, f"s{i}/local_gs", *rls.local_gs(sys_), **base)
            put_local(d, f"s{i}/local_sor", *rls.local_sor(sys_, omega=om), **base, omega=om)
            put_local(d, f"s{i}/local_ch", *rls.local_ch(sys_), **base)
    np.savez_compressed(os.path.join(HERE, "pa2000.npz"), **d)


def fixture_cora():
    """Config 1: cora-shape R-MAT, 50 seeds, LocalGD PPR alpha=0.1 eps=1e-6."""
    d = {}
    g = to_ref(rmat_graph(2708, 5278, seed=0))
    put_graph(d, "cora", g)
    seeds = sample_sources(g, 50, seed=0)
    d["seeds"] = seeds
    sw, ops, pushes, conv = [], [], [], []
    xs = []
    for i, s in enumerate(seeds):
        sys_ = rsys.make_ppr_system(g, 0.1, int(s), 1e-6)
        st, rp = rls.local_gd(sys_)
        sw.append(rp.sweeps)
        ops.append(rp.total_ops)
        pushes.append(sum(rp.notes["frontier_sizes"]))
        conv.append(rp.converged)
        xs.append(st.x)
        if i < 3:
            put_local(d, f"s{i}/local_gd", st, rp, graph="cora", problem="ppr", alpha=0.1,
                      eps=1e-6, source=int(s))
    d["batch/sweeps"] = np.asarray(sw, dtype=np.int64)
    d["batch/total_ops"] = np.asarray(ops, dtype=np.int64)
    d["batch/pushes"] = np.asarray(pushes, dtype=np.int64)
    d["batch/converged"] = np.asarray(conv)
    d["batch/x"] = np.stack(xs)
    np.savez_compressed(os.path.join(HERE, "cora.npz"), **d)


def fixture_dynamic():
    """Warm-started repair: event_adjust + run_snapshots (dynamic and static)."""
    d = {}
    g0 = rsyn.erdos_renyi(120, 0.05, seed=6)
    put_graph(d, "er120", g0)
    rng = np.random.default_rng(6)
    batches, sim = [], g0
    for _ in range(4):
        batch = []
        for _ in range(10):
            while True:
                u, v = int(rng.integers(sim.n)), int(rng.integers(sim.n))
                if u != v:
                    break
            u, v = min(u, v), max(u, v)
            e = EdgeEvent("delete" if sim.has_edge(u, v) else "insert", u, v)
            batch.append(e)
            sim = apply_event(sim, e)
        batches.append(batch)
    ev = []
    for bi, batch in enumerate(batches):
        for e in batch:
            ev.append((bi, 1 if e.kind == "insert" else 0, e.u, e.v))
    d["events"] = np.asarray(ev, dtype=np.int64)
    alpha, eps = 0.2, 0.2 * 1e-4
    for mode in ("dynamic", "static"):
        pair0 = rdyn.make_pair(g0, alpha, eps, 0)
        reps, pair, gf = rdyn.run_snapshots(g0, batches, pair0, mode=mode)
        d[f"{mode}/p"], d[f"{mode}/r"] = pair.p, pair.r
        d[f"{mode}/sweeps"] = np.asarray([r.sweeps for r in reps], dtype=np.int64)
        d[f"{mode}/total_ops"] = np.asarray([r.total_ops for r in reps], dtype=np.int64)
        d[f"{mode}/ops_accumulated"] = np.asarray([r.notes["ops_accumulated"] for r in reps])
        d[f"{mode}/vol_flat"] = np.concatenate([np.asarray(r.vol_log, dtype=np.int64) for r in reps])
        d[f"{mode}/signs_flat"] = np.concatenate(
            [np.asarray(r.notes["sweep_signs"], dtype=np.int8) for r in reps])
    put_graph(d, "final", gf)
    # single-event adjustments on a converged pair
    g = rsyn.erdos_renyi(50, 0.1, seed=3)
    put_graph(d, "er50", g)
    pair, _ = rdyn.repair(g, rdyn.make_pair(g, 0.2, 1e-4, 0))
    d["adj/p0"], d["adj/r0"] = pair.p, pair.r
    e_ins = EdgeEvent("insert", 0, 49) if not g.has_edge(0, 49) else EdgeEvent("delete", 0, 49)
    a1 = rdyn.event_adjust(g, pair, e_ins)
    d["adj/ev1"] = np.asarray([1 if e_ins.kind == "insert" else 0, e_ins.u, e_ins.v])
    d["adj/p1"], d["adj/r1"] = a1.p, a1.r
    nb = int(g.neighbors(5)[0])
    e_del = EdgeEvent("delete", min(5, nb), max(5, nb))
    a2 = rdyn.event_adjust(g, pair, e_del)
    d["adj/ev2"] = np.asarray([0, e_del.u, e_del.v])
    d["adj/p2"], d["adj/r2"] = a2.p, a2.r
    np.savez_compressed(os.path.join(HERE, "dynamic.npz"), **d)


if __name__ == "__main__":
    fixture_small()
    fixture_pa()
    fixture_cora()
    fixture_dynamic()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
