"""Batched signed solvers on the GPU: LocalCH (PPR / Katz) seed batches and
the resident pair pool (warm-started signed LocalGD after edge events)
against the reference's golden vectors and the CPU oracle.  Integer work
(sweeps, operation counts, convergence / divergence) is identical per seed;
x, p, r agree within 1e-9 relative l1 (the atomic scatter only changes the
summation order)."""

import numpy as np
import pytest

from conftest import golden_graph, load_golden
from helpers import build_system, local_cases, param
from oracle import oracle as O
from paper_2410_21634_b200 import systems as S
from paper_2410_21634_b200.batch import BatchSolver, local_ch_batch
from paper_2410_21634_b200.metrics import sample_sources
from paper_2410_21634_b200.synth import rmat_graph

pytestmark = pytest.mark.gpu
X_RTOL = 1e-9


def _close(a, ref, rtol=X_RTOL):
    return np.abs(a - ref).sum() <= rtol * max(np.abs(ref).sum(), 1e-300)


def _check_seed(out, i, x_ref, n):
    x = out.x_dense(i, n)
    nodes, _ = out.x_sparse(i)
    assert len(np.unique(nodes)) == len(nodes)
    assert set(np.flatnonzero(x_ref).tolist()) <= set(nodes.tolist())
    assert _close(x, x_ref)


@pytest.mark.parametrize("slots", [0, 1, 3])
def test_ch_batch_matches_reference_pa(gpu, pa, slots):
    g = golden_graph(pa, "pa2000")
    keys = [k for k in local_cases(pa) if k.endswith("/local_ch")]
    seeds = np.array([int(param(pa, k, "source")) for k in keys])
    out = local_ch_batch(g, seeds, 0.1, 1e-6, slots=slots)
    for i, k in enumerate(keys):
        assert out.sweeps[i] == pa[f"{k}/sweeps"] and out.total_ops[i] == pa[f"{k}/total_ops"]
        assert out.converged[i] == bool(pa[f"{k}/converged"])
        _check_seed(out, i, pa[f"{k}/x"], g.n)


@pytest.mark.parametrize("key", ["er500/ppr/local_ch", "er60/ppr/local_ch", "er60/katz/local_ch"])
def test_ch_batch_matches_reference_small(gpu, small, key):
    sys_ = build_system(small, key)
    g = sys_.graph
    prob = str(param(small, key, "problem"))
    mu, L = param(small, key, "mu"), param(small, key, "L")
    for relabel in (True, False):
        out = local_ch_batch(g, [sys_.source], sys_.alpha, sys_.eps, problem=prob, mu=mu, L=L,
                             relabel=relabel)
        assert out.sweeps[0] == small[f"{key}/sweeps"]
        assert out.total_ops[0] == small[f"{key}/total_ops"]
        assert out.converged[0] == bool(small[f"{key}/converged"])
        _check_seed(out, 0, small[f"{key}/x"], g.n)


@pytest.mark.parametrize("tail", ["default", "from-round-1", "off"])
@pytest.mark.parametrize("problem", ["ppr", "katz"])
def test_ch_batch_rmat_matches_oracle(gpu, monkeypatch, problem, tail):
    """tail: the CTA-local tail (k_s_tail) at its default trigger, from round 1
    on (nearly the whole solve block-local), or off (round kernel only)."""
    if tail == "from-round-1":
        monkeypatch.setenv("GDIFF_TAIL_T", "1")
        monkeypatch.setenv("GDIFF_TAIL_F", str(1 << 30))
    elif tail == "off":
        monkeypatch.setenv("GDIFF_TAIL", "0")
    from paper_2410_21634_b200.graph import spectral_norm_estimate
    g = rmat_graph(20000, 150000, seed=5)
    seeds = sample_sources(g, 40, seed=2)
    if problem == "ppr":
        alpha, eps, lam = 0.1, 1e-6, None
        mk = lambda s: S.make_ppr_system(g, alpha, s, eps)
    else:
        lam = spectral_norm_estimate(g, iters=200, seed=0)
        alpha, eps = 1.0 / (lam + 1.0), 1e-6
        mk = lambda s: S.make_katz_system(g, alpha, s, eps, lam_hat=lam)
    out = local_ch_batch(g, seeds, alpha, eps, problem=problem, lam_hat=lam, slots=16)
    for i, s in enumerate(seeds):
        ref = O.local_ch(mk(int(s)), record_trace=False) if problem == "ppr" else \
            O.local_ch(mk(int(s)), *_katz_bounds(g, alpha, lam), record_trace=False)
        assert out.sweeps[i] == ref["sweeps"] and out.total_ops[i] == ref["total_ops"], i
        assert out.converged[i] == bool(ref["converged"])
        _check_seed(out, i, ref["x"], g.n)


def _katz_bounds(g, alpha, lam):
    lam = min(max(lam, 1e-12), float(g.d_max))
    return 1.0 - alpha * lam, 1.0 + alpha * lam


@pytest.mark.parametrize("tail", ["default", "from-round-1"])
def test_ch_batch_divergence_and_sweep_cap(gpu, monkeypatch, tail):
    """Bad bounds make LocalCH diverge (abort at l1 > 10 ||b||_1); a sweep cap
    stops unconverged -- both per seed exactly as the reference (also with the
    CTA-local tail running nearly the whole solve)."""
    if tail == "from-round-1":
        monkeypatch.setenv("GDIFF_TAIL_T", "1")
        monkeypatch.setenv("GDIFF_TAIL_F", str(1 << 30))
    g = rmat_graph(5000, 30000, seed=3)
    seeds = sample_sources(g, 12, seed=4)
    solver = BatchSolver(g, 0.1, 1e-6, slots=5, method="local-ch", mu=0.6, L=0.7,
                         max_sweeps=400)
    out = solver.solve(seeds)
    diverged = 0
    for i, s in enumerate(seeds):
        ref = O.local_ch(S.make_ppr_system(g, 0.1, int(s), 1e-6), mu=0.6, L=0.7, max_sweeps=400,
                         record_trace=False)
        assert out.sweeps[i] == ref["sweeps"] and out.total_ops[i] == ref["total_ops"]
        assert out.converged[i] == bool(ref["converged"])
        diverged += int(ref["diverged"])
    assert diverged > 0
    capped = local_ch_batch(g, seeds, 0.1, 1e-6, max_sweeps=4)
    assert (capped.sweeps == 4).all() and not capped.converged.any()
    solver.close()


def test_ch_batch_solver_reuse(gpu):
    g = rmat_graph(5000, 30000, seed=9)
    seeds = sample_sources(g, 30, seed=1)
    solver = BatchSolver(g, 0.15, 1e-5, slots=8, method="local-ch", max_sweeps=2000)
    a = solver.solve(seeds)
    a = {k: np.array(getattr(a, k)) for k in ("sweeps", "total_ops", "pushes")}
    b = solver.solve(seeds[::-1].copy())
    assert np.array_equal(b.total_ops[::-1], a["total_ops"])
    assert np.array_equal(b.sweeps[::-1], a["sweeps"])
    solver.close()


# ---- resident pair pool (config 5, batched) --------------------------------

def _warm_ref(g, p, r, alpha, eps):
    w = S.arc_weights_for(g, 1.0 - alpha, "gen", 0.0)
    th = S.theta_vector(g, eps)
    return O.local_gd_warm(g.offsets, g.targets, w, th, p, r, signed=True, record_trace=False)


def _pool_against_oracle(g, batches, sources, alpha, eps):
    from paper_2410_21634_b200.dynamic import PairPool, event_adjust_many
    from paper_2410_21634_b200.graph import apply_events
    pool = PairPool(g, sources, alpha, eps)
    n = g.n
    for i, s in enumerate(sources):
        p, r = np.zeros(n), np.zeros(n)
        r[s] = alpha
        ref = _warm_ref(g, p, r, alpha, eps)
        assert pool.last["sweeps"][i] == ref["sweeps"] and pool.last["total_ops"][i] == ref["total_ops"]
        got = pool.pair(i)
        assert _close(got.p, p) and _close(got.r, r)
    for batch in batches:
        before = [pool.pair(i) for i in range(len(sources))]
        st = pool.update(batch)
        g2 = apply_events(g, batch)
        for i in range(len(sources)):
            adj = event_adjust_many(g, before[i], batch)
            p, r = adj.p.copy(), adj.r.copy()
            ref = _warm_ref(g2, p, r, alpha, eps)
            assert st["sweeps"][i] == ref["sweeps"] and st["total_ops"][i] == ref["total_ops"]
            assert st["converged"][i] == int(ref["converged"])
            got = pool.pair(i)
            assert _close(got.p, p) and _close(got.r, r, rtol=1e-7)
            assert np.abs(got.consistency_residual(g2)).max() <= 1e-9
        g = g2
    pool.close()


def test_pair_pool_dynamic_fixture(gpu, dyn):
    from paper_2410_21634_b200.graph import EdgeEvent
    g = golden_graph(dyn, "er120")
    ev = dyn["events"]
    batches = [[EdgeEvent("insert" if k else "delete", int(u), int(v)) for b, k, u, v in ev if b == bi]
               for bi in range(int(ev[:, 0].max()) + 1)]
    sources = [int(s) for s in np.flatnonzero(g.degrees > 0)[:9]]
    _pool_against_oracle(g, batches, sources, 0.2, 0.2 * 1e-4)


def test_pair_pool_rmat_stream(gpu):
    from paper_2410_21634_b200.graph import EdgeEvent, apply_events
    g = rmat_graph(6000, 40000, seed=11)
    rng = np.random.default_rng(0)
    batches, sim = [], g
    for _ in range(4):
        b = []
        for _ in range(60):
            u, v = sorted(rng.choice(g.n, 2, replace=False).tolist())
            if any((e.u, e.v) == (u, v) for e in b):
                continue
            b.append(EdgeEvent("delete" if sim.has_edge(u, v) else "insert", u, v))
        sim = apply_events(sim, b)
        batches.append(b)
    sources = sample_sources(g, 24, seed=3).tolist()
    _pool_against_oracle(g, batches, sources, 0.15, 1e-5)


def test_device_graph_edit_matches_host(gpu, small):
    """gd_graph_apply_events == graph.apply_events (canonical CSR), including
    repeated edits of one edge, deletes down to isolated nodes, and the
    reference's errors on invalid events."""
    from paper_2410_21634_b200.device import DeviceGraph
    from paper_2410_21634_b200.graph import EdgeEvent, GraphStructureError, apply_events
    from paper_2410_21634_b200._lib import GdiffError
    rng = np.random.default_rng(7)
    for g in (golden_graph(small, "er60"), rmat_graph(3000, 20000, seed=2)):
        dg = DeviceGraph.from_host(g)
        sim = g
        for _ in range(3):
            evs = []
            for _ in range(300):
                u, v = sorted(rng.choice(min(g.n, 80), 2, replace=False).tolist())
                e = EdgeEvent("delete" if sim.has_edge(u, v) else "insert", u, v)
                evs.append(e)
                sim = apply_events(sim, [e])
            host = apply_events(g, evs)
            dn = dg.apply_events(evs)
            back = dn.to_host()
            assert np.array_equal(back.offsets, host.offsets)
            assert np.array_equal(back.targets, host.targets)
            assert dn.d_max == host.d_max and dn.n_arcs == host.targets.shape[0]
            dg.close()
            dg, g = dn, host
        bad = [EdgeEvent("delete", 0, 1)] if not g.has_edge(0, 1) else [EdgeEvent("insert", 0, 1)]
        with pytest.raises(GdiffError):
            dg.apply_events(bad)
        with pytest.raises(GraphStructureError):
            apply_events(g, bad * 70)
        dg.close()


@pytest.mark.parametrize("group", ["1", "4"])
def test_signed_grouped_mode(gpu, monkeypatch, group):
    """LocalCH batches and the pair pool in the slot-grouped mode."""
    monkeypatch.setenv("GDIFF_SLOT_GROUP", group)
    monkeypatch.setenv("GDIFF_GROUP_MIN", "0")  # every round grouped
    g = rmat_graph(20000, 150000, seed=5)
    seeds = sample_sources(g, 24, seed=2)
    out = local_ch_batch(g, seeds, 0.1, 1e-6, slots=10)
    for i, s in enumerate(seeds):
        ref = O.local_ch(S.make_ppr_system(g, 0.1, int(s), 1e-6), record_trace=False)
        assert out.sweeps[i] == ref["sweeps"] and out.total_ops[i] == ref["total_ops"], i
        _check_seed(out, i, ref["x"], g.n)
    from paper_2410_21634_b200.graph import EdgeEvent, apply_events
    rng = np.random.default_rng(1)
    b = []
    for _ in range(50):
        u, v = sorted(rng.choice(g.n, 2, replace=False).tolist())
        if not g.has_edge(u, v) and all((e.u, e.v) != (u, v) for e in b):
            b.append(EdgeEvent("insert", u, v))
    _pool_against_oracle(g, [b], sample_sources(g, 12, seed=4).tolist(), 0.15, 1e-5)


def test_pair_pool_push_is_the_reference_run_snapshots(gpu, dyn):
    """PairPool(method="push"): the reference's own repair (signed FIFO push,
    src/dynamic.py:131-162) for every resident pair -- the golden dynamic
    stream of the reference itself bit for bit (p, r, per-snapshot sweeps and
    operation counts), and every source of an R-MAT stream bitwise with the
    per-pair run_snapshots loop (src/dynamic.py:165-196)."""
    from paper_2410_21634_b200.dynamic import PairPool, make_pair, run_snapshots
    from paper_2410_21634_b200.graph import EdgeEvent, apply_events
    g0 = golden_graph(dyn, "er120")
    ev = dyn["events"]
    batches = [[EdgeEvent("insert" if k else "delete", int(u), int(v))
                for b, k, u, v in ev if b == bi] for bi in range(int(ev[:, 0].max()) + 1)]
    pool = PairPool(g0, [0], 0.2, 0.2 * 1e-4, method="push")
    sweeps, ops = [int(pool.last["sweeps"][0])], [int(pool.last["total_ops"][0])]
    for b in batches:
        st = pool.update(b)
        sweeps.append(int(st["sweeps"][0]))
        ops.append(int(st["total_ops"][0]))
    got = pool.pair(0)
    assert np.array_equal(got.p, dyn["dynamic/p"]) and np.array_equal(got.r, dyn["dynamic/r"])
    assert sweeps == dyn["dynamic/sweeps"].tolist() and ops == dyn["dynamic/total_ops"].tolist()
    pool.close()
    # R-MAT stream, many sources at once
    g = rmat_graph(6000, 40000, seed=11)
    rng = np.random.default_rng(0)
    stream, sim = [], g
    for _ in range(3):
        b = []
        for _ in range(80):
            u, v = sorted(rng.choice(g.n, 2, replace=False).tolist())
            if any((e.u, e.v) == (u, v) for e in b):
                continue
            b.append(EdgeEvent("delete" if sim.has_edge(u, v) else "insert", u, v))
        sim = apply_events(sim, b)
        stream.append(b)
    sources = sample_sources(g, 24, seed=3).tolist()
    alpha, eps = 0.15, 0.15 * 1e-5
    pool = PairPool(g, sources, alpha, eps, method="push")
    stats = [pool.last] + [pool.update(b) for b in stream]
    for i, s in enumerate(sources):
        reps, pair, _ = run_snapshots(g, stream, make_pair(g, alpha, eps, int(s)), mode="dynamic")
        assert [int(st["sweeps"][i]) for st in stats] == [r.sweeps for r in reps]
        assert [int(st["total_ops"][i]) for st in stats] == [r.total_ops for r in reps]
        got = pool.pair(i)
        assert np.array_equal(got.p, pair.p) and np.array_equal(got.r, pair.r)
    pool.close()


# ---- LocalHB (heavy-ball momentum; restatement, tests/golden/hb.npz) -------

def test_local_hb_single_bitwise(gpu):
    """gd_local_hb == the reference's own _SweepDriver with heavy-ball
    coefficients (golden hb.npz), bit for bit: x, r, sweeps, ops, logs."""
    from conftest import load_golden
    from paper_2410_21634_b200.graph import CsrGraph
    from paper_2410_21634_b200.local_solvers import local_hb
    d = load_golden("hb.npz")
    g = CsrGraph(n=int(d["graph/n"]), offsets=d["graph/offsets"], targets=d["graph/targets"])
    for i in range(int(d["cases"])):
        k = f"c{i}"
        prob, alpha, eps, s = str(d[f"{k}/problem"]), float(d[f"{k}/alpha"]), float(d[f"{k}/eps"]), int(d[f"{k}/source"])
        sys_ = (S.make_ppr_system(g, alpha, s, eps) if prob == "ppr"
                else S.make_katz_system(g, alpha, s, eps, lam_hat=0.0))
        st, rep = local_hb(sys_, mu=float(d[f"{k}/mu"]), L=float(d[f"{k}/L"]))
        assert np.array_equal(st.x, d[f"{k}/x"]) and np.array_equal(st.r, d[f"{k}/r"]), k
        assert rep.sweeps == d[f"{k}/sweeps"] and rep.total_ops == d[f"{k}/total_ops"], k
        assert np.array_equal(np.asarray(rep.vol_log), d[f"{k}/vol_log"]), k
        np.testing.assert_allclose(rep.residual_l1_trace, d[f"{k}/l1_log"], rtol=1e-12)


@pytest.mark.parametrize("problem", ["ppr", "katz"])
def test_local_hb_batch_matches_oracle(gpu, problem):
    """Batched LocalHB (signed round kernel, constant coefficients): sweeps,
    ops, pushes, convergence identical to the restatement per seed, x to 1e-9."""
    from paper_2410_21634_b200.batch import BatchSolver
    g = rmat_graph(20000, 150000, seed=5)
    seeds = sample_sources(g, 32, seed=4)
    if problem == "ppr":
        alpha, mu, L = 0.1, 0.1, 1.9
    else:
        alpha = 0.9 / float(g.degrees.max())
        lam = float(g.degrees.max())
        mu, L = 1.0 - alpha * lam, 1.0 + alpha * lam
    solver = BatchSolver(g, alpha, 1e-6, method="local-hb", problem=problem, mu=mu, L=L, slots=8)
    out = solver.solve(seeds)
    solver.close()
    ref = O.batch_local_ch(g, alpha, 1e-6, seeds, 8, mu=mu, L=L, problem=problem, hb=True,
                           gpu=out, topk=50)
    assert np.array_equal(out.sweeps, ref["sweeps"])
    assert np.array_equal(out.total_ops, ref["total_ops"])
    assert np.array_equal(out.converged, ref["converged"])
    assert (ref["x_l1_rel"] <= 1e-9).all() and ref["topk_identical_up_to_ties"].all()
