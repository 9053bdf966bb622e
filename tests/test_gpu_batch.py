"""Batched multi-seed LocalGD on the GPU against the reference (golden
vectors) and the CPU oracle: identical per-seed sweeps, operation counts
and push counts (the frontier sets), x within 1e-9 relative l1 (north-star
tolerance; the atomic scatter only changes summation order)."""

import numpy as np
import pytest

from conftest import golden_graph
from oracle import oracle as O
from paper_2410_21634_b200 import systems as S
from paper_2410_21634_b200.batch import BatchSolver, local_gd_batch
from paper_2410_21634_b200.metrics import sample_sources
from paper_2410_21634_b200.synth import rmat_graph

pytestmark = pytest.mark.gpu
X_RTOL = 1e-9


def _check_x(out, i, x_ref):
    n = x_ref.shape[0]
    x = out.x_dense(i, n)
    nodes, _ = out.x_sparse(i)
    assert len(np.unique(nodes)) == len(nodes)
    assert set(nodes.tolist()) == set(np.flatnonzero(x_ref).tolist())
    assert np.abs(x - x_ref).sum() <= X_RTOL * np.abs(x_ref).sum()
    top = np.argsort(-x_ref, kind="stable")[:10]
    assert np.array_equal(np.argsort(-x, kind="stable")[:10], top)


# one CTA per seed (small graphs) / the round kernel with slots refilled in-kernel
# (large graphs) / the same kernel in synchronous waves (GDIFF_STREAM=0)
MODES = ["cta", "cta-global", "stream", "waves"]


def set_mode(monkeypatch, mode):
    """cta: one CTA per seed (shared-memory state when the graph fits);
    cta-global: the same with the state in HBM; stream / waves: round kernel."""
    cta = mode in ("cta", "cta-global")
    monkeypatch.setenv("GDIFF_BATCH_MODE", "cta" if cta else "rounds")
    if mode == "cta-global":
        monkeypatch.setenv("GDIFF_CTA_SMEM", "0")
    else:
        monkeypatch.delenv("GDIFF_CTA_SMEM", raising=False)
    if cta:
        monkeypatch.delenv("GDIFF_STREAM", raising=False)
    else:
        monkeypatch.setenv("GDIFF_STREAM", "0" if mode == "waves" else "1")


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("slots,relabel", [(0, True), (1, True), (7, False), (64, True), (64, False)])
def test_cora_config1_batch(gpu, cora, monkeypatch, mode, slots, relabel):
    set_mode(monkeypatch, mode)
    g = golden_graph(cora, "cora")
    seeds = cora["seeds"]
    out = local_gd_batch(g, seeds, 0.1, 1e-6, slots=slots, relabel=relabel)
    assert np.array_equal(out.sweeps, cora["batch/sweeps"])
    assert np.array_equal(out.total_ops, cora["batch/total_ops"])
    assert np.array_equal(out.pushes, cora["batch/pushes"])
    assert out.converged.all()
    for i in range(len(seeds)):
        _check_x(out, i, cora["batch/x"][i])


def test_pa_batch_matches_reference(gpu, pa):
    g = golden_graph(pa, "pa2000")
    out = local_gd_batch(g, pa["seeds"], 0.1, 1e-6, slots=3)
    for i in range(len(pa["seeds"])):
        k = f"s{i}/local_gd"
        assert out.sweeps[i] == pa[f"{k}/sweeps"] and out.total_ops[i] == pa[f"{k}/total_ops"]
        assert out.pushes[i] == pa[f"{k}/frontier_sizes"].sum()
        _check_x(out, i, pa[f"{k}/x"])


@pytest.mark.parametrize("mode", MODES + ["waves-notail", "waves-tailcap"])
def test_rmat_batch_matches_oracle(gpu, monkeypatch, mode):
    """waves-notail: the round kernel without CTA-local tails; waves-tailcap: tail
    lists of 4 entries per slot, so a tail overflows and the solve is redone
    without tails (the results must not show it)."""
    if mode.startswith("waves-"):
        monkeypatch.setenv("GDIFF_TAIL" if mode == "waves-notail" else "GDIFF_TAIL_CAP",
                           "0" if mode == "waves-notail" else "4")
        mode = "waves"
    set_mode(monkeypatch, mode)
    g = rmat_graph(20000, 150000, seed=5)
    seeds = sample_sources(g, 48, seed=0)
    ref = O.batch_local_gd(g, 0.1, 1e-6, seeds, threads=8)
    out = local_gd_batch(g, seeds, 0.1, 1e-6, slots=16)
    assert np.array_equal(out.sweeps, ref["sweeps"])
    assert out.converged.all()
    assert np.array_equal(out.total_ops, ref["total_ops"])
    assert np.array_equal(out.pushes, ref["pushes"])
    xs = np.array([out.x_sparse(i)[1].sum() for i in range(len(seeds))])
    np.testing.assert_allclose(xs, ref["xsum"], rtol=1e-12)


@pytest.mark.parametrize("mode", MODES)
def test_solver_reuse_and_device_path(gpu, monkeypatch, mode):
    import torch
    set_mode(monkeypatch, mode)
    g = rmat_graph(5000, 30000, seed=9)
    seeds = sample_sources(g, 40, seed=1)
    solver = BatchSolver(g, 0.15, 1e-5, slots=8)
    a = solver.solve(seeds)
    a = {k: np.array(getattr(a, k)) for k in ("sweeps", "total_ops", "pushes")}
    b = solver.solve(seeds[::-1].copy())
    assert np.array_equal(b.total_ops[::-1], a["total_ops"])
    d = solver.solve_device(torch.as_tensor(seeds, device="cuda"))
    assert np.array_equal(d["total_ops"].cpu().numpy(), a["total_ops"])
    assert np.array_equal(d["sweeps"].cpu().numpy(), a["sweeps"])
    # waves: init, round kernel, CTA-local tail, extract, reset per wave of 8
    assert d["kernel_launches"] == {"waves": 5 * 5, "stream": 1 + 5, "cta": 1, "cta-global": 1}[mode]
    # (5,000 nodes: one seed's state fits in shared memory)
    assert solver.mode == {"waves": "rounds", "stream": "stream", "cta": "cta-smem",
                           "cta-global": "cta"}[mode]
    assert solver.last_kernel_ms > 0.0


@pytest.mark.parametrize("mode", MODES)
def test_edge_cases(gpu, monkeypatch, mode):
    from paper_2410_21634_b200.graph import from_edges
    set_mode(monkeypatch, mode)
    # isolated nodes, a leaf, max_sweeps cap, empty batch
    g = from_edges(6, [(0, 1), (1, 2), (2, 0), (3, 4)])
    out = local_gd_batch(g, [0, 3], 0.2, 1e-9, max_sweeps=2)
    assert (out.sweeps == 2).all() and not out.converged.any()
    out = local_gd_batch(g, np.empty(0, np.int64), 0.2, 1e-4)
    assert out.sweeps.shape == (0,)
    with pytest.raises(ValueError):
        local_gd_batch(g, [5], 0.2, 1e-4)  # degree-0 source
    # eps large enough that the seed itself is inactive: zero sweeps
    out = local_gd_batch(g, [0], 0.2, 10.0)
    assert out.sweeps[0] == 0 and out.total_ops[0] == 0 and out.converged[0]


def test_device_generator_equals_host(gpu):
    from paper_2410_21634_b200.gen import rmat_csr_device, rmat_csr_device_big
    for n, m, seed in ((2708, 5278, 0), (20000, 150000, 5)):
        h = rmat_graph(n, m, seed=seed)
        for fn, kw in ((rmat_csr_device, {}), (rmat_csr_device_big, {"buckets": 7, "chunk": 50000})):
            row, col = fn(n, m, seed=seed, **kw)
            assert np.array_equal(row.cpu().numpy(), h.offsets), fn.__name__
            assert np.array_equal(col.cpu().numpy().astype(np.int64), h.targets), fn.__name__


# ---- batched FIFO (LocalSOR / LocalGS): bit-identical per seed ------------

@pytest.mark.parametrize("mode", ["win", "warp"])  # exact windows (CTA per seed) / warp chain
@pytest.mark.parametrize("omega", [1.0, 1.39301, 0.7])
@pytest.mark.parametrize("slots", [0, 5])
def test_sor_batch_bitwise_vs_oracle(gpu, cora, monkeypatch, mode, omega, slots):
    monkeypatch.setenv("GDIFF_SOR_MODE", mode)
    from paper_2410_21634_b200.batch import local_sor_batch
    from paper_2410_21634_b200.systems import make_ppr_system
    g = golden_graph(cora, "cora")
    seeds = cora["seeds"][:24]
    out = local_sor_batch(g, seeds, 0.1, 1e-6, omega=omega, slots=slots)
    for i, s in enumerate(seeds):
        ref = O.local_sor(make_ppr_system(g, 0.1, int(s), 1e-6), omega)
        assert out.sweeps[i] == ref["sweeps"] and out.total_ops[i] == ref["total_ops"]
        assert bool(out.converged[i]) == ref["converged"]
        assert np.array_equal(out.x_dense(i, g.n), ref["x"]), (i, s)


def test_sor_batch_matches_reference_golden(gpu, pa):
    from paper_2410_21634_b200.batch import local_sor_batch
    g = golden_graph(pa, "pa2000")
    seeds = pa["seeds"][:4]
    for meth, omega in (("local_gs", 1.0), ("local_sor", float(pa["s0/local_sor/param/omega"]))):
        out = local_sor_batch(g, seeds, 0.1, 1e-6, omega=omega, slots=2)
        for i in range(4):
            k = f"s{i}/{meth}"
            assert out.sweeps[i] == pa[f"{k}/sweeps"] and out.total_ops[i] == pa[f"{k}/total_ops"]
            assert np.array_equal(out.x_dense(i, g.n), pa[f"{k}/x"])


def test_sor_batch_max_sweeps(gpu):
    from paper_2410_21634_b200.batch import local_sor_batch
    from paper_2410_21634_b200.graph import from_edges
    g = from_edges(4, [(0, 1), (1, 2), (2, 0)])
    out = local_sor_batch(g, [0, 1], 0.2, 1e-9, max_sweeps=2)
    assert (out.sweeps == 2).all() and not out.converged.any()


# ---- batched heat kernel (layered stage sweeps) ---------------------------

@pytest.mark.parametrize("tau", [0.5, 1.0, 5.0])
def test_hk_batch_matches_reference(gpu, small, tau):
    from paper_2410_21634_b200.batch import local_hk_batch
    g = golden_graph(small, "er60")
    out = local_hk_batch(g, [0, 0, 0], tau, 1e-4, slots=2)
    k = f"er60/hk/tau{tau}"
    for i in range(3):
        assert out.sweeps[i] == small[f"{k}/sweeps"] and out.total_ops[i] == small[f"{k}/total_ops"]
        f = small[f"{k}/f_hat"]
        assert np.abs(out.x_dense(i, g.n) - f).sum() <= X_RTOL * np.abs(f).sum()


@pytest.mark.parametrize("tau,eps", [(1.0, 1e-5), (5.0, 1e-6), (10.0, 1e-6)])
def test_hk_batch_matches_oracle(gpu, tau, eps):
    from paper_2410_21634_b200.batch import local_hk_batch
    g = rmat_graph(20000, 150000, seed=2)
    seeds = sample_sources(g, 20, seed=3)
    for slots, relabel in ((8, True), (3, False)):
        out = local_hk_batch(g, seeds, tau, eps, slots=slots, relabel=relabel)
        for i, s in enumerate(seeds):
            ref = O.local_hk(g, tau, int(s), eps)
            assert out.sweeps[i] == ref["sweeps"] and out.total_ops[i] == ref["total_ops"], i
            assert out.converged[i]
            f = ref["f_hat"]
            x = out.x_dense(i, g.n)
            assert np.abs(x - f).sum() <= X_RTOL * np.abs(f).sum()
            assert set(np.flatnonzero(f).tolist()) <= set(out.x_sparse(i)[0].tolist())


# ---- edge cases -------------------------------------------------------------

@pytest.mark.parametrize("mode", MODES)
def test_batch_edge_cases(gpu, monkeypatch, mode):
    """Empty batches, duplicate seeds, sweep caps and a frontier-capacity
    overflow (reported as an error, the solver stays usable)."""
    from paper_2410_21634_b200._lib import GdiffError
    set_mode(monkeypatch, mode)
    g = rmat_graph(5000, 30000, seed=4)
    seeds = sample_sources(g, 24, seed=2)
    for method in ("local-gd", "local-ch", "local-sor"):
        solver = BatchSolver(g, 0.1, 1e-5, slots=8, method=method, max_sweeps=1_000_000)
        empty = solver.solve(np.empty(0, np.int64))
        assert empty.sweeps.shape == (0,) and empty.x_nodes.shape == (0,)
        dup = np.array([seeds[0]] * 5 + [seeds[1]] * 3)
        out = solver.solve(dup)
        assert len(set(out.total_ops[:5].tolist())) == 1 and len(set(out.sweeps[5:].tolist())) == 1
        assert np.array_equal(out.x_dense(0, g.n), out.x_dense(4, g.n)) or method == "local-ch" \
            or np.abs(out.x_dense(0, g.n) - out.x_dense(4, g.n)).sum() <= 1e-12
        solver.close()
    # sweep cap: identical to the reference's max_sweeps behaviour
    capped = local_gd_batch(g, seeds, 0.1, 1e-7, max_sweeps=3, slots=8)
    ref = O.batch_local_gd(g, 0.1, 1e-7, seeds, threads=4, max_sweeps=3)
    assert np.array_equal(capped.sweeps, ref["sweeps"]) and np.array_equal(capped.total_ops, ref["total_ops"])
    assert np.array_equal(capped.converged, ref["converged"])
    # capacity overflow, then a normal solve on the same solver
    tiny = BatchSolver(g, 0.1, 1e-6, slots=8, frontier_cap=64)
    with pytest.raises(GdiffError):
        tiny.solve(seeds)
    tiny.close()
    solver = BatchSolver(g, 0.1, 1e-6, slots=8)
    a = solver.solve(seeds)
    ref = O.batch_local_gd(g, 0.1, 1e-6, seeds, threads=4)
    assert np.array_equal(a.total_ops, ref["total_ops"])
    solver.close()


def test_batch_rejects_bad_input(gpu):
    g = rmat_graph(2000, 8000, seed=1)
    iso = int(np.flatnonzero(g.degrees == 0)[0]) if (g.degrees == 0).any() else None
    with pytest.raises(ValueError):
        local_gd_batch(g, [g.n], 0.1, 1e-6)
    if iso is not None:
        with pytest.raises(ValueError):
            local_gd_batch(g, [iso], 0.1, 1e-6)
    with pytest.raises(ValueError):
        BatchSolver(g, 1.5, 1e-6)
    with pytest.raises(ValueError):
        BatchSolver(g, 0.1, 1e-6, method="local-sor", omega=2.5)
    with pytest.raises(ValueError):
        BatchSolver(g, 0.1, 1e-6, method="local-ch", mu=0.5, L=0.4)


@pytest.mark.parametrize("group", ["1", "3"])
def test_grouped_mode_matches_oracle(gpu, monkeypatch, group):
    """Slot-grouped frontier + windowed phase B (the mode large graphs use,
    forced here on a small one) gives the reference's integer work, for
    LocalGD and the heat kernel."""
    from paper_2410_21634_b200.batch import local_hk_batch
    monkeypatch.setenv("GDIFF_SLOT_GROUP", group)
    monkeypatch.setenv("GDIFF_BATCH_MODE", "rounds")
    monkeypatch.setenv("GDIFF_GROUP_MIN", "0")  # every round grouped
    g = rmat_graph(20000, 150000, seed=5)
    seeds = sample_sources(g, 40, seed=0)
    ref = O.batch_local_gd(g, 0.1, 1e-6, seeds, threads=8)
    out = local_gd_batch(g, seeds, 0.1, 1e-6, slots=16)
    assert np.array_equal(out.sweeps, ref["sweeps"]) and np.array_equal(out.total_ops, ref["total_ops"])
    assert np.array_equal(out.pushes, ref["pushes"])
    xs = np.array([out.x_sparse(i)[1].sum() for i in range(len(seeds))])
    np.testing.assert_allclose(xs, ref["xsum"], rtol=1e-12)
    hk = local_hk_batch(g, seeds[:12], 5.0, 1e-6, slots=5)
    for i, s in enumerate(seeds[:12]):
        r = O.local_hk(g, 5.0, int(s), 1e-6)
        assert hk.sweeps[i] == r["sweeps"] and hk.total_ops[i] == r["total_ops"]
        f = r["f_hat"]
        assert np.abs(hk.x_dense(i, g.n) - f).sum() <= X_RTOL * np.abs(f).sum()


@pytest.mark.parametrize("method", ["local-gd", "local-ch", "local-sor"])
def test_batch_sparse_r(gpu, method):
    """want_r: each seed's final residual as a sparse vector, against the
    CPU oracle's dense r (bitwise for the FIFO batch, 1e-9 otherwise)."""
    g = rmat_graph(20000, 150000, seed=6)
    seeds = sample_sources(g, 12, seed=1)
    solver = BatchSolver(g, 0.1, 1e-6, slots=5, method=method, want_r=True, max_sweeps=100000)
    out = solver.solve(seeds)
    for i, s in enumerate(seeds):
        sys_ = S.make_ppr_system(g, 0.1, int(s), 1e-6)
        ref = (O.local_gd(sys_, record_trace=False) if method == "local-gd" else
               O.local_ch(sys_, record_trace=False) if method == "local-ch" else
               O.local_sor(sys_, 1.0))
        r = out.r_dense(i, g.n)
        nodes, _ = out.r_sparse(i)
        assert len(np.unique(nodes)) == len(nodes)
        if method == "local-sor":
            assert np.array_equal(r, ref["r"])
        else:
            assert np.abs(r - ref["r"]).sum() <= 1e-9 * np.abs(ref["r"]).sum() + 1e-300
            assert set(np.flatnonzero(ref["r"]).tolist()) <= set(nodes.tolist())
    solver.close()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", MODES)
def test_host_entry_streams_x_per_wave(gpu, monkeypatch, mode):
    """gd_batch_solve_host copies each finished wave's sparse x while the next
    wave runs: the host result equals a device-path solve per seed, on a cold
    call (host buffers too small: capacity path) and on warm calls."""
    import torch
    set_mode(monkeypatch, mode)
    g = rmat_graph(20000, 150000, seed=3)
    seeds = sample_sources(g, 70, seed=4)
    solver = BatchSolver(g, 0.1, 1e-6, slots=8)
    for pinned in (False, True, True):
        out = {"pinned": pinned}
        h = solver.solve(seeds, out=out)
        d = solver.solve_device(torch.as_tensor(seeds, device="cuda"))
        assert h.x_nodes.shape[0] == d["x_total"]
        off, cnt = d["x_offset"].cpu().numpy(), d["x_count"].cpu().numpy()
        dn, dv = d["x_nodes"].cpu().numpy(), d["x_vals"].cpu().numpy()
        assert np.array_equal(h.x_count, cnt)
        for i in range(len(seeds)):  # pool positions are per call in the CTA mode
            a = np.argsort(h.x_nodes[h.x_offset[i]:h.x_offset[i] + cnt[i]], kind="stable")
            b = np.argsort(dn[off[i]:off[i] + cnt[i]], kind="stable")
            assert np.array_equal(h.x_nodes[h.x_offset[i]:][:cnt[i]][a], dn[off[i]:][:cnt[i]][b])
            # fp64 atomics: values agree to rounding between two solves
            np.testing.assert_allclose(h.x_vals[h.x_offset[i]:][:cnt[i]][a],
                                       dv[off[i]:][:cnt[i]][b], rtol=1e-9, atol=1e-15)
    solver.close()


@pytest.mark.parametrize("mode", ["cta", "waves"])
def test_batch_sweep_logs_are_the_reference_report(gpu, monkeypatch, mode):
    """log_sweeps: each seed's LocalReport fields from a batched solve --
    vol_log and frontier_sizes identical to the reference's local_gd, gamma_log
    and the l1 trace to rounding (src/reports.py:51-79, local_solvers.py:448-467)."""
    set_mode(monkeypatch, mode)
    g = rmat_graph(20000, 150000, seed=5)
    seeds = sample_sources(g, 24, seed=3)
    solver = BatchSolver(g, 0.1, 1e-6, slots=8, log_sweeps=256)
    out = solver.solve(seeds)
    solver.close()
    for i, s in enumerate(seeds):
        ref = O.local_gd(S.make_ppr_system(g, 0.1, int(s), 1e-6))
        rep = out.report(i)
        assert rep.sweeps == ref["sweeps"] and rep.total_ops == ref["total_ops"]
        assert rep.vol_log == [int(v) for v in ref["vol_log"]]
        assert rep.notes["frontier_sizes"] == [int(v) for v in ref["frontier_sizes"]]
        np.testing.assert_allclose(rep.gamma_log, ref["gamma_log"], rtol=1e-12)
        np.testing.assert_allclose(rep.residual_l1_trace, ref["l1_log"], rtol=1e-12, atol=1e-300)
