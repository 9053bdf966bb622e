"""GPU parity: the CUDA path through the C ABI against the reference's golden
vectors and the CPU oracle.  Integer work (sweeps, operation counts,
frontier traces) and x / r are bit-identical for the single-system solvers;
residual-l1 / gamma logs (device reductions) agree to 1e-12 relative."""

import numpy as np
import pytest

from conftest import golden_graph, load_golden
from helpers import assert_matches, build_system, local_cases, method_of, report_dict, solver_kwargs
from paper_2410_21634_b200 import local_solvers as LS
from paper_2410_21634_b200 import systems as S
from paper_2410_21634_b200.global_solvers import GlobalConfig, gradient_descent

pytestmark = pytest.mark.gpu
FIXTURES = ["small.npz", "pa2000.npz", "cora.npz"]


def _gpu_run(d, key):
    sys_ = build_system(d, key)
    m, kw = method_of(key), solver_kwargs(d, key)
    if m == "local_gd":
        return report_dict(*LS.local_gd(sys_, **kw))
    if m == "local_ch":
        return report_dict(*LS.local_ch(sys_, **kw))
    if m == "local_gs" or m.startswith("local_gs_"):
        return report_dict(*LS.local_gs(sys_, **kw))
    if m.startswith("local_sor"):
        return report_dict(*LS.local_sor(sys_, **kw))
    raise ValueError(m)


@pytest.mark.parametrize("fixture", FIXTURES)
def test_local_solvers_match_reference(gpu, fixture):
    d = load_golden(fixture)
    for key in local_cases(d):
        assert_matches(d, key, _gpu_run(d, key), logs_exact=False)


@pytest.mark.parametrize("tau", [0.5, 1.0, 5.0])
def test_heat_kernel_matches_reference(gpu, small, tau):
    g = golden_graph(small, "er60")
    f, rep = LS.local_hk(g, tau, 0, 1e-4)
    k = f"er60/hk/tau{tau}"
    assert np.array_equal(f, small[f"{k}/f_hat"])
    assert rep.sweeps == small[f"{k}/sweeps"] and rep.total_ops == small[f"{k}/total_ops"]
    assert rep.vol_log == small[f"{k}/vol_log"].tolist()
    assert rep.notes["stage_count"] == small[f"{k}/stage_count"]
    np.testing.assert_allclose(rep.residual_l1_trace, small[f"{k}/l1_log"], rtol=1e-12)
    # the reference test's oracle bound (tests/test_local_solvers.py:213-233)
    sys_ = S.make_hk_system(g, tau, 0, 1e-4)
    assert np.abs(f - small[f"{k}/series60"]).sum() <= 1e-4 + S.hk_paper_bound(sys_.op.stage_count)


@pytest.mark.parametrize("tau,eps", [(1.0, 1e-5), (5.0, 1e-6), (10.0, 1e-7)])
def test_heat_kernel_layered_matches_oracle(gpu, tau, eps):
    """The layered-sweep heat kernel reproduces the FIFO reference push bit
    for bit (f_hat, every stage's v and r, vol log) on an R-MAT graph."""
    from oracle import oracle as O
    from paper_2410_21634_b200.metrics import sample_sources
    from paper_2410_21634_b200.synth import rmat_graph
    g = rmat_graph(20000, 150000, seed=2)
    for s in sample_sources(g, 3, seed=1):
        f, rep = LS.local_hk(g, tau, int(s), eps)
        ref = O.local_hk(g, tau, int(s), eps)
        assert np.array_equal(f, ref["f_hat"])
        assert rep.sweeps == ref["sweeps"] and rep.total_ops == ref["total_ops"]
        assert rep.vol_log == ref["vol_log"].tolist()
        assert rep.notes["residual_mass"] == ref["residual_mass"]
        np.testing.assert_allclose(rep.residual_l1_trace, ref["l1_log"], rtol=1e-12)
        np.testing.assert_allclose(rep.gamma_log, ref["gamma_log"], rtol=1e-12)


def test_heat_kernel_tiny_tau(gpu, small):
    f, rep = LS.local_hk(golden_graph(small, "p2"), 1e-9, 0, 1e-3)
    assert rep.converged and rep.sweeps == 1
    np.testing.assert_allclose(f, [1.0, 0.0], atol=1e-8)
    assert np.array_equal(f, small["p2/hk/tiny/f_hat"])


def test_global_gd_matches_reference(gpu, small):
    g = golden_graph(small, "er500")
    st, rep = gradient_descent(S.make_ppr_system(g, 0.15, 0, 1e-6, symmetrized=True))
    k = "er500/ppr/gd"
    assert np.array_equal(st.x, small[f"{k}/x"]) and np.array_equal(st.r, small[f"{k}/r"])
    assert rep.sweeps == small[f"{k}/sweeps"] and rep.total_ops == small[f"{k}/total_ops"]
    np.testing.assert_allclose(rep.residual_l1_trace, small[f"{k}/l1_log"], rtol=1e-12)


def test_dynamic_snapshots_match_reference(gpu, dyn):
    from paper_2410_21634_b200.dynamic import make_pair, run_snapshots
    from paper_2410_21634_b200.graph import EdgeEvent
    g0 = golden_graph(dyn, "er120")
    ev = dyn["events"]
    batches = [[EdgeEvent("insert" if k else "delete", int(u), int(v))
                for b, k, u, v in ev if b == bi] for bi in range(int(ev[:, 0].max()) + 1)]
    for mode in ("dynamic", "static"):
        reps, pair, gf = run_snapshots(g0, batches, make_pair(g0, 0.2, 0.2 * 1e-4, 0), mode=mode)
        assert np.array_equal(pair.p, dyn[f"{mode}/p"]) and np.array_equal(pair.r, dyn[f"{mode}/r"])
        assert [r.sweeps for r in reps] == dyn[f"{mode}/sweeps"].tolist()
        assert [r.total_ops for r in reps] == dyn[f"{mode}/total_ops"].tolist()
        assert np.array_equal(np.concatenate([np.asarray(r.vol_log, np.int64) for r in reps]),
                              dyn[f"{mode}/vol_flat"])
        assert np.array_equal(np.concatenate([np.asarray(r.notes["sweep_signs"], np.int8) for r in reps]),
                              dyn[f"{mode}/signs_flat"])
    assert np.array_equal(gf.targets, golden_graph(dyn, "final").targets)


# ---- reference test bodies with the GPU solvers swapped in ----------------

def test_single_sweep_closure(gpu):
    from paper_2410_21634_b200.synth import path_graph
    sys_ = S.make_ppr_system(path_graph(2), 0.9, 0, 0.9)
    st, rep = LS.local_gd(sys_)
    assert rep.converged and rep.sweeps == 1
    assert np.array_equal(st.x, sys_.b)


def test_error_contract_p2(gpu):
    from paper_2410_21634_b200.metrics import error_norms
    from paper_2410_21634_b200.synth import path_graph
    g = path_graph(2)
    sys_ = S.make_ppr_system(g, 0.5, 0, 0.01, symmetrized=True)
    st, _ = LS.local_gd(sys_)
    assert error_norms(st.x, S.dense_solve(sys_), g)["linf_dscaled"] <= 0.01
    st, rep = LS.local_ch(S.make_ppr_system(g, 0.5, 0, 1e-4, symmetrized=True))
    assert rep.converged
    assert error_norms(st.x, S.dense_solve(sys_), g)["linf_dscaled"] <= 1e-4


@pytest.mark.parametrize("seed", range(6))
def test_ppr_ops_bound(gpu, seed):
    from paper_2410_21634_b200.synth import erdos_renyi
    g = erdos_renyi(80, 0.08, seed=seed)
    _, rep = LS.local_gs(S.make_ppr_system(g, 0.15, 0, 1e-4))
    assert rep.converged and rep.total_ops <= int(np.ceil(1.0 / (1e-4 * 0.15)))


def test_validation_errors(gpu, small):
    g = golden_graph(small, "k3")
    sys_ = S.make_ppr_system(g, 0.5, 0, 0.1)
    bad = S.DiffusionSystem(op=sys_.op, b=-sys_.b, theta_coeff=sys_.theta_coeff, problem="ppr",
                            alpha=0.5, eps=0.1, source=0)
    with pytest.raises(ValueError):
        LS.local_gd(bad)
    with pytest.raises(ValueError):
        LS.local_sor(sys_, omega=2.5)
    with pytest.raises(ValueError):
        LS.local_ch(sys_, mu=1.0, L=1.0)


def test_zero_source_and_nonconvergence(gpu, small):
    g = golden_graph(small, "er60")
    sys_ = S.make_ppr_system(g, 0.5, 0, 0.1)
    z = S.DiffusionSystem(op=sys_.op, b=np.zeros(g.n), theta_coeff=sys_.theta_coeff,
                          problem="ppr", alpha=0.5, eps=0.1, source=0)
    for fn in (LS.local_gd, LS.local_gs, LS.local_ch):
        st, rep = fn(z)
        assert rep.converged and rep.sweeps == 0 and rep.total_ops == 0
    _, rep = LS.local_gs(S.make_ppr_system(g, 0.1, 0, 1e-9), max_sweeps=2)
    assert not rep.converged and rep.sweeps == 2
    _, rep = LS.local_gd(S.make_ppr_system(g, 0.1, 0, 1e-9), max_sweeps=3)
    assert not rep.converged and rep.sweeps == 3


def test_reference_style_system_with_arc_array(gpu, small):
    """A system whose operator is given only as a per-arc array (the
    reference's OperatorQ layout) goes through the GD_W_ARC / GD_T_ARRAY path
    with the same bits."""
    from types import SimpleNamespace
    from oracle import oracle as O
    g = golden_graph(small, "er500")
    sys_ = S.make_ppr_system(g, 0.15, 0, 1e-6)
    w = S.arc_weights_for(g, 0.85, "sym")  # a non-rule operator
    op = SimpleNamespace(pkind="sym", beta=0.85, arc_weights=w, graph=g)
    alt = SimpleNamespace(op=op, b=sys_.b, theta=sys_.theta, problem="gen", graph=g, dim=g.n,
                          eps=1e-6, alpha=0.15, beta_exp=0.5)
    st, rep = LS.local_gd(alt)
    ref_sys = SimpleNamespace(op=op, b=sys_.b, theta=sys_.theta, graph=g, dim=g.n)
    ref = O.local_gd(ref_sys)
    assert np.array_equal(st.x, ref["x"]) and np.array_equal(st.r, ref["r"])
    assert rep.sweeps == ref["sweeps"] and rep.total_ops == ref["total_ops"]



def test_warm_gd_repair_matches_oracle(gpu, dyn):
    """Config 5 form: warm-started signed LocalGD repair after edge events,
    bit-identical with the oracle restatement; consistency invariant holds."""
    from oracle import oracle as O
    from paper_2410_21634_b200.dynamic import event_adjust_many, make_pair, repair_gd
    from paper_2410_21634_b200.graph import EdgeEvent, apply_events
    g = golden_graph(dyn, "er120")
    pair, rep = repair_gd(g, make_pair(g, 0.2, 0.2 * 1e-4, 0))
    assert rep.converged
    ev = dyn["events"]
    for bi in range(int(ev[:, 0].max()) + 1):
        batch = [EdgeEvent("insert" if k else "delete", int(u), int(v)) for b, k, u, v in ev if b == bi]
        pair = event_adjust_many(g, pair, batch)
        g = apply_events(g, batch)
        p2, r2 = pair.p.copy(), pair.r.copy()
        w = S.arc_weights_for(g, 0.8, "gen", 0.0)
        th = S.theta_vector(g, 0.2 * 1e-4)
        ref = O.local_gd_warm(g.offsets, g.targets, w, th, p2, r2, signed=True)
        pair, rep = repair_gd(g, pair)
        assert np.array_equal(pair.p, p2) and np.array_equal(pair.r, r2)
        assert rep.sweeps == ref["sweeps"] and rep.total_ops == ref["total_ops"]
        assert np.abs(pair.consistency_residual(g)).max() <= 1e-9
        fin = np.isfinite(th)
        assert np.all(np.abs(pair.r[fin]) < th[fin])


@pytest.mark.parametrize("seed", [0, 3])
def test_spectral_norm_gpu(gpu, seed):
    from paper_2410_21634_b200.graph import spectral_norm_estimate
    from paper_2410_21634_b200.synth import rmat_graph
    g = rmat_graph(20000, 150000, seed=seed)
    host = spectral_norm_estimate(g, iters=200, seed=0, device=False)
    dev = spectral_norm_estimate(g, iters=200, seed=0, device=True)
    assert abs(dev - host) <= 1e-9 * abs(host)


# ---- global Chebyshev / heat-kernel Taylor -----------

@pytest.mark.parametrize("key", ["er500/ppr/ch", "er60/ppr/ch", "er60/katz/ch", "er60/ppr/ch_cap"])
def test_global_chebyshev_matches_reference(gpu, glob, key):
    from paper_2410_21634_b200.global_solvers import GlobalConfig, chebyshev
    gname, prob, which = key.split("/")
    g = golden_graph(glob, gname)
    if prob == "ppr":
        sys_ = S.make_ppr_system(g, 0.15, 0, 1e-6) if gname == "er500" else \
            S.make_ppr_system(g, 0.2, 3, 1e-8)
        cfg = GlobalConfig(max_sweeps=3) if which == "ch_cap" else None
    else:
        ka = float(glob["katz_alpha"])
        sys_ = S.make_katz_system(g, ka, 0, 1e-6, lam_hat=0.0)
        cfg = GlobalConfig(mu=1.0 - ka * g.d_max, L=1.0 + ka * g.d_max)
    st, rep = chebyshev(sys_, cfg)
    assert np.array_equal(st.x, glob[f"{key}/x"]) and np.array_equal(st.r, glob[f"{key}/r"])
    assert rep.sweeps == glob[f"{key}/sweeps"] and rep.total_ops == glob[f"{key}/total_ops"]
    assert rep.converged == bool(glob[f"{key}/converged"])
    np.testing.assert_allclose(rep.residual_l1_trace, glob[f"{key}/l1_log"], rtol=1e-12)
    np.testing.assert_allclose(rep.notes["l2_trace"], glob[f"{key}/l2_log"], rtol=1e-12)
    assert rep.notes["delta_trace"] == glob[f"{key}/delta_log"].tolist()


@pytest.mark.parametrize("tau", [1.0, 5.0])
def test_hk_taylor_matches_reference(gpu, glob, tau):
    from paper_2410_21634_b200.global_solvers import hk_taylor_global
    g = golden_graph(glob, "er500")
    st, rep = hk_taylor_global(S.make_hk_system(g, tau, 0, 1e-5))
    k = f"er500/hk/taylor{tau}"
    assert np.array_equal(st.x, glob[f"{k}/x"]) and np.array_equal(st.r, glob[f"{k}/r"])
    assert rep.sweeps == glob[f"{k}/sweeps"] and rep.total_ops == glob[f"{k}/total_ops"]


@pytest.mark.parametrize("beta", [0.0, 0.5, 1.0])
def test_beta_push_matches_reference(gpu, glob, beta):
    """Degree-generalized signed feature push."""
    from paper_2410_21634_b200.dynamic import beta_push
    g = golden_graph(glob, "er500")
    pair, rep = beta_push(g, glob["betapush/source"], 0.15, beta, 1e-4)
    k = f"er500/betapush{beta}"
    assert np.array_equal(pair.p, glob[f"{k}/p"]) and np.array_equal(pair.r, glob[f"{k}/r"])
    assert rep.sweeps == glob[f"{k}/sweeps"] and rep.total_ops == glob[f"{k}/total_ops"]
    assert rep.notes["parked_mass"] == glob[f"{k}/parked"]


@pytest.mark.parametrize("beta", [0.0, 0.5, 1.0])
def test_beta_push_batch_columns_bitwise(gpu, glob, beta):
    """Multi-column feature push: every column equals beta_push on it."""
    from paper_2410_21634_b200.dynamic import beta_push, beta_push_batch
    from paper_2410_21634_b200.synth import rmat_graph
    for g in (golden_graph(glob, "er500"), rmat_graph(5000, 30000, seed=3)):
        rng = np.random.default_rng(int(beta * 10) + g.n)
        src = rng.standard_normal((g.n, 7)) * (rng.random((g.n, 7)) < 0.03)
        out = beta_push_batch(g, src, 0.15, beta, 1e-4, omega=1.2)
        for c in range(src.shape[1]):
            pair, rep = beta_push(g, src[:, c], 0.15, beta, 1e-4, omega=1.2)
            assert np.array_equal(out["p"][:, c], pair.p) and np.array_equal(out["r"][:, c], pair.r)
            assert out["sweeps"][c] == rep.sweeps and out["total_ops"][c] == rep.total_ops
            assert out["parked_mass"][c] == rep.notes["parked_mass"]
    # the reference's golden column
    g = golden_graph(glob, "er500")
    out = beta_push_batch(g, glob["betapush/source"], 0.15, beta, 1e-4)
    k = f"er500/betapush{beta}"
    assert np.array_equal(out["p"][:, 0], glob[f"{k}/p"]) and np.array_equal(out["r"][:, 0], glob[f"{k}/r"])
