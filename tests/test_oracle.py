"""The CPU oracle is pinned bit-for-bit against vectors produced by running the
reference implementation (tests/golden/make_golden.py)."""

import numpy as np
import pytest

from conftest import golden_graph, load_golden
from helpers import assert_matches, build_system, local_cases, method_of, solver_kwargs
from oracle import oracle as O
from paper_2410_21634_b200 import systems as S
from paper_2410_21634_b200.metrics import sample_sources

FIXTURES = ["small.npz", "pa2000.npz", "cora.npz"]


def _oracle_run(d, key):
    sys_ = build_system(d, key)
    m, kw = method_of(key), solver_kwargs(d, key)
    if m == "local_gd":
        return O.local_gd(sys_, **kw)
    if m == "local_ch":
        return O.local_ch(sys_, **kw)
    if m == "local_gs" or m.startswith("local_gs_"):
        return O.local_sor(sys_, 1.0, **kw)
    if m.startswith("local_sor"):
        return O.local_sor(sys_, **kw)
    raise ValueError(m)


@pytest.mark.parametrize("fixture", FIXTURES)
def test_oracle_local_solvers_bitwise(fixture):
    d = load_golden(fixture)
    keys = local_cases(d)
    assert keys
    for key in keys:
        assert_matches(d, key, _oracle_run(d, key), logs_exact=True)


@pytest.mark.parametrize("tau", [0.5, 1.0, 5.0])
def test_oracle_heat_kernel_bitwise(small, tau):
    g = golden_graph(small, "er60")
    out = O.local_hk(g, tau, 0, 1e-4)
    k = f"er60/hk/tau{tau}"
    assert np.array_equal(out["f_hat"], small[f"{k}/f_hat"])
    assert out["sweeps"] == small[f"{k}/sweeps"]
    assert out["total_ops"] == small[f"{k}/total_ops"]
    assert np.array_equal(out["vol_log"], small[f"{k}/vol_log"])
    assert np.array_equal(out["gamma_log"], small[f"{k}/gamma_log"])
    assert np.array_equal(out["l1_log"], small[f"{k}/l1_log"])
    assert out["stage_count"] == small[f"{k}/stage_count"]
    assert out["residual_mass"] == small[f"{k}/residual_mass"]


def test_oracle_global_gd_bitwise(small):
    g = golden_graph(small, "er500")
    sys_ = S.make_ppr_system(g, 0.15, 0, 1e-6, symmetrized=True)
    out = O.gradient_descent(sys_)
    k = "er500/ppr/gd"
    assert np.array_equal(out["x"], small[f"{k}/x"]) and np.array_equal(out["r"], small[f"{k}/r"])
    assert out["sweeps"] == small[f"{k}/sweeps"] and out["total_ops"] == small[f"{k}/total_ops"]
    assert np.array_equal(out["l1_log"], small[f"{k}/l1_log"])
    np.testing.assert_allclose(out["l2_log"], small[f"{k}/l2_log"], rtol=1e-12)


def test_oracle_batch_matches_reference_per_seed(cora):
    """Config 1 (cora-shape, 50 seeds): the threaded CPU baseline reproduces
    the reference's per-seed sweeps / ops / pushes and sum(x)."""
    g = golden_graph(cora, "cora")
    seeds = cora["seeds"]
    assert np.array_equal(sample_sources(g, 50, seed=0), seeds)
    out = O.batch_local_gd(g, 0.1, 1e-6, seeds, threads=4)
    assert np.array_equal(out["sweeps"], cora["batch/sweeps"])
    assert np.array_equal(out["total_ops"], cora["batch/total_ops"])
    assert np.array_equal(out["pushes"], cora["batch/pushes"])
    assert out["converged"].all()
    ref_sums = np.array([O.pairwise_sum(x) for x in cora["batch/x"]])
    assert np.array_equal(out["xsum"], ref_sums)


@pytest.mark.parametrize("n", [1, 2, 7, 8, 9, 15, 16, 17, 127, 128, 129, 255, 256, 1000, 4099])
def test_pairwise_sum_is_numpys(n):
    rng = np.random.default_rng(n)
    a = rng.standard_normal(n) * 10.0 ** rng.uniform(-6, 3, n)
    assert O.pairwise_sum(a) == float(a.sum())
    assert O.pairwise_sum(a, take_abs=True) == float(np.abs(a).sum())


def test_oracle_zero_source_and_max_sweeps(small):
    g = golden_graph(small, "er60")
    sys_ = S.make_ppr_system(g, 0.5, 0, 0.1)
    z = S.DiffusionSystem(op=sys_.op, b=np.zeros(g.n), theta_coeff=sys_.theta_coeff,
                          problem="ppr", alpha=0.5, eps=0.1, source=0)
    out = O.local_gd(z)
    assert out["sweeps"] == 0 and out["total_ops"] == 0 and out["converged"]
    out = O.local_sor(S.make_ppr_system(g, 0.1, 0, 1e-9), 1.0, max_sweeps=2)
    assert not out["converged"] and out["sweeps"] == 2


def test_warm_gd_restatement_is_the_reference_sweep_loop(small):
    """Cold start (x=0, r=b, unsigned) of the warm LocalGD restatement is the
    reference local_gd bit for bit, so the warm form composes only reference
    kernels."""
    g = golden_graph(small, "er500")
    sys_ = S.make_ppr_system(g, 0.15, 0, 1e-6)
    k = "er500/ppr/local_gd"
    x, r = np.zeros(g.n), sys_.b.copy()
    out = O.local_gd_warm(g.offsets, g.targets, sys_.op.arc_weights, sys_.theta, x, r, signed=False)
    assert np.array_equal(x, small[f"{k}/x"]) and np.array_equal(r, small[f"{k}/r"])
    assert out["sweeps"] == small[f"{k}/sweeps"]
    assert np.array_equal(np.concatenate(out["frontier_trace"]), small[f"{k}/trace_flat"])


def test_oracle_batch_local_ch_matches_reference(pa):
    """Threaded LocalCH CPU baseline == the reference's per-seed local_ch."""
    from helpers import local_cases, param
    g = golden_graph(pa, "pa2000")
    keys = [k for k in local_cases(pa) if k.endswith("/local_ch")]
    seeds = [int(param(pa, k, "source")) for k in keys]
    out = O.batch_local_ch(g, 0.1, 1e-6, seeds, threads=3, mu=0.1, L=1.9)
    for i, k in enumerate(keys):
        assert out["sweeps"][i] == pa[f"{k}/sweeps"] and out["total_ops"][i] == pa[f"{k}/total_ops"]
        assert out["xsum"][i] == O.pairwise_sum(pa[f"{k}/x"])


def test_oracle_batch_local_hk_matches_single(small):
    """Threaded heat-kernel CPU baseline == per-seed local_hk (golden er60)."""
    g = golden_graph(small, "er60")
    out = O.batch_local_hk(g, 1.0, 1e-4, [0, 0], threads=2)
    k = "er60/hk/tau1.0"
    assert (out["sweeps"] == small[f"{k}/sweeps"]).all()
    assert (out["total_ops"] == small[f"{k}/total_ops"]).all()
    np.testing.assert_allclose(out["fsum"], small[f"{k}/f_hat"].sum(), rtol=1e-12)


class _Sparse:
    """A BatchOutput-shaped container of per-seed sparse x (test helper)."""

    def __init__(self, xs):
        nodes, vals, off, cnt = [], [], [], []
        pos = 0
        for x in xs:
            nz = np.flatnonzero(x)
            nodes.append(nz.astype(np.int32))
            vals.append(x[nz])
            off.append(pos)
            cnt.append(nz.size)
            pos += nz.size
        self.x_offset, self.x_count = np.array(off, np.int64), np.array(cnt, np.int64)
        self.x_nodes = np.concatenate(nodes) if nodes else np.empty(0, np.int32)
        self.x_vals = np.concatenate(vals) if vals else np.empty(0)


def test_oracle_x_parity_against_reference_vectors(cora):
    """The per-seed comparison (l1 of x_gpu - x_ref, top-k ranking) measures 0
    and identical rankings on the reference's own x (golden cora batch), and
    sees a perturbation / a swapped top-2."""
    g = golden_graph(cora, "cora")
    seeds, xs = cora["seeds"], cora["batch/x"]
    out = O.batch_local_gd(g, 0.1, 1e-6, seeds, threads=4, gpu=_Sparse(xs))
    assert (out["x_l1_diff"] == 0).all() and out["topk_identical"].all()
    np.testing.assert_allclose(out["x_l1_ref"], [np.abs(x).sum() for x in xs], rtol=1e-12)
    bad = [x.copy() for x in xs]
    bad[3][np.argmax(bad[3])] *= 1 + 1e-6
    top2 = np.argsort(-bad[5])[:2]
    bad[5][top2] = bad[5][top2[::-1]]
    out = O.batch_local_gd(g, 0.1, 1e-6, seeds, threads=4, gpu=_Sparse(bad))
    assert out["x_l1_rel"][3] > 1e-8 and out["topk_identical"][3]
    assert not out["topk_identical"][5] and not out["topk_identical_up_to_ties"][5]
    assert out["x_l1_diff"][0] == 0


def test_oracle_rule_mode_is_the_reference_local_gd(cora, pa):
    """orc_batch_gd_rule (int32 targets, rule weights / thresholds, dirty-list
    reset: the papers100M checker) == the reference per seed: x bitwise,
    sweeps, ops, pushes (golden cora batch), and == the array form on pa2000."""
    g = golden_graph(cora, "cora")
    seeds = cora["seeds"]
    out = O.batch_gd_rule(g.n, g.offsets, g.targets.astype(np.int32), 0.1, 1e-6, seeds, 3,
                          gpu=_Sparse(cora["batch/x"]))
    assert np.array_equal(out["sweeps"], cora["batch/sweeps"])
    assert np.array_equal(out["total_ops"], cora["batch/total_ops"])
    assert np.array_equal(out["pushes"], cora["batch/pushes"])
    assert (out["x_l1_diff"] == 0).all() and out["topk_identical"].all()
    gp = golden_graph(pa, "pa2000")
    sd = sample_sources(gp, 40, seed=3)
    a = O.batch_local_gd(gp, 0.15, 1e-7, sd, threads=2)
    b = O.batch_gd_rule(gp.n, gp.offsets, gp.targets.astype(np.int32), 0.15, 1e-7, sd, 2)
    for f in ("sweeps", "total_ops", "pushes", "converged"):
        assert np.array_equal(a[f], b[f]), f


def test_oracle_heavy_ball_restatement_bitwise():
    """LocalHB (heavy-ball; not in the reference): the C restatement equals the
    reference's own _SweepDriver run with heavy-ball coefficients bit for bit
    (tests/golden/hb.npz from tests/golden/make_golden_hb.py): x, r, sweeps,
    ops, logs -- PPR and Katz cases."""
    from conftest import load_golden
    from paper_2410_21634_b200.graph import CsrGraph
    d = load_golden("hb.npz")
    g = CsrGraph(n=int(d["graph/n"]), offsets=d["graph/offsets"], targets=d["graph/targets"])
    for i in range(int(d["cases"])):
        k = f"c{i}"
        prob, alpha, eps, s = str(d[f"{k}/problem"]), float(d[f"{k}/alpha"]), float(d[f"{k}/eps"]), int(d[f"{k}/source"])
        sys_ = (S.make_ppr_system(g, alpha, s, eps) if prob == "ppr"
                else S.make_katz_system(g, alpha, s, eps, lam_hat=0.0))
        out = O.local_ch(sys_, mu=float(d[f"{k}/mu"]), L=float(d[f"{k}/L"]), hb=True)
        assert np.array_equal(out["x"], d[f"{k}/x"]) and np.array_equal(out["r"], d[f"{k}/r"]), k
        assert out["sweeps"] == d[f"{k}/sweeps"] and out["total_ops"] == d[f"{k}/total_ops"], k
        assert np.array_equal(out["vol_log"], d[f"{k}/vol_log"]), k
        assert np.array_equal(out["gamma_log"], d[f"{k}/gamma_log"]), k
        assert np.array_equal(out["l1_log"], d[f"{k}/l1_log"]), k
        assert bool(out["converged"]) == bool(d[f"{k}/converged"]), k
