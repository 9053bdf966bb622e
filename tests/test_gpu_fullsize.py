"""Full-size checks of the headline path: batched LocalGD-PPR,
alpha = 0.1, eps = 1e-7, on the R-MAT products-shape graph (2,385,902 nodes,
61,859,140 edges) that bench.py measures, generated and CSR-built on the GPU.

At this size the oracle is too slow for every seed, so the batch is checked
through properties that hold for any size, plus the oracle on a sample:

* mass: a LocalGD push moves r_u into x_u and scatters (1 - alpha) r_u to the
  neighbours (src/local_solvers.py:267-292 with the "rw" weights of
  src/systems.py:85-108), so alpha * sum(x) + sum(r) = alpha for b = alpha e_s;
* termination: every final residual is below its threshold theta_v = eps alpha d_v
  (the empty-frontier exit, src/local_solvers.py:444-458);
* x > 0 on its support (unsigned diffusion);
* sweeps, operation counts and pushes identical to the reference algorithm
  (oracle/ C port) on every 12th seed, sum(x) within 1e-12 relative.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_products_shape_batch_properties(gpu):
    from bench import SHAPES, host_graph_full, make_graph
    from oracle import oracle as O
    from paper_2410_21634_b200.batch import BatchSolver
    from paper_2410_21634_b200.metrics import sample_sources

    alpha, eps = 0.1, 1e-7
    n, _ = SHAPES["products"]
    dg, row, col, row_h = make_graph("products", 0, 0)
    hg = host_graph_full(n, row_h, col, alpha, eps)
    del row, col
    seeds = sample_sources(hg, 96, seed=0)
    solver = BatchSolver(dg, alpha, eps, want_r=True)
    try:
        out = solver.solve(seeds)
    finally:
        solver.close()
    assert out.converged.all()
    for i in range(len(seeds)):
        xn, xv = out.x_sparse(i)
        rn, rv = out.r_sparse(i)
        assert xv.size and (xv > 0).all()
        assert len(np.unique(xn)) == xn.size
        assert (np.abs(rv) < hg.theta[rn]).all()
        mass = alpha * xv.sum() + rv.sum()
        assert abs(mass - alpha) <= 1e-11, (i, mass)
    idx = np.arange(0, len(seeds), 12)
    ref = O.batch_local_gd(hg, alpha, eps, seeds[idx], threads=8, arc_w=hg.arc_w, theta=hg.theta)
    assert np.array_equal(out.sweeps[idx], ref["sweeps"])
    assert np.array_equal(out.total_ops[idx], ref["total_ops"])
    assert np.array_equal(out.pushes[idx], ref["pushes"])
    xs = np.array([out.x_sparse(i)[1].sum() for i in idx])
    np.testing.assert_allclose(xs, ref["xsum"], rtol=1e-12)


def test_papers100m_shape_batch_properties(gpu):
    """Config 4's graph (111,059,433 nodes, 1.6 B edges, built on the GPU): the
    size-independent properties only (the reference layout would need ~50 GB
    of host memory per solve)."""
    from bench import SHAPES, _HostGraph, make_graph
    from paper_2410_21634_b200.batch import BatchSolver
    from paper_2410_21634_b200.metrics import sample_sources
    from paper_2410_21634_b200.systems import theta_vector

    alpha, eps = 0.1, 1e-6
    n, _ = SHAPES["papers100M"]
    dg, row, col, row_h = make_graph("papers100M", 0, 0)
    del row, col
    hg = _HostGraph(n, row_h)
    theta = theta_vector(hg, eps * alpha)
    seeds = sample_sources(hg, 64, seed=0)
    solver = BatchSolver(dg, alpha, eps, want_r=True)
    try:
        out = solver.solve(seeds)
    finally:
        solver.close()
    assert out.converged.all()
    assert (out.total_ops > 0).all()
    for i in range(len(seeds)):
        xn, xv = out.x_sparse(i)
        rn, rv = out.r_sparse(i)
        assert xv.size and (xv > 0).all()
        assert (np.abs(rv) < theta[rn]).all()
        assert abs(alpha * xv.sum() + rv.sum() - alpha) <= 1e-11
    # every pushed node was pushed at least once: support of x <= pushes
    assert (out.x_count <= out.pushes).all()


def test_products_shape_local_ch_batch(gpu):
    """Config 3's LocalCH-PPR (mu = alpha, L = 2 - alpha, src/local_solvers.py:541-558)
    at the products shape: termination and sweeps / ops / convergence identical to
    the reference algorithm on a seed sample."""
    import math

    from bench import SHAPES, host_graph_full, make_graph
    from oracle import oracle as O
    from paper_2410_21634_b200.batch import BatchSolver
    from paper_2410_21634_b200.metrics import sample_sources

    alpha, eps = 0.1, 1e-7
    mu, L = alpha, 2.0 - alpha
    cap = max(1000, int(10 * math.log(1.0 / eps) / mu))
    n, _ = SHAPES["products"]
    dg, row, col, row_h = make_graph("products", 0, 0)
    hg = host_graph_full(n, row_h, col, alpha, eps)
    del row, col
    seeds = sample_sources(hg, 32, seed=1)
    solver = BatchSolver(dg, alpha, eps, method="local-ch", mu=mu, L=L, max_sweeps=cap,
                         want_r=True)
    try:
        out = solver.solve(seeds)
    finally:
        solver.close()
    assert out.converged.all()
    for i in range(len(seeds)):
        rn, rv = out.r_sparse(i)
        assert (np.abs(rv) < hg.theta[rn]).all()
    idx = np.arange(0, len(seeds), 8)
    ref = O.batch_local_ch(hg, alpha, eps, seeds[idx], threads=8, mu=mu, L=L, max_sweeps=cap)
    assert np.array_equal(out.sweeps[idx], ref["sweeps"])
    assert np.array_equal(out.total_ops[idx], ref["total_ops"])
    assert np.array_equal(out.converged[idx], ref["converged"])
    xs = np.array([out.x_sparse(i)[1].sum() for i in idx])
    np.testing.assert_allclose(xs, ref["xsum"], rtol=1e-9)
