"""Host-side mirror of the reference interface: graphs, generators, systems,
seed sampling, dynamic pair algebra (no GPU needed)."""

import io

import numpy as np
import pytest

from conftest import golden_graph
from paper_2410_21634_b200 import graph as G
from paper_2410_21634_b200 import synth, systems as S
from paper_2410_21634_b200.dynamic import PprPair, event_adjust, parse_events
from paper_2410_21634_b200.graph import EdgeEvent
from paper_2410_21634_b200.metrics import b_alg_bytes, error_norms, sample_sources


def _same(g1, g2):
    return g1.n == g2.n and np.array_equal(g1.offsets, g2.offsets) and np.array_equal(g1.targets, g2.targets)


def test_generators_reproduce_reference_graphs(small, pa, cora):
    assert _same(synth.erdos_renyi(500, 0.02, seed=21), golden_graph(small, "er500"))
    assert _same(synth.erdos_renyi(60, 0.1, seed=7), golden_graph(small, "er60"))
    assert _same(synth.complete_graph(3), golden_graph(small, "k3"))
    assert _same(synth.path_graph(2), golden_graph(small, "p2"))
    assert _same(synth.preferential_attachment(2000, 3, seed=1), golden_graph(pa, "pa2000"))
    assert _same(synth.rmat_graph(2708, 5278, seed=0), golden_graph(cora, "cora"))


def test_rmat_shape_and_canonical_csr():
    g = synth.rmat_graph(5000, 20000, seed=3)
    assert g.m == 20000 and g.n == 5000
    g.validate()
    # rebuilding from its own edge set is the identity (canonical form)
    src = np.repeat(np.arange(g.n), g.degrees)
    keep = src < g.targets
    assert _same(G.csr_from_pairs(g.n, np.stack([src[keep], g.targets[keep]], 1)), g)


def test_sample_sources_matches_reference(pa, cora):
    assert np.array_equal(sample_sources(golden_graph(pa, "pa2000"), 8, seed=0), pa["seeds"])
    assert np.array_equal(sample_sources(golden_graph(cora, "cora"), 50, seed=0), cora["seeds"])


def test_arc_weight_rule_is_bitwise(small):
    """The per-node rule fl(fl(1/d_u) beta) the device uses equals the
    reference's per-arc array (src/systems.py:85-108) bit for bit."""
    g = golden_graph(small, "er500")
    w = S.arc_weights_for(g, 0.85, "rw")
    d = np.repeat(g.degrees.astype(np.float64), g.degrees)
    assert np.array_equal(w, (1.0 / d) * 0.85)
    assert np.array_equal(S.arc_weights_for(g, 0.85, "gen", 0.0), w)
    th = S.theta_vector(g, 1e-6 * 0.15)
    assert np.array_equal(th[g.degrees > 0], (1e-6 * 0.15) * g.degrees[g.degrees > 0])


def test_apply_event_equals_rebuild(small):
    g = golden_graph(small, "er60")
    rng = np.random.default_rng(0)
    for _ in range(40):
        u, v = sorted(rng.choice(g.n, 2, replace=False).tolist())
        e = EdgeEvent("delete" if g.has_edge(u, v) else "insert", u, v)
        g2 = G.apply_event(g, e)
        src = np.repeat(np.arange(g.n), g.degrees)
        edges = {(a, b) for a, b in zip(src.tolist(), g.targets.tolist()) if a < b}
        edges = edges - {(u, v)} if e.kind == "delete" else edges | {(u, v)}
        assert _same(g2, G.from_edges(g.n, sorted(edges)))
        g2.validate()
        g = g2


def test_event_adjust_matches_reference(dyn):
    g = golden_graph(dyn, "er50")
    pair = PprPair(p=dyn["adj/p0"].copy(), r=dyn["adj/r0"].copy(), alpha=0.2, eps=1e-4, source=0)
    for ev, p_ref, r_ref in (("adj/ev1", "adj/p1", "adj/r1"), ("adj/ev2", "adj/p2", "adj/r2")):
        kind, u, v = dyn[ev].tolist()
        out = event_adjust(g, pair, EdgeEvent("insert" if kind else "delete", u, v))
        assert np.array_equal(out.p, dyn[p_ref]) and np.array_equal(out.r, dyn[r_ref])
        g2 = G.apply_event(g, EdgeEvent("insert" if kind else "delete", u, v))
        assert np.abs(out.consistency_residual(g2)).max() <= 1e-9


def test_parse_events_and_errors():
    batches = parse_events(io.StringIO("# c\nI 0 1\nD 2 3\n---\nI 4 5\n"))
    assert [[(e.kind, e.u, e.v) for e in b] for b in batches] == [
        [("insert", 0, 1), ("delete", 2, 3)], [("insert", 4, 5)]]
    with pytest.raises(G.GraphFormatError):
        parse_events(io.StringIO("X 1 2\n"))
    with pytest.raises(ValueError):
        EdgeEvent("insert", 3, 3)


def test_system_builders_validate(small):
    g = golden_graph(small, "er60")
    with pytest.raises(S.SystemError):
        S.make_ppr_system(g, 0.0, 0, 1e-4)
    with pytest.raises(S.SystemError):
        S.make_ppr_system(g, 0.2, g.n, 1e-4)
    with pytest.raises(S.SystemError):
        S.make_hk_system(g, -1.0, 0, 1e-4)
    sys_ = S.make_hk_system(g, 1.0, 0, 1e-4)
    assert sys_.dim == (sys_.op.stage_count + 1) * g.n
    assert S.hk_stage_count(10.0, 1e-7) == 31


def test_known_answers_dense():
    """Known-answer values of the reference tests (tests/test_systems.py:13-63)."""
    p2, k3 = synth.path_graph(2), synth.complete_graph(3)
    np.testing.assert_allclose(S.dense_solve(S.make_ppr_system(p2, 0.5, 0, 0.1)), [2 / 3, 1 / 3], atol=1e-12)
    np.testing.assert_allclose(S.dense_solve(S.make_ppr_system(k3, 0.5, 0, 0.1)), [0.6, 0.2, 0.2], atol=1e-12)
    np.testing.assert_allclose(S.dense_solve(S.make_katz_system(p2, 0.25, 0, 0.1)), [1 / 15, 4 / 15], atol=1e-12)
    np.testing.assert_allclose(S.dense_solve(S.make_katz_system(k3, 0.25, 0, 0.1)), [0.2, 0.4, 0.4], atol=1e-12)


def test_error_norms_and_b_alg():
    g = synth.path_graph(3)
    e = error_norms(np.array([1.0, 0.0, 0.0]), np.zeros(3), g)
    assert e["l1"] == 1.0 and e["linf_dscaled"] == 1.0
    assert b_alg_bytes(100, 10) == 20 * 100 + 52 * 10


def test_csr_cache_roundtrip(tmp_path, small):
    g = golden_graph(small, "er500")
    p = tmp_path / "g.csr"
    G.save_csr_cache(g, p)
    assert _same(G.load_csr_cache(p), g)


def test_bulk_events_equal_sequential(small):
    """event_adjust_many / vectorised apply_events == the per-event reference path."""
    from paper_2410_21634_b200.dynamic import event_adjust_many, make_pair
    g = golden_graph(small, "er500")
    rng = np.random.default_rng(4)
    pair = make_pair(g, 0.2, 1e-4, 0)
    pair.p[:] = rng.random(g.n)
    pair.r[:] = rng.random(g.n) - 0.5
    sim, evs = g, []
    for _ in range(400):  # includes repeated edits of the same edge
        u, v = sorted(rng.choice(60, 2, replace=False).tolist())
        e = EdgeEvent("delete" if sim.has_edge(u, v) else "insert", u, v)
        evs.append(e)
        sim = G.apply_event(sim, e)
    seq = pair
    gg = g
    for e in evs:
        seq = event_adjust(gg, seq, e)
        gg = G.apply_event(gg, e)
    bulk = event_adjust_many(g, pair, evs)
    assert np.array_equal(bulk.p, seq.p) and np.array_equal(bulk.r, seq.r)
    assert _same(G.apply_events(g, evs), gg)
    with pytest.raises(G.GraphStructureError):
        G.apply_events(g, evs + [EdgeEvent("insert", evs[-1].u, evs[-1].v)] * 70
                       if evs[-1].kind == "insert" else evs + [EdgeEvent("delete", evs[-1].u, evs[-1].v)] * 70)


def test_torch_rmat_stream_is_the_library_stream():
    """gen.rmat_keys_torch (the reference arm's generator: torch ops, no
    libgdiff) draws the same candidate keys as synth.rmat_edges + permute_ids
    (the host twin of csrc/generate.cu) and builds the same CSR."""
    import torch

    from paper_2410_21634_b200.gen import rmat_csr_device, rmat_keys_torch
    from paper_2410_21634_b200.synth import permute_ids, rmat_edges, rmat_graph

    for n, scale, seed in [(2708, 12, 0), (169_343, 18, 3), (111_059_433, 27, 1)]:
        cand = rmat_edges(scale, 12345, 4000, seed)
        a = permute_ids(cand[:, 0], scale, seed).astype(np.int64)
        b = permute_ids(cand[:, 1], scale, seed).astype(np.int64)
        ok = (a < n) & (b < n) & (a != b)
        want = np.where(ok, np.minimum(a, b) * n + np.maximum(a, b), -1)
        got = rmat_keys_torch(scale, n, 12345, 4000, seed, (0.57, 0.19, 0.19),
                              torch.device("cpu"), chunk=999).numpy()
        assert np.array_equal(want, got), n
    row, col = rmat_csr_device(2708, 5278, seed=0, native=False)
    g = rmat_graph(2708, 5278, seed=0)
    assert np.array_equal(row.numpy(), g.offsets)
    assert np.array_equal(col.numpy().astype(np.int64), g.targets)
