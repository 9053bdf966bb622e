"""GDCSR v1 straight into device graphs, bench records with a backend column,
and the ``bench`` CLI.

CPU tests: header parsing and its errors, record writers in the reference's
formats (src/metrics.py:195-213).  GPU tests: a cache file loaded into HBM
equals the host-built graph, corrupted files raise the reference's
GraphStructureError, and ``cli bench`` on the cora-shape config reproduces
the reference's per-source operation counts (golden) for local-gd and the
oracle's for global gd."""

import json
import struct

import numpy as np
import pytest

from conftest import golden_graph
from paper_2410_21634_b200 import graph as G
from paper_2410_21634_b200.gdcsr import read_gdcsr_header
from paper_2410_21634_b200.records import (BENCH_CSV_COLUMNS, BenchRecord, speedup_ratio,
                                           write_records_csv, write_records_jsonl)


def _write_raw(path, n, offs, tg, magic=b"GDCSR", ver=1):
    with open(path, "wb") as fh:
        fh.write(magic + struct.pack("<B", ver) + struct.pack("<qq", n, len(tg)))
        fh.write(np.asarray(offs, "<i8").tobytes())
        fh.write(np.asarray(tg, "<i8").tobytes())


def test_header_and_format_errors(tmp_path, small):
    g = golden_graph(small, "k3")
    p = tmp_path / "g.csr"
    G.save_csr_cache(g, p)
    assert read_gdcsr_header(p) == (g.n, g.targets.shape[0])
    bad = tmp_path / "bad.csr"
    _write_raw(bad, g.n, g.offsets, g.targets, magic=b"XXCSR")
    with pytest.raises(G.GraphFormatError, match="not a CSR cache file"):
        read_gdcsr_header(bad)
    _write_raw(bad, g.n, g.offsets, g.targets, ver=2)
    with pytest.raises(G.GraphFormatError, match="unsupported cache version 2"):
        read_gdcsr_header(bad)
    raw = open(p, "rb").read()
    open(bad, "wb").write(raw[:-8])
    with pytest.raises(G.GraphFormatError, match="truncated"):
        read_gdcsr_header(bad)


def _recs():
    return [BenchRecord("g", "ppr", "gd", 1e-6, 3, 100, 5, True, 0.5, 0.1, 0.0),
            BenchRecord("g", "ppr", "local-gd", 1e-6, 3, 20, 4, True, 0.1, 0.1, 0.0)]


def test_record_writers_match_reference_format(tmp_path):
    recs = _recs()
    p = tmp_path / "r.jsonl"
    write_records_jsonl(recs, p)
    lines = open(p).read().splitlines()
    d = json.loads(lines[0])
    # the reference's keys (src/metrics.py:47-60) minus wall_seconds, plus backend
    assert list(d) == sorted(["alpha", "converged", "eps", "graph_id", "method", "omega",
                              "problem", "source", "sweeps", "total_ops", "backend"])
    assert d["backend"] == "cuda" and d["total_ops"] == 100
    write_records_jsonl(recs, p, timing=True)
    assert json.loads(open(p).readline())["wall_seconds"] == 0.5
    c = tmp_path / "r.csv"
    write_records_csv(recs, c)
    head = open(c).readline().strip().split(",")
    assert head == [k for k in BENCH_CSV_COLUMNS if k != "wall_seconds"]
    assert speedup_ratio(recs[:1], recs[1:]) == 5.0
    with pytest.raises(ValueError, match="differ in length"):
        speedup_ratio(recs, recs[:1])


def test_cli_usage_errors(tmp_path):
    from paper_2410_21634_b200.cli import main
    assert main(["bench"]) == 1
    assert main(["bench", "--graph", str(tmp_path / "missing.csr"), "--problem", "ppr"]) == 1


# ---------------------------------------------------------------- GPU


@pytest.mark.gpu
def test_load_device_graph_equals_host(gpu, tmp_path, cora, small):
    from paper_2410_21634_b200.device import DeviceGraph
    from paper_2410_21634_b200.gdcsr import load_device_graph, save_device_graph

    for g in (golden_graph(cora, "cora"), golden_graph(small, "k3")):
        p = tmp_path / "g.csr"
        G.save_csr_cache(g, p)
        dg = load_device_graph(p)
        h = dg.to_host()
        assert h.n == g.n and np.array_equal(h.offsets, g.offsets)
        assert np.array_equal(h.targets, g.targets)
        assert dg.d_max == int(np.diff(g.offsets).max())
        q = tmp_path / "g2.csr"
        save_device_graph(DeviceGraph.from_host(g), q)
        assert open(p, "rb").read() == open(q, "rb").read()


@pytest.mark.gpu
def test_load_device_graph_structure_errors(gpu, tmp_path, small):
    from paper_2410_21634_b200.gdcsr import load_device_graph

    g = golden_graph(small, "k3")
    o, t = g.offsets.copy(), g.targets.copy()
    p = tmp_path / "bad.csr"
    cases = []
    t1 = t.copy(); t1[0] = g.n                       # out of range
    cases.append((o, t1, "out of range"))
    t2 = t.copy(); t2[0] = 0                         # node 0's row holds 0: self loop
    cases.append((o, t2, "self-loop"))
    t3 = t.copy(); t3[0], t3[1] = t3[1], t3[0]       # row not ascending
    cases.append((o, t3, "strictly sorted"))
    o4 = o.copy(); o4[0] = 1
    cases.append((o4, t, "bad offsets"))
    for offs, tg, msg in cases:
        _write_raw(p, g.n, offs, tg)
        with pytest.raises(G.GraphStructureError, match=msg):
            load_device_graph(p)
    # drop one direction of an edge: missing reverse arc
    pa = G.from_edges(4, [(0, 1), (1, 2), (2, 3)])
    keep = np.ones(pa.targets.shape[0], bool)
    keep[0] = False                                  # remove 0 -> 1
    offs = pa.offsets.copy()
    offs[1:] -= 1
    _write_raw(p, 4, offs, pa.targets[keep])
    with pytest.raises(G.GraphStructureError, match="reverse arc"):
        load_device_graph(p)


@pytest.mark.gpu
def test_cli_bench_matches_reference_ops(gpu, tmp_path, cora):
    from oracle import oracle as O
    from paper_2410_21634_b200 import systems as S
    from paper_2410_21634_b200.cli import main

    g = golden_graph(cora, "cora")
    p = tmp_path / "cora.csr"
    G.save_csr_cache(g, p)
    out = tmp_path / "rec.jsonl"
    rc = main(["bench", "--graph", str(p), "--problem", "ppr", "--methods", "gd,sor",
               "--omega", "auto", "--eps", "1e-6", "--num-sources", "50", "--out", str(out)])
    assert rc == 0
    recs = [json.loads(s) for s in open(out)]
    seeds = cora["seeds"]
    loc = [r for r in recs if r["method"] == "local-gd"]
    glob = [r for r in recs if r["method"] == "gd"]
    sor = [r for r in recs if r["method"] == "local-sor"]
    assert [r["source"] for r in loc] == seeds.tolist()
    assert [r["total_ops"] for r in loc] == cora["batch/total_ops"].tolist()
    assert [r["sweeps"] for r in loc] == cora["batch/sweeps"].tolist()
    assert all(r["backend"] == "cuda" for r in recs)
    for r in glob[:5]:
        ref = O.gradient_descent(S.make_ppr_system(g, 0.1, r["source"], 1e-6))
        assert r["total_ops"] == ref["total_ops"] and r["sweeps"] == ref["sweeps"]
    for r in sor[:5]:
        ref = O.local_sor(S.make_ppr_system(g, 0.1, r["source"], 1e-6), r["omega"])
        assert r["total_ops"] == ref["total_ops"] and r["sweeps"] == ref["sweeps"]


def test_chunked_device_validation_on_cpu_tensors():
    """gdcsr._validate_device in small row ranges (the papers100M-scale form:
    O(chunk) temporaries) accepts a valid CSR and rejects each structural
    error of CsrGraph.validate (src/graph.py:105-123); run on CPU tensors."""
    import numpy as np
    import pytest
    import torch

    from paper_2410_21634_b200.gdcsr import GraphStructureError, _validate_device
    from paper_2410_21634_b200.synth import rmat_graph

    g = rmat_graph(3000, 12000, seed=2)
    row = torch.as_tensor(g.offsets)
    col = torch.as_tensor(g.targets.astype(np.int32))
    for chunk in (1, 97, 5000, 1 << 26):
        _validate_device(g.n, row, col, torch, chunk=chunk)
    # a missing reverse arc: drop one arc of a row (and shift offsets)
    u = int(np.argmax(g.degrees))
    a = int(g.offsets[u])
    col2 = torch.cat([col[:a], col[a + 1:]])
    row2 = row.clone()
    row2[u + 1:] -= 1
    with pytest.raises(GraphStructureError):
        _validate_device(g.n, row2, col2, torch, chunk=300)
    # unsorted row
    col3 = col.clone()
    col3[a], col3[a + 1] = col[a + 1], col[a]
    with pytest.raises(GraphStructureError):
        _validate_device(g.n, row, col3, torch, chunk=300)
    # self loop: replace the arc u->v by u->u (and keep rows sorted is not needed)
    col4 = col.clone()
    col4[a] = u
    with pytest.raises(GraphStructureError):
        _validate_device(g.n, row, col4, torch, chunk=300)
