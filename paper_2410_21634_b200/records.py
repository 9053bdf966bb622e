"""Benchmark records with a ``backend`` column, and the batched bench driver.

Mirrors the reference's ``BenchRecord`` / ``write_records_jsonl`` /
``write_records_csv`` / ``speedup_ratio`` (src/metrics.py:47-69, :195-213,
:71-82) and its ``cmd_bench`` loop (src/cli.py:150-190: for every method
family F run F and local-F on every sampled source).  Records gain one
column, ``backend`` ("cuda" here, "cpu" for the reference), so GPU and CPU
runs can share one JSONL/CSV file; with ``backend`` dropped the records are
field-for-field the reference's.

On the device the local methods run as one batch over all sources
(``BatchSolver``), the global method per source (``gradient_descent``);
``wall_seconds`` of a batched record is the batch's wall time divided by the
number of sources.
"""

from __future__ import annotations

import csv
import json
import time
from dataclasses import asdict, dataclass

import numpy as np

__all__ = ["BenchRecord", "BENCH_CSV_COLUMNS", "write_records_jsonl", "write_records_csv",
           "speedup_ratio", "bench_family", "LOCAL_BATCH_METHODS"]


@dataclass
class BenchRecord:
    """One run of a method on a (graph, problem, source) triple
    (src/metrics.py:47-64) plus the backend that produced it."""

    graph_id: str
    problem: str
    method: str
    eps: float
    source: int
    total_ops: int
    sweeps: int
    converged: bool
    wall_seconds: float = 0.0
    alpha: float = 0.0
    omega: float = 0.0
    backend: str = "cuda"

    def key(self) -> tuple:
        return (self.graph_id, self.problem, self.eps, self.source)


BENCH_CSV_COLUMNS = ["graph_id", "problem", "method", "eps", "source", "total_ops", "sweeps",
                     "converged", "alpha", "omega", "wall_seconds", "backend"]


def write_records_jsonl(records, path, timing: bool = False) -> None:
    """One JSON object per line, keys sorted, wall time only with ``timing``
    (src/metrics.py:195-204)."""
    with open(path, "w") as fh:
        for rec in records:
            d = asdict(rec)
            if not timing:
                d.pop("wall_seconds")
            fh.write(json.dumps(d, sort_keys=True))
            fh.write("\n")


def write_records_csv(records, path, timing: bool = False) -> None:
    """src/metrics.py:207-213, with the backend column last."""
    cols = [c for c in BENCH_CSV_COLUMNS if timing or c != "wall_seconds"]
    with open(path, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=cols, extrasaction="ignore")
        w.writeheader()
        for rec in records:
            w.writerow(asdict(rec))


def speedup_ratio(global_records, local_records) -> float:
    """Summed operations, global over local, on matching configs
    (src/metrics.py:71-82; same ValueErrors)."""
    if len(global_records) != len(local_records):
        raise ValueError("record lists differ in length")
    for gr, lr in zip(global_records, local_records):
        if gr.key() != lr.key():
            raise ValueError(f"mismatched configs: {gr.key()} vs {lr.key()}")
    local_total = sum(r.total_ops for r in local_records)
    if local_total == 0:
        raise ValueError("local operation count is zero")
    return sum(r.total_ops for r in global_records) / local_total


LOCAL_BATCH_METHODS = ("local-gd", "local-gs", "local-sor", "local-ch")


def _local_batch(g, method, problem, alpha, eps, omega, sources, max_sweeps):
    from .batch import BatchSolver, local_ch_batch

    if method == "local-ch":
        return local_ch_batch(g, sources, alpha, eps, problem=problem, max_sweeps=max_sweeps)
    if problem != "ppr":
        raise ValueError(f"{method} batches support problem 'ppr' only")
    kw = {"method": "local-sor", "omega": 1.0 if method == "local-gs" else omega} \
        if method in ("local-gs", "local-sor") else {}
    solver = BatchSolver(g, alpha, eps, max_sweeps=max_sweeps or 1_000_000, **kw)
    try:
        return solver.solve(np.asarray(sources, np.int64))
    finally:
        solver.close()


def bench_family(g, graph_id: str, family: str, sources, alpha: float, eps: float,
                 problem: str = "ppr", omega: float = 1.0, max_sweeps: int | None = None):
    """Records for F and local-F on every source (src/cli.py:150-190), the
    local method as one device batch, the global one per source.  Families:
    "gd" (global GD / LocalGD), "gs" (local-gs), "sor" (local-sor), "ch"
    (local-ch).  Only families with a device global solver emit the global
    records; the others emit the local ones."""
    from .global_solvers import DEFAULT_GLOBAL_SWEEPS, GlobalConfig, gradient_descent
    from .systems import make_katz_system, make_ppr_system

    sources = np.asarray(sources, np.int64)
    method = f"local-{family}"
    if method not in LOCAL_BATCH_METHODS:
        raise ValueError(f"unknown method family {family}")
    records = []
    if family == "gd":
        for s in sources:
            sys_ = (make_ppr_system(g, alpha, int(s), eps, symmetrized=True) if problem == "ppr"
                    else make_katz_system(g, alpha, int(s), eps))
            t0 = time.perf_counter()
            _, rep = gradient_descent(sys_, GlobalConfig(max_sweeps=max_sweeps or DEFAULT_GLOBAL_SWEEPS))
            wall = time.perf_counter() - t0
            records.append(BenchRecord(graph_id, problem, "gd", float(eps), int(s),
                                       int(rep.total_ops), int(rep.sweeps), bool(rep.converged),
                                       wall, float(alpha), 0.0))
    t0 = time.perf_counter()
    out = _local_batch(g, method, problem, alpha, eps, omega, sources, max_sweeps)
    wall = (time.perf_counter() - t0) / max(1, sources.size)
    om = float(omega) if family == "sor" else 0.0
    for i, s in enumerate(sources):
        records.append(BenchRecord(graph_id, problem, method, float(eps), int(s),
                                   int(out.total_ops[i]), int(out.sweeps[i]),
                                   bool(out.converged[i]), wall, float(alpha), om))
    return records
