"""Seed sampling and error norms used by the solvers' callers.

``sample_sources`` defines the seed batch of every config (same draws as
src/metrics.py:174-192); ``error_norms`` is the parity metric of
src/metrics.py:157-171.
"""

from __future__ import annotations

import numpy as np

__all__ = ["sample_sources", "error_norms", "participation_ratio", "b_alg_bytes"]


def sample_sources(g, count: int, seed: int = 0) -> np.ndarray:
    """One node per degree-rank bucket, degree-0 nodes excluded."""
    rng = np.random.default_rng(seed)
    deg = np.asarray(g.degrees)
    elig = np.flatnonzero(deg > 0)
    if elig.size == 0:
        raise ValueError("no nodes with positive degree")
    count = min(count, elig.size)
    ranked = elig[np.argsort(deg[elig], kind="stable")]
    cuts = np.linspace(0, ranked.size, count + 1).astype(np.int64)
    out = np.empty(count, dtype=np.int64)
    for i in range(count):
        out[i] = ranked[rng.integers(cuts[i], max(cuts[i] + 1, cuts[i + 1]))]
    return out


def error_norms(f_hat, f_star, g) -> dict:
    f_hat = np.asarray(f_hat, dtype=np.float64)
    f_star = np.asarray(f_star, dtype=np.float64)
    if f_hat.shape != f_star.shape or f_hat.shape != (g.n,):
        raise ValueError("vector length mismatch")
    gap = f_hat - f_star
    pos = np.asarray(g.degrees) > 0
    scaled = np.abs(gap[pos]) / np.asarray(g.degrees)[pos]
    return {
        "linf_dscaled": float(scaled.max()) if scaled.size else 0.0,
        "linf_degree0": float(np.abs(gap[~pos]).max()) if (~pos).any() else 0.0,
        "l1": float(np.abs(gap).sum()),
        "l2": float(np.sqrt((gap * gap).sum())),
    }


def participation_ratio(f) -> float:
    f = np.asarray(f, dtype=np.float64)
    sq = f * f
    s2 = sq.sum()
    if s2 == 0.0:
        raise ValueError("participation ratio of the zero vector is undefined")
    return float(s2 * s2 / (f.shape[0] * (sq * sq).sum()))


def b_alg_bytes(total_ops: int, pushes: int, method: str = "local-gd") -> int:
    """Algorithmic HBM bytes of one local solve.

    20 B per arc touched (4 B col_idx + 8 B r[v] read + 8 B r[v] write) and
    52 B per pushed node (frontier id, row_ptr pair, r[u] rw, x[u] rw);
    LocalCH adds 24 B per push (momentum value + stamp), FIFO solvers 8 B.
    """
    if method == "local-hk":
        # heat kernel: its dense stages (>= 97 % of the operations at tau = 10,
        # eps = 1e-7 on the benchmark graphs) run as a pull -- per arc and slot an
        # 8 B gather of c[u][k] plus the 8 B (neighbour, degree) record once per
        # 14-slot chunk; per push r read + write, x read + write, c write (40 B)
        # and the pulled r_next write (8 B).  The few sparse stages are charged
        # the same (fewer bytes than their push would move: conservative).
        return int(8.6 * int(total_ops)) + 48 * int(pushes)
    per_push = 52 + (24 if method in ("local-ch", "local-hb") else 0) + (8 if method in ("local-sor", "local-gs") else 0)
    return 20 * int(total_ops) + per_push * int(pushes)
