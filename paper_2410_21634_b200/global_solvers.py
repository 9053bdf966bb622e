"""Global solvers on the device -- the north star's "global power-iteration
GD on GPU" reference point (src/global_solvers.py:124-152), global Chebyshev
(:155-204) and the heat-kernel Taylor stages (:207-235).

Bit-exact with the reference: the pull form over sorted symmetric rows adds
each node's incoming contributions in ascending source order, which is the
order of the reference's scatter loop (_scatter_full :63-71), and the
elementwise updates repeat the numpy expressions' roundings.  (Global GS/SOR,
:87-121, is a sequential node-order sweep and stays out of scope.)
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np

from . import _lib as gdl
from .device import device_graph, operator_for, report_arrays
from .reports import SolveReport, SolverState

__all__ = ["GlobalConfig", "gradient_descent", "chebyshev", "hk_taylor_global",
           "DEFAULT_GLOBAL_SWEEPS"]

DEFAULT_GLOBAL_SWEEPS = 10_000


@dataclass
class GlobalConfig:
    omega: float = 1.0
    mu: float | None = None
    L: float | None = None
    max_sweeps: int = DEFAULT_GLOBAL_SWEEPS

    def __post_init__(self):
        if not 0.0 < self.omega <= 2.0:
            raise ValueError("omega must be in (0, 2]")
        if self.mu is not None and self.L is not None and not 0.0 < self.mu <= self.L:
            raise ValueError("need 0 < mu <= L")


def gradient_descent(sys, cfg: GlobalConfig | None = None) -> tuple[SolverState, SolveReport]:
    """x += r, r <- beta P r over all nodes until no node is active."""
    cfg = cfg or GlobalConfig()
    if sys.problem == "hk":
        raise ValueError("use hk_taylor_global for heat-kernel systems")
    lib = gdl.load()
    dg = device_graph(sys.graph)
    o, keep = operator_for(sys)
    b = np.ascontiguousarray(sys.b, dtype=np.float64)
    x, r = np.empty(sys.dim), np.empty(sys.dim)
    rep = gdl.Report()
    t0 = time.perf_counter()
    gdl.check(lib.gd_gradient_descent(dg.handle, C.byref(o), gdl.ptr(b), gdl.ptr(x), gdl.ptr(r),
                                      int(cfg.max_sweeps), C.byref(rep)))
    wall = time.perf_counter() - t0
    out = report_arrays(rep)
    report = SolveReport(method="gd", problem=sys.problem, converged=out["converged"],
                         sweeps=out["sweeps"], total_ops=out["total_ops"], eps=float(sys.eps),
                         residual_l1_trace=[float(v) for v in out["l1_log"]], wall_seconds=wall)
    report.notes["l2_trace"] = [float(v) for v in out["l2_log"]]
    return SolverState(x=x, r=r, sweeps=out["sweeps"], ops=out["total_ops"]), report


def chebyshev(sys, cfg: GlobalConfig | None = None) -> tuple[SolverState, SolveReport]:
    """Two-term Chebyshev recurrence over all nodes; stop when no |r_u| >= theta_u."""
    from .local_solvers import cheby_bounds

    cfg = cfg or GlobalConfig()
    if sys.problem == "hk":
        raise ValueError("use hk_taylor_global for heat-kernel systems")
    mu, L = cheby_bounds(sys, cfg.mu, cfg.L)
    if mu >= L:
        raise ValueError(f"need mu < L, got mu={mu}, L={L}")
    lib = gdl.load()
    dg = device_graph(sys.graph)
    o, keep = operator_for(sys)
    b = np.ascontiguousarray(sys.b, dtype=np.float64)
    x, r = np.empty(sys.dim), np.empty(sys.dim)
    rep = gdl.Report()
    t0 = time.perf_counter()
    gdl.check(lib.gd_chebyshev(dg.handle, C.byref(o), gdl.ptr(b), gdl.ptr(x), gdl.ptr(r),
                               float(mu), float(L), int(cfg.max_sweeps), C.byref(rep)))
    wall = time.perf_counter() - t0
    out = report_arrays(rep)
    delta, deltas = (L - mu) / (L + mu), []
    for t in range(out["sweeps"]):  # the reference's delta_trace (:183-199)
        if t > 0:
            delta = 1.0 / (2.0 * (L + mu) / (L - mu) - delta)
        deltas.append(delta)
    report = SolveReport(method="ch", problem=sys.problem, converged=out["converged"],
                         sweeps=out["sweeps"], total_ops=out["total_ops"], eps=float(sys.eps),
                         residual_l1_trace=[float(v) for v in out["l1_log"]], wall_seconds=wall,
                         notes={"mu": mu, "L": L})
    report.notes["l2_trace"] = [float(v) for v in out["l2_log"]]
    report.notes["delta_trace"] = deltas
    return SolverState(x=x, r=r, sweeps=out["sweeps"], ops=out["total_ops"]), report


def hk_taylor_global(sys, cfg: GlobalConfig | None = None) -> tuple[SolverState, SolveReport]:
    """Dense stage propagation of the truncated heat-kernel Taylor sum."""
    cfg = cfg or GlobalConfig()
    if sys.problem != "hk":
        raise ValueError("hk_taylor_global requires a heat-kernel system")
    g = sys.graph
    N = int(sys.op.stage_count)
    lib = gdl.load()
    dg = device_graph(g)
    sw = np.ascontiguousarray(sys.op.stage_weights if N else np.zeros(1), dtype=np.float64)
    b0 = np.ascontiguousarray(sys.b[:g.n], dtype=np.float64)
    v = np.empty((N + 1) * g.n)
    t0 = time.perf_counter()
    gdl.check(lib.gd_hk_taylor(dg.handle, N, gdl.ptr(sw), gdl.ptr(b0), gdl.ptr(v)))
    wall = time.perf_counter() - t0
    ops = N * int(g.degrees.sum())
    report = SolveReport(method="hk-taylor", problem=sys.problem, converged=True, sweeps=N,
                         total_ops=ops, eps=float(sys.eps), residual_l1_trace=[],
                         wall_seconds=wall, notes={"stage_count": N, "tau": sys.tau})
    return SolverState(x=v, r=sys.residual(v), sweeps=N, ops=ops), report
