"""Global gradient descent on the device -- the north star's "global
power-iteration GD on GPU" reference point (src/global_solvers.py:124-152).

Bit-exact with the reference: the pull form over sorted symmetric rows adds
each node's incoming contributions in ascending source order, which is the
order of the reference's scatter loop (_scatter_full :63-71).
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np

from . import _lib as gdl
from .device import device_graph, operator_for, report_arrays
from .reports import SolveReport, SolverState

__all__ = ["GlobalConfig", "gradient_descent", "DEFAULT_GLOBAL_SWEEPS"]

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
