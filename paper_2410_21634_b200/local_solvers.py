"""Frontier-restricted solvers on the B200: drop-in for the reference module.

Same names, arguments, validation errors and return types as
src/local_solvers.py (``local_gd`` :428, ``local_ch`` :473, ``local_sor``
:221, ``local_gs`` :256, ``push_sweeps`` :191, ``local_hk`` :664,
``optimal_omega`` :36).  Each call runs one system on the GPU through
libgdiff.so and is bit-identical with the reference: the same x and r, the
same frontier trace, sweep count and operation counts.  The residual-l1 /
gamma logs are float instrumentation reduced on the device and agree with
the reference to ~1e-15 relative.

There is no CPU fallback: without the CUDA library or a GPU these raise.
"""

from __future__ import annotations

import ctypes as C
import math
import time

import numpy as np

from . import _lib as gdl
from .device import device_graph, operator_for, report_arrays
from .reports import LocalReport, SolverState

__all__ = ["local_gs", "local_sor", "local_gd", "local_ch", "local_hb", "local_hk", "optimal_omega",
           "push_sweeps", "cheby_bounds", "DEFAULT_MAX_SWEEPS"]

DEFAULT_MAX_SWEEPS = 1_000_000


def optimal_omega(alpha: float) -> float:
    """omega* = 2 / (1 + sqrt(1 - (alpha - 1)^2)), in (1, 2)."""
    if not 0.0 < alpha < 1.0:
        raise ValueError("alpha must be in (0, 1)")
    return 2.0 / (1.0 + math.sqrt(1.0 - (alpha - 1.0) ** 2))


def _report(method, sys, out, eps, wall, guarantees_disabled=False, notes=None) -> LocalReport:
    return LocalReport(
        method=method, problem=sys.problem, converged=bool(out["converged"]),
        sweeps=int(out["sweeps"]), total_ops=int(out["total_ops"]), eps=float(eps),
        residual_l1_trace=[float(v) for v in out["l1_log"]], wall_seconds=wall,
        gamma_log=[float(v) for v in out["gamma_log"]],
        vol_log=[int(v) for v in out["vol_log"]],
        min_residual=float(out["min_residual"]), support_size=int(out["support_size"]),
        guarantees_disabled=guarantees_disabled, notes=notes or {},
    )


def _sys_graph(sys):
    return device_graph(sys.graph)


def push_sweeps(sys_or_arrays, x, r, seeds, omega=1.0, x_gain=1.0, signed=False,
                max_sweeps=DEFAULT_MAX_SWEEPS):
    """FIFO push in place; returns the reference kernel's tuple
    (converged, sweeps, total_ops, vol_log, gamma_log, l1_log, min_r, sign_log)."""
    lib = gdl.load()
    keep = []
    if hasattr(sys_or_arrays, "op"):
        sys = sys_or_arrays
        dg = _sys_graph(sys)
        o, keep = operator_for(sys)
    else:
        from .graph import CsrGraph

        offsets, targets, arc_w, theta = sys_or_arrays
        g = CsrGraph(n=int(np.asarray(offsets).shape[0] - 1), offsets=np.asarray(offsets),
                     targets=np.asarray(targets))
        dg = device_graph(g)
        keep.append(g)
        w = np.ascontiguousarray(arc_w, dtype=np.float64)
        th = np.ascontiguousarray(theta, dtype=np.float64)
        keep += [w, th]
        o = gdl.Operator(weight_rule=gdl.GD_W_ARC, theta_rule=gdl.GD_T_ARRAY, beta=0.0,
                       theta_coeff=0.0, arc_w=gdl.ptr(w), theta=gdl.ptr(th))
    if x.dtype != np.float64 or r.dtype != np.float64 or not (x.flags.c_contiguous and r.flags.c_contiguous):
        raise ValueError("x and r must be contiguous float64 arrays")
    sd = np.ascontiguousarray(seeds, dtype=np.int64)
    rep = gdl.Report()
    gdl.check(lib.gd_push_kernel(dg.handle, C.byref(o), gdl.ptr(x), gdl.ptr(r), gdl.ptr(sd, C.c_int64),
                               int(sd.shape[0]), float(omega), float(x_gain), int(bool(signed)),
                               int(max_sweeps), C.byref(rep)))
    out = report_arrays(rep)
    return (out["converged"], out["sweeps"], out["total_ops"], out["vol_log"], out["gamma_log"],
            out["l1_log"], out["min_residual"], out["sign_log"])


def local_sor(sys, omega: float, eps: float | None = None,
              max_sweeps: int = DEFAULT_MAX_SWEEPS) -> tuple[SolverState, LocalReport]:
    """Sequential relaxed push; signed frontier when omega > 1."""
    if not 0.0 < omega <= 2.0:
        raise ValueError("omega must be in (0, 2]")
    if sys.problem == "hk":
        raise ValueError("use local_hk for heat-kernel systems")
    if np.any(sys.b < 0):
        raise ValueError("local push requires a nonnegative source")
    eps = sys.eps if eps is None else eps
    signed = omega > 1.0
    x = np.zeros(sys.dim)
    r = np.array(sys.b, dtype=np.float64)
    seeds = np.flatnonzero(sys.b)
    t0 = time.perf_counter()
    conv, sweeps, ops, vol, gam, l1, mn, sgn = push_sweeps(sys, x, r, seeds, omega=omega,
                                                           signed=signed, max_sweeps=max_sweeps)
    wall = time.perf_counter() - t0
    out = {"converged": conv, "sweeps": sweeps, "total_ops": ops, "vol_log": vol,
           "gamma_log": gam, "l1_log": l1, "min_residual": mn,
           "support_size": int(np.count_nonzero(r))}
    rep = _report("local-sor" if omega != 1.0 else "local-gs", sys, out, eps, wall,
                  guarantees_disabled=signed,
                  notes={"omega": omega, "sweep_signs": [int(v) for v in sgn]})
    return SolverState(x=x, r=r, sweeps=rep.sweeps, ops=rep.total_ops), rep


def local_gs(sys, eps: float | None = None,
             max_sweeps: int = DEFAULT_MAX_SWEEPS) -> tuple[SolverState, LocalReport]:
    return local_sor(sys, omega=1.0, eps=eps, max_sweeps=max_sweeps)


def local_gd(sys, eps: float | None = None, max_sweeps: int = DEFAULT_MAX_SWEEPS,
             parallel: bool = False) -> tuple[SolverState, LocalReport]:
    """Restricted gradient step x += r_S, r -= Q r_S, all of S_t at once.

    ``parallel`` is accepted for signature compatibility; the device path is
    always parallel and always produces the sequential reference's bits.
    """
    if sys.problem == "hk":
        raise ValueError("use local_hk for heat-kernel systems")
    if np.any(sys.b < 0):
        raise ValueError("local_gd requires a nonnegative source")
    eps = sys.eps if eps is None else eps
    lib = gdl.load()
    dg = _sys_graph(sys)
    o, keep = operator_for(sys)
    b = np.ascontiguousarray(sys.b, dtype=np.float64)
    x, r = np.empty(sys.dim), np.empty(sys.dim)
    rep = gdl.Report()
    t0 = time.perf_counter()
    gdl.check(lib.gd_local_gd(dg.handle, C.byref(o), gdl.ptr(b), gdl.ptr(x), gdl.ptr(r), int(max_sweeps),
                            1, C.byref(rep)))
    wall = time.perf_counter() - t0
    out = report_arrays(rep, with_trace=True)
    report = _report("local-gd", sys, out, eps, wall, notes={"parallel": parallel})
    report.notes["frontier_sizes"] = [int(v) for v in out["frontier_sizes"]]
    state = SolverState(x=x, r=r, sweeps=out["sweeps"], ops=out["total_ops"],
                        frontier_trace=out["frontier_trace"])
    return state, report


def cheby_bounds(sys, mu=None, L_=None):
    """Default eigenvalue bounds (src/local_solvers.py:541-558)."""
    if mu is not None and L_ is not None:
        return float(mu), float(L_)
    if sys.problem in ("ppr", "gen"):
        return sys.alpha, 2.0 - sys.alpha
    if sys.problem == "katz":
        from .graph import spectral_norm_estimate

        g = sys.graph
        try:
            lam = spectral_norm_estimate(g, iters=200, seed=0)
        except Exception:
            lam = float(g.d_max)
        lam = min(max(lam, 1e-12), float(g.d_max))
        return 1.0 - sys.alpha * lam, 1.0 + sys.alpha * lam
    raise ValueError(f"no default Chebyshev bounds for {sys.problem}")


def local_ch(sys, mu: float | None = None, L: float | None = None, eps: float | None = None,
             max_sweeps: int | None = None) -> tuple[SolverState, LocalReport]:
    """Momentum-carrying restricted Chebyshev updates (signed frontier)."""
    if sys.problem == "hk":
        raise ValueError("use local_hk for heat-kernel systems")
    mu, Lb = cheby_bounds(sys, mu, L)
    if mu >= Lb:
        raise ValueError(f"need mu < L, got mu={mu}, L={Lb}")
    eps = sys.eps if eps is None else eps
    if max_sweeps is None:
        gap = max(mu, 1e-12)
        max_sweeps = max(1000, int(10 * math.log(max(1.0 / max(eps, 1e-300), 2.0)) / gap))
    lib = gdl.load()
    dg = _sys_graph(sys)
    o, keep = operator_for(sys)
    b = np.ascontiguousarray(sys.b, dtype=np.float64)
    x, r = np.empty(sys.dim), np.empty(sys.dim)
    rep = gdl.Report()
    t0 = time.perf_counter()
    gdl.check(lib.gd_local_ch(dg.handle, C.byref(o), gdl.ptr(b), gdl.ptr(x), gdl.ptr(r), float(mu),
                             float(Lb), int(max_sweeps), 0, C.byref(rep)))
    wall = time.perf_counter() - t0
    out = report_arrays(rep)
    report = _report("local-ch", sys, out, eps, wall, guarantees_disabled=True,
                     notes={"mu": mu, "L": Lb, "diverged": out["diverged"]})
    return SolverState(x=x, r=r, sweeps=out["sweeps"], ops=out["total_ops"]), report


def local_hb(sys, mu: float | None = None, L: float | None = None, eps: float | None = None,
             max_sweeps: int | None = None) -> tuple[SolverState, LocalReport]:
    """Heavy-ball momentum (LocalHB): local_ch's sweep loop, signed frontier,
    momentum stamps and divergence abort (src/local_solvers.py:473-538) with
    Polyak's stationary coefficients for eigenvalues in [mu, L]:
    eta = 4/(sqrt(L)+sqrt(mu))^2, beta = ((sqrt(L)-sqrt(mu))/(sqrt(L)+sqrt(mu)))^2.
    Not in the reference: bit-exact with the restatement in oracle/
    (orc_local_hb, pinned to the reference's own _SweepDriver by
    tests/golden/hb.npz)."""
    if sys.problem == "hk":
        raise ValueError("use local_hk for heat-kernel systems")
    mu, Lb = cheby_bounds(sys, mu, L)
    if mu >= Lb:
        raise ValueError(f"need mu < L, got mu={mu}, L={Lb}")
    eps = sys.eps if eps is None else eps
    if max_sweeps is None:
        gap = max(mu, 1e-12)
        max_sweeps = max(1000, int(10 * math.log(max(1.0 / max(eps, 1e-300), 2.0)) / gap))
    lib = gdl.load()
    dg = _sys_graph(sys)
    o, keep = operator_for(sys)
    b = np.ascontiguousarray(sys.b, dtype=np.float64)
    x, r = np.empty(sys.dim), np.empty(sys.dim)
    rep = gdl.Report()
    t0 = time.perf_counter()
    gdl.check(lib.gd_local_hb(dg.handle, C.byref(o), gdl.ptr(b), gdl.ptr(x), gdl.ptr(r), float(mu),
                             float(Lb), int(max_sweeps), 0, C.byref(rep)))
    wall = time.perf_counter() - t0
    out = report_arrays(rep)
    report = _report("local-hb", sys, out, eps, wall, guarantees_disabled=True,
                     notes={"mu": mu, "L": Lb, "diverged": out["diverged"]})
    return SolverState(x=x, r=r, sweeps=out["sweeps"], ops=out["total_ops"]), report


def local_hk(g, tau: float, s: int, eps: float,
             max_sweeps: int = DEFAULT_MAX_SWEEPS) -> tuple[np.ndarray, LocalReport]:
    """Push on the stage-expanded heat-kernel system; returns (f_hat, report)."""
    from .systems import make_hk_system

    sys = make_hk_system(g, tau, s, eps)
    N = sys.op.stage_count
    lib = gdl.load()
    dg = device_graph(g)
    sw = np.ascontiguousarray(sys.op.stage_weights if N else np.zeros(1), dtype=np.float64)
    v = np.zeros(sys.dim)
    r = np.array(sys.b, dtype=np.float64)
    rep = gdl.Report()
    t0 = time.perf_counter()
    gdl.check(lib.gd_hk_push(dg.handle, int(N), gdl.ptr(sw), float(sys.theta_coeff), gdl.ptr(v),
                            gdl.ptr(r), int(s), int(max_sweeps), C.byref(rep)))
    wall = time.perf_counter() - t0
    out = report_arrays(rep)
    report = _report("local-hk", sys, out, eps, wall, notes={"tau": tau, "stage_count": N})
    report.notes["residual_mass"] = float(np.abs(r).sum())
    return sys.back_transform(v), report
