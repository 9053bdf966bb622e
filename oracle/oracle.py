"""ctypes front end of the CPU oracle (liboracle.so, built from gdiff_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py -- never by the product
package.  Each wrapper mirrors one reference solver entry point and returns a
plain dict of its outputs.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)


class _Report(C.Structure):
    _fields_ = [
        ("converged", C.c_int32), ("diverged", C.c_int32),
        ("sweeps", C.c_int64), ("total_ops", C.c_int64),
        ("min_residual", C.c_double), ("support_size", C.c_int64),
        ("n_logs", C.c_int64),
        ("vol_log", _i64p), ("gamma_log", _f64p), ("l1_log", _f64p),
        ("sign_log", C.POINTER(C.c_int8)), ("frontier_sizes", _i64p),
        ("trace", _i64p), ("trace_len", C.c_int64), ("l2_log", _f64p),
        ("cap", C.c_int64), ("trace_cap", C.c_int64),
    ]


def build() -> str:
    """Compile liboracle.so in place (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return os.path.join(_HERE, "liboracle.so")


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        src = os.path.join(_HERE, "gdiff_oracle.c")
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
            build()
        L = C.CDLL(path)
        assert L.orc_report_sizeof() == C.sizeof(_Report)
        L.orc_pairwise_sum.restype = C.c_double
        _LIB = L
    return _LIB


def _p(a, ct=C.c_double):
    return a.ctypes.data_as(C.POINTER(ct))


def _arr64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _arrf(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _unpack(rep: _Report, with_trace: bool = False) -> dict:
    k = rep.n_logs
    out = {
        "converged": bool(rep.converged), "diverged": bool(rep.diverged),
        "sweeps": int(rep.sweeps), "total_ops": int(rep.total_ops),
        "min_residual": float(rep.min_residual), "support_size": int(rep.support_size),
        "vol_log": np.ctypeslib.as_array(rep.vol_log, (k,)).copy() if k else np.empty(0, np.int64),
        "gamma_log": np.ctypeslib.as_array(rep.gamma_log, (k,)).copy() if k else np.empty(0),
        "l1_log": np.ctypeslib.as_array(rep.l1_log, (k + 1,)).copy(),
        "sign_log": np.ctypeslib.as_array(rep.sign_log, (k,)).copy() if k else np.empty(0, np.int8),
        "frontier_sizes": np.ctypeslib.as_array(rep.frontier_sizes, (k,)).copy() if k else np.empty(0, np.int64),
        "l2_log": np.ctypeslib.as_array(rep.l2_log, (k + 1,)).copy(),
    }
    if with_trace:
        flat = (np.ctypeslib.as_array(rep.trace, (rep.trace_len,)).copy()
                if rep.trace_len else np.empty(0, np.int64))
        cuts = np.cumsum(out["frontier_sizes"])[:-1]
        out["frontier_trace"] = np.split(flat, cuts) if k else []
    lib().orc_report_free(C.byref(rep))
    return out


def _sys_arrays(sys):
    g = sys.graph
    return (_arr64(g.offsets), _arr64(g.targets), _arrf(sys.op.arc_weights), _arrf(sys.theta))


def local_gd(sys, max_sweeps: int = 1_000_000, record_trace: bool = True) -> dict:
    """src/local_solvers.py:428-470 (parallel=False)."""
    off, tg, w, th = _sys_arrays(sys)
    n = sys.dim
    b = _arrf(sys.b)
    x, r = np.zeros(n), np.zeros(n)
    rep = _Report()
    lib().orc_local_gd(C.c_int64(n), _p(off, C.c_int64), _p(tg, C.c_int64), _p(w), _p(th), _p(b),
                       _p(x), _p(r), C.c_int64(max_sweeps), C.c_int32(int(record_trace)), C.byref(rep))
    out = _unpack(rep, with_trace=record_trace)
    out.update(x=x, r=r)
    return out


def local_gd_warm(offsets, targets, arc_w, theta, x, r, signed=True, max_sweeps=1_000_000,
                  record_trace=True) -> dict:
    """Warm-started signed LocalGD from (x, r), in place."""
    off, tg, w, th = _arr64(offsets), _arr64(targets), _arrf(arc_w), _arrf(theta)
    assert x.dtype == np.float64 and r.dtype == np.float64 and x.flags.c_contiguous
    rep = _Report()
    lib().orc_local_gd_warm(C.c_int64(th.shape[0]), _p(off, C.c_int64), _p(tg, C.c_int64), _p(w),
                            _p(th), _p(x), _p(r), C.c_int32(int(signed)), C.c_int64(max_sweeps),
                            C.c_int32(int(record_trace)), C.byref(rep))
    return _unpack(rep, with_trace=record_trace)


def cheby_bounds(sys, mu=None, L=None):
    """src/local_solvers.py:541-558."""
    if mu is not None and L is not None:
        return float(mu), float(L)
    if sys.problem in ("ppr", "gen"):
        return sys.alpha, 2.0 - sys.alpha
    if sys.problem == "katz":
        from paper_2410_21634_b200.graph import spectral_norm_estimate
        g = sys.graph
        lam = spectral_norm_estimate(g, iters=200, seed=0)
        lam = min(max(lam, 1e-12), float(g.d_max))
        return 1.0 - sys.alpha * lam, 1.0 + sys.alpha * lam
    raise ValueError(f"no default Chebyshev bounds for {sys.problem}")


def local_ch(sys, mu=None, L=None, eps=None, max_sweeps=None, record_trace=True,
             hb: bool = False) -> dict:
    """src/local_solvers.py:473-538; hb=True: its heavy-ball restatement
    (orc_local_hb, pinned by tests/golden/hb.npz)."""
    mu, L = cheby_bounds(sys, mu, L)
    eps = sys.eps if eps is None else eps
    if max_sweeps is None:
        gap = max(mu, 1e-12)
        max_sweeps = max(1000, int(10 * math.log(max(1.0 / max(eps, 1e-300), 2.0)) / gap))
    off, tg, w, th = _sys_arrays(sys)
    n = sys.dim
    b = _arrf(sys.b)
    x, r = np.zeros(n), np.zeros(n)
    rep = _Report()
    fn = lib().orc_local_hb if hb else lib().orc_local_ch
    fn(C.c_int64(n), _p(off, C.c_int64), _p(tg, C.c_int64), _p(w), _p(th), _p(b),
       _p(x), _p(r), C.c_double(mu), C.c_double(L), C.c_int64(max_sweeps),
       C.c_int32(int(record_trace)), C.byref(rep))
    out = _unpack(rep, with_trace=record_trace)
    out.update(x=x, r=r, mu=mu, L=L)
    return out


def push_kernel(offsets, targets, arc_w, theta, x, r, seeds, omega=1.0, x_gain=1.0,
                signed=False, max_sweeps=1_000_000) -> dict:
    """src/local_solvers.py:48-188; x and r are updated in place."""
    off, tg, w, th = _arr64(offsets), _arr64(targets), _arrf(arc_w), _arrf(theta)
    assert x.dtype == np.float64 and r.dtype == np.float64 and x.flags.c_contiguous
    sd = _arr64(seeds)
    rep = _Report()
    lib().orc_push_kernel(C.c_int64(th.shape[0]), _p(off, C.c_int64), _p(tg, C.c_int64), _p(w),
                          _p(th), _p(x), _p(r), _p(sd, C.c_int64), C.c_int64(sd.shape[0]),
                          C.c_double(omega), C.c_double(x_gain), C.c_int32(int(signed)),
                          C.c_int64(max_sweeps), C.byref(rep))
    return _unpack(rep)


def local_sor(sys, omega: float, max_sweeps: int = 1_000_000) -> dict:
    """src/local_solvers.py:221-253."""
    x = np.zeros(sys.dim)
    r = _arrf(sys.b).copy()
    seeds = np.flatnonzero(sys.b)
    g = sys.graph
    out = push_kernel(g.offsets, g.targets, sys.op.arc_weights, sys.theta, x, r, seeds,
                      omega=omega, signed=omega > 1.0, max_sweeps=max_sweeps)
    out.update(x=x, r=r)
    return out


def local_hk(g, tau: float, s: int, eps: float, max_sweeps: int = 1_000_000) -> dict:
    """src/local_solvers.py:664-696; returns f_hat and the raw (v, r)."""
    from paper_2410_21634_b200.systems import make_hk_system
    sys = make_hk_system(g, tau, s, eps)
    N = sys.op.stage_count
    base_w = _arrf(sys.op.arc_weights)
    stage_w = _arrf(sys.op.stage_weights if N else np.zeros(1))
    th = _arrf(sys.theta)
    v = np.zeros(sys.dim)
    r = _arrf(sys.b).copy()
    off, tg = _arr64(g.offsets), _arr64(g.targets)
    rep = _Report()
    lib().orc_hk_push(C.c_int64(g.n), C.c_int64(N), _p(off, C.c_int64), _p(tg, C.c_int64),
                      _p(base_w), _p(stage_w), _p(th), _p(v), _p(r), C.c_int64(s),
                      C.c_int64(max_sweeps), C.byref(rep))
    out = _unpack(rep)
    out.update(v=v, r=r, f_hat=sys.back_transform(v), stage_count=N,
               residual_mass=float(np.abs(r).sum()))
    return out


def gradient_descent(sys, max_sweeps: int = 10_000) -> dict:
    """src/global_solvers.py:124-152."""
    off, tg, w, th = _sys_arrays(sys)
    n = sys.dim
    b = _arrf(sys.b)
    x, r = np.zeros(n), np.zeros(n)
    rep = _Report()
    lib().orc_gradient_descent(C.c_int64(n), _p(off, C.c_int64), _p(tg, C.c_int64), _p(w), _p(th),
                               _p(b), _p(x), _p(r), C.c_int64(max_sweeps), C.byref(rep))
    out = _unpack(rep)
    out.update(x=x, r=r)
    return out


def _cmp_args(gpu, k: int, topk: int):
    """ctypes arguments of the optional per-seed GPU comparison (x as sparse
    (node, value) segments, caller ids) and the arrays it fills."""
    if gpu is None:
        nul = C.c_void_p()
        return [nul] * 4 + [nul, nul, nul, C.c_int32(0)], None
    g_off = _arr64(gpu.x_offset)
    g_cnt = _arr64(gpu.x_count)
    g_nodes = np.ascontiguousarray(gpu.x_nodes, dtype=np.int32)
    g_vals = _arrf(gpu.x_vals)
    l1d, l1r, tk = np.zeros(k), np.zeros(k), np.zeros(k, np.int32)
    keep = (g_off, g_cnt, g_nodes, g_vals)
    args = [_p(g_off, C.c_int64), _p(g_cnt, C.c_int64), _p(g_nodes, C.c_int32), _p(g_vals),
            _p(l1d), _p(l1r), _p(tk, C.c_int32), C.c_int32(topk)]
    return args, (l1d, l1r, tk, keep)


def _cmp_out(out: dict, res) -> dict:
    if res is not None:
        l1d, l1r, tk, _ = res
        out["x_l1_diff"], out["x_l1_ref"] = l1d, l1r
        out["x_l1_rel"] = l1d / np.where(l1r > 0, l1r, 1.0)
        out["topk_identical"] = (tk & 1).astype(bool)
        out["topk_identical_up_to_ties"] = (tk & 2).astype(bool)
    return out


def batch_local_gd(g, alpha: float, eps: float, seeds, threads: int,
                   max_sweeps: int = 1_000_000, arc_w=None, theta=None, method: str = "local-gd",
                   omega: float = 1.0, gpu=None, topk: int = 100, xsum: bool = True) -> dict:
    """Per-seed reference local_gd (or local_sor) over many host threads (CPU
    baseline).  gpu: a BatchOutput of the same seeds -> per-seed l1 of
    x_gpu - x_ref, l1 of x_ref and the top-k ranking check."""
    from paper_2410_21634_b200.systems import arc_weights_for, theta_vector
    off, tg = _arr64(g.offsets), _arr64(g.targets)
    w = _arrf(arc_w if arc_w is not None else arc_weights_for(g, 1.0 - alpha, "rw"))
    th = _arrf(theta if theta is not None else theta_vector(g, eps * alpha))
    sd = _arr64(seeds)
    k = sd.shape[0]
    sw, ops, pu = np.zeros(k, np.int64), np.zeros(k, np.int64), np.zeros(k, np.int64)
    cv = np.zeros(k, np.int32)
    xs = np.zeros(k)
    cargs, cres = _cmp_args(gpu, k, topk)
    lib().orc_batch_local(C.c_int64(g.n), _p(off, C.c_int64), _p(tg, C.c_int64), _p(w), _p(th),
                             C.c_double(alpha), C.c_int32(1 if method == "local-sor" else 0),
                             C.c_double(omega), _p(sd, C.c_int64), C.c_int64(k),
                             C.c_int64(max_sweeps), C.c_int32(threads), _p(sw, C.c_int64),
                             _p(ops, C.c_int64), _p(pu, C.c_int64), _p(cv, C.c_int32),
                             _p(xs) if xsum else C.c_void_p(), *cargs)
    return _cmp_out({"sweeps": sw, "total_ops": ops, "pushes": pu, "converged": cv.astype(bool),
                     "xsum": xs}, cres)


def batch_gd_rule(n: int, offsets, targets32, alpha: float, eps: float, seeds, threads: int,
                  max_sweeps: int = 1_000_000, gpu=None, topk: int = 100) -> dict:
    """Reference LocalGD-PPR per seed with the operator / thresholds evaluated
    from their rules and int32 targets (papers100M scale; no l1 logs): a
    checker for the device batch, never a timed baseline."""
    off = _arr64(offsets)
    tg = np.ascontiguousarray(targets32, dtype=np.int32)
    sd = _arr64(seeds)
    k = sd.shape[0]
    sw, ops, pu = np.zeros(k, np.int64), np.zeros(k, np.int64), np.zeros(k, np.int64)
    cv = np.zeros(k, np.int32)
    cargs, cres = _cmp_args(gpu, k, topk)
    lib().orc_batch_gd_rule(C.c_int64(n), _p(off, C.c_int64), _p(tg, C.c_int32), C.c_double(alpha),
                            C.c_double(eps), _p(sd, C.c_int64), C.c_int64(k), C.c_int64(max_sweeps),
                            C.c_int32(threads), _p(sw, C.c_int64), _p(ops, C.c_int64),
                            _p(pu, C.c_int64), _p(cv, C.c_int32), *cargs)
    return _cmp_out({"sweeps": sw, "total_ops": ops, "pushes": pu, "converged": cv.astype(bool)},
                    cres)


def batch_local_ch(g, alpha: float, eps: float, seeds, threads: int, mu: float, L: float,
                   problem: str = "ppr", max_sweeps: int | None = None, gpu=None,
                   topk: int = 100, hb: bool = False) -> dict:
    """Per-seed reference local_ch over many host threads (CPU baseline of
    the LocalCH batch): PPR (b = alpha e_s) or Katz (b = e_s, w = alpha)."""
    from paper_2410_21634_b200.systems import arc_weights_for, theta_vector
    if max_sweeps is None:
        gap = max(mu, 1e-12)
        max_sweeps = max(1000, int(10 * math.log(max(1.0 / max(eps, 1e-300), 2.0)) / gap))
    off, tg = _arr64(g.offsets), _arr64(g.targets)
    if problem == "ppr":
        w, th, bval = arc_weights_for(g, 1.0 - alpha, "rw"), theta_vector(g, eps * alpha), alpha
    else:
        w, th, bval = np.full(tg.shape[0], float(alpha)), theta_vector(g, eps), 1.0
    w, th = _arrf(w), _arrf(th)
    sd = _arr64(seeds)
    k = sd.shape[0]
    sw, ops = np.zeros(k, np.int64), np.zeros(k, np.int64)
    cv = np.zeros(k, np.int32)
    xs = np.zeros(k)
    cargs, cres = _cmp_args(gpu, k, topk)
    lib().orc_batch_local_ch(C.c_int64(g.n), _p(off, C.c_int64), _p(tg, C.c_int64), _p(w), _p(th),
                             C.c_double(bval), C.c_double(mu), C.c_double(L), _p(sd, C.c_int64),
                             C.c_int64(k), C.c_int64(max_sweeps), C.c_int32(threads),
                             _p(sw, C.c_int64), _p(ops, C.c_int64), _p(cv, C.c_int32), _p(xs),
                             *cargs, C.c_int32(int(hb)))
    return _cmp_out({"sweeps": sw, "total_ops": ops, "converged": cv.astype(bool), "xsum": xs},
                    cres)


def batch_local_hk(g, tau: float, eps: float, seeds, threads: int,
                   max_sweeps: int = 1_000_000, gpu=None, topk: int = 100) -> dict:
    """Per-seed reference local_hk over many host threads (CPU baseline of
    the heat-kernel batch); dense (N+1) n state per thread as the reference."""
    from paper_2410_21634_b200.systems import make_hk_system
    sd = _arr64(seeds)
    sys = make_hk_system(g, tau, int(sd[0]) if sd.size else 0, eps)
    N = sys.op.stage_count
    base_w = _arrf(sys.op.arc_weights)
    stage_w = _arrf(sys.op.stage_weights if N else np.zeros(1))
    th = _arrf(sys.theta)
    off, tg = _arr64(g.offsets), _arr64(g.targets)
    k = sd.shape[0]
    sw, ops = np.zeros(k, np.int64), np.zeros(k, np.int64)
    cv = np.zeros(k, np.int32)
    fs = np.zeros(k)
    cargs, cres = _cmp_args(gpu, k, topk)
    lib().orc_batch_hk(C.c_int64(g.n), C.c_int64(N), _p(off, C.c_int64), _p(tg, C.c_int64),
                       _p(base_w), _p(stage_w), _p(th), C.c_double(tau), _p(sd, C.c_int64),
                       C.c_int64(k), C.c_int64(max_sweeps), C.c_int32(threads), _p(sw, C.c_int64),
                       _p(ops, C.c_int64), _p(cv, C.c_int32), _p(fs), *cargs)
    return _cmp_out({"sweeps": sw, "total_ops": ops, "converged": cv.astype(bool), "fsum": fs,
                     "stage_count": N}, cres)


def pairwise_sum(a, take_abs: bool = False) -> float:
    a = _arrf(a)
    return float(lib().orc_pairwise_sum(_p(a), C.c_int64(a.shape[0]), C.c_int32(int(take_abs))))
