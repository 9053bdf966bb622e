"""Shared parity helpers: rebuild golden systems, compare solver outputs."""

from __future__ import annotations

import numpy as np

from conftest import golden_graph
from paper_2410_21634_b200 import systems as S


def local_cases(d):
    """Keys of single-system fixtures, e.g. 'er500/ppr/local_gd'."""
    return sorted(k[:-len("/param/problem")] for k in d if k.endswith("/param/problem"))


def param(d, key, name, default=None):
    k = f"{key}/param/{name}"
    if k not in d:
        return default
    v = d[k]
    return v.item() if v.shape == () else v


def build_system(d, key):
    g = golden_graph(d, str(param(d, key, "graph")))
    prob = str(param(d, key, "problem"))
    alpha, eps, s = float(param(d, key, "alpha")), float(param(d, key, "eps")), int(param(d, key, "source"))
    if prob == "ppr":
        return S.make_ppr_system(g, alpha, s, eps)
    if prob == "katz":
        return S.make_katz_system(g, alpha, s, eps, lam_hat=0.0)
    raise ValueError(prob)


def method_of(key):
    return key.rsplit("/", 1)[1]


def solver_kwargs(d, key):
    m = method_of(key)
    kw = {}
    if m.startswith("local_sor"):
        kw["omega"] = float(param(d, key, "omega"))
    if m == "local_ch" and param(d, key, "mu") is not None:
        kw["mu"], kw["L"] = float(param(d, key, "mu")), float(param(d, key, "L"))
    if param(d, key, "max_sweeps") is not None:
        kw["max_sweeps"] = int(param(d, key, "max_sweeps"))
    return kw


def assert_matches(d, key, out, logs_exact=True, rtol_logs=1e-12):
    """out: dict with x, r, sweeps, total_ops, vol_log, gamma_log, l1_log,
    min_residual, support_size, converged (+ frontier_sizes / trace / signs)."""
    assert np.array_equal(out["x"], d[f"{key}/x"]), f"{key}: x differs"
    assert np.array_equal(out["r"], d[f"{key}/r"]), f"{key}: r differs"
    assert int(out["sweeps"]) == int(d[f"{key}/sweeps"]), key
    assert int(out["total_ops"]) == int(d[f"{key}/total_ops"]), key
    assert bool(out["converged"]) == bool(d[f"{key}/converged"]), key
    assert np.array_equal(np.asarray(out["vol_log"], dtype=np.int64), d[f"{key}/vol_log"]), key
    assert int(out["support_size"]) == int(d[f"{key}/support_size"]), key
    for name, gk in (("gamma_log", "gamma_log"), ("l1_log", "l1_log")):
        got, ref = np.asarray(out[name], dtype=np.float64), d[f"{key}/{gk}"]
        assert got.shape == ref.shape, (key, name)
        if logs_exact:
            assert np.array_equal(got, ref), (key, name)
        else:
            np.testing.assert_allclose(got, ref, rtol=rtol_logs, atol=1e-300, err_msg=f"{key} {name}")
    if logs_exact:
        assert float(out["min_residual"]) == float(d[f"{key}/min_residual"]), key
    else:
        assert np.isclose(float(out["min_residual"]), float(d[f"{key}/min_residual"]),
                          rtol=1e-12, atol=1e-300), key
    if f"{key}/frontier_sizes" in d and "frontier_sizes" in out:
        assert np.array_equal(np.asarray(out["frontier_sizes"]), d[f"{key}/frontier_sizes"]), key
    if f"{key}/trace_flat" in d and out.get("frontier_trace") is not None:
        tr = out["frontier_trace"]
        flat = np.concatenate(tr).astype(np.int64) if len(tr) else np.empty(0, np.int64)
        assert np.array_equal(flat, d[f"{key}/trace_flat"]), f"{key}: frontier trace differs"
        assert np.array_equal([len(f) for f in tr], d[f"{key}/trace_sizes"]), key
    if f"{key}/sweep_signs" in d and "sign_log" in out:
        assert np.array_equal(np.asarray(out["sign_log"], dtype=np.int8), d[f"{key}/sweep_signs"]), key
    if f"{key}/diverged" in d and "diverged" in out:
        assert bool(out["diverged"]) == bool(d[f"{key}/diverged"]), key


def report_dict(state, report):
    """(SolverState, LocalReport) -> the dict assert_matches expects."""
    out = {"x": state.x, "r": state.r, "sweeps": report.sweeps, "total_ops": report.total_ops,
           "converged": report.converged, "vol_log": report.vol_log,
           "gamma_log": report.gamma_log, "l1_log": report.residual_l1_trace,
           "min_residual": report.min_residual, "support_size": report.support_size}
    if "frontier_sizes" in report.notes:
        out["frontier_sizes"] = report.notes["frontier_sizes"]
    if state.frontier_trace is not None:
        out["frontier_trace"] = state.frontier_trace
    if "sweep_signs" in report.notes:
        out["sign_log"] = report.notes["sweep_signs"]
    if "diverged" in report.notes:
        out["diverged"] = report.notes["diverged"]
    return out
