"""Golden vectors for LocalHB (heavy-ball momentum), generated with the
REFERENCE's own sweep machinery.

The reference has no heavy-ball solver (its momentum method is LocalCH,
src/local_solvers.py:473-538).  LocalHB is restated here exactly as local_ch is
written -- the reference's _SweepDriver (signed frontier, _apply_update_seq,
_filter_frontier, _l1_and_min), the momentum stamps and the divergence abort --
with Polyak's stationary coefficients for eigenvalues in [mu, L] instead of the
Chebyshev recurrence:

    eta = 4 / (sqrt(L) + sqrt(mu))^2,   beta = ((sqrt(L) - sqrt(mu)) / (sqrt(L) + sqrt(mu)))^2
    sweep 0: vals = eta * r_S;  sweep t > 0: vals = eta * r_S + beta * prev_S

(the limit the Chebyshev coefficients of local_ch converge to).  Every array
operation is the reference's, so the fixture pins the C restatement
(oracle/gdiff_oracle.c orc_local_hb) and the device solvers to the reference's
kernels.  Run in the authoring container:

    PYTHONPATH=/root/reference/pkg/src:. NUMBA_CACHE_DIR=/tmp/nb \\
        python tests/golden/make_golden_hb.py
"""
from __future__ import annotations

import math
import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from graphdiff import local_solvers as rls  # noqa: E402  (the reference)
from graphdiff import systems as rsys  # noqa: E402
from graphdiff.graph import CsrGraph as RefCsr  # noqa: E402
from graphdiff.metrics import sample_sources  # noqa: E402

from paper_2410_21634_b200.synth import rmat_graph  # noqa: E402

warnings.simplefilter("ignore")


def hb_coefficients(mu: float, L: float):
    sq, sm = math.sqrt(L), math.sqrt(mu)
    return 4.0 / ((sq + sm) * (sq + sm)), ((sq - sm) / (sq + sm)) ** 2


def local_hb_reference(sys, mu, L, max_sweeps=None):
    """local_ch (src/local_solvers.py:473-538) with heavy-ball coefficients."""
    eps = sys.eps
    if max_sweeps is None:
        gap = max(mu, 1e-12)
        max_sweeps = max(1000, int(10 * math.log(max(1.0 / max(eps, 1e-300), 2.0)) / gap))
    drv = rls._SweepDriver(sys, signed=True, parallel=False)
    eta, beta = hb_coefficients(mu, L)
    mom = np.zeros(sys.dim)
    mom_stamp = np.full(sys.dim, -2, np.int64)
    b_l1 = float(np.abs(sys.b).sum())
    sweeps, total_ops, converged, aborted = 0, 0, True, False
    while drv.frontier.shape[0]:
        if sweeps >= max_sweeps:
            converged = False
            break
        fr = drv.frontier
        svol = drv.frontier_volume()
        rvals = drv.r[fr]
        sgamma = float(np.abs(rvals).sum())
        if sweeps == 0:
            vals = eta * rvals
        else:
            prev = np.where(mom_stamp[fr] == sweeps - 1, mom[fr], 0.0)
            vals = eta * rvals + beta * prev
        drv.x[fr] += vals
        mom[fr] = vals
        mom_stamp[fr] = sweeps
        drv.apply(vals)
        drv.log_sweep(svol, sgamma)
        total_ops += svol
        sweeps += 1
        if drv.l1_log[-1] > 10.0 * b_l1:
            converged, aborted = False, True
            break
    return {"x": drv.x, "r": drv.r, "sweeps": sweeps, "total_ops": total_ops,
            "converged": converged, "diverged": aborted, "vol_log": np.asarray(drv.vol_log),
            "gamma_log": np.asarray(drv.gamma_log), "l1_log": np.asarray(drv.l1_log),
            "min_residual": drv.min_r}


def main():
    d = {}
    g = rmat_graph(2000, 9000, seed=4)
    rg = RefCsr(n=g.n, offsets=np.asarray(g.offsets), targets=np.asarray(g.targets))
    d["graph/n"] = np.int64(g.n)
    d["graph/offsets"] = np.asarray(g.offsets, np.int64)
    d["graph/targets"] = np.asarray(g.targets, np.int64)
    seeds = sample_sources(rg, 6, seed=1)
    cases = []
    for s in seeds:
        cases.append(("ppr", 0.1, 1e-6, int(s), None, None))
    cases.append(("ppr", 0.15, 1e-7, int(seeds[2]), None, None))
    lam = float(rsys.default_katz_alpha(rg)) if hasattr(rsys, "default_katz_alpha") else None
    cases.append(("katz", 0.9 / float(rg.d_max), 1e-6, int(seeds[0]), None, None))
    for i, (prob, alpha, eps, s, mu, L) in enumerate(cases):
        if prob == "ppr":
            sys_ = rsys.make_ppr_system(rg, alpha, s, eps, symmetrized=True)
            mu, L = alpha, 2.0 - alpha
        else:
            sys_ = rsys.make_katz_system(rg, alpha, s, eps, lam_hat=0.0)
            lam_e = float(rg.d_max)
            mu, L = 1.0 - alpha * lam_e, 1.0 + alpha * lam_e
        out = local_hb_reference(sys_, mu, L)
        k = f"c{i}"
        d[f"{k}/problem"] = np.str_(prob)
        d[f"{k}/alpha"], d[f"{k}/eps"], d[f"{k}/source"] = np.float64(alpha), np.float64(eps), np.int64(s)
        d[f"{k}/mu"], d[f"{k}/L"] = np.float64(mu), np.float64(L)
        for name in ("x", "r", "vol_log", "gamma_log", "l1_log"):
            d[f"{k}/{name}"] = np.asarray(out[name])
        for name in ("sweeps", "total_ops"):
            d[f"{k}/{name}"] = np.int64(out[name])
        d[f"{k}/converged"] = np.bool_(out["converged"])
        d[f"{k}/diverged"] = np.bool_(out["diverged"])
        d[f"{k}/min_residual"] = np.float64(out["min_residual"])
        print(k, prob, s, out["sweeps"], out["total_ops"], out["converged"], out["diverged"])
    d["cases"] = np.int64(len(cases))
    d["source"] = np.str_("graphdiff._SweepDriver + local_ch loop with heavy-ball coefficients "
                          "(tests/golden/make_golden_hb.py)")
    _ = lam
    np.savez_compressed(os.path.join(HERE, "hb.npz"), **d)


if __name__ == "__main__":
    main()
