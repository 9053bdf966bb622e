"""Golden vectors of the reference's global Chebyshev and heat-kernel Taylor
solvers (src/global_solvers.py:155-235) and the degree-generalized feature
push (src/dynamic.py:199-222), produced by running the reference.

    PYTHONPATH=/root/reference/pkg/src:. NUMBA_CACHE_DIR=/tmp/nb \\
        python tests/golden/make_golden_global.py
"""

from __future__ import annotations

import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from graphdiff import global_solvers as rgs  # noqa: E402  (the reference)
from graphdiff import synth as rsyn  # noqa: E402
from graphdiff import systems as rsys  # noqa: E402

warnings.simplefilter("ignore")


def main():
    d = {}
    er500 = rsyn.erdos_renyi(500, 0.02, seed=21)
    er60 = rsyn.erdos_renyi(60, 0.1, seed=7)
    for name, g in (("er500", er500), ("er60", er60)):
        d[f"graph/{name}/n"] = np.int64(g.n)
        d[f"graph/{name}/offsets"] = np.asarray(g.offsets, dtype=np.int64)
        d[f"graph/{name}/targets"] = np.asarray(g.targets, dtype=np.int64)

    def put(key, st, rp):
        d[f"{key}/x"], d[f"{key}/r"] = np.asarray(st.x), np.asarray(st.r)
        d[f"{key}/sweeps"] = np.int64(rp.sweeps)
        d[f"{key}/total_ops"] = np.int64(rp.total_ops)
        d[f"{key}/converged"] = np.bool_(rp.converged)
        d[f"{key}/l1_log"] = np.asarray(rp.residual_l1_trace, dtype=np.float64)
        if "l2_trace" in rp.notes:
            d[f"{key}/l2_log"] = np.asarray(rp.notes["l2_trace"], dtype=np.float64)
            d[f"{key}/delta_log"] = np.asarray(rp.notes["delta_trace"], dtype=np.float64)

    put("er500/ppr/ch", *rgs.chebyshev(rsys.make_ppr_system(er500, 0.15, 0, 1e-6)))
    put("er60/ppr/ch", *rgs.chebyshev(rsys.make_ppr_system(er60, 0.2, 3, 1e-8)))
    ka = 0.9 / er60.d_max
    put("er60/katz/ch", *rgs.chebyshev(rsys.make_katz_system(er60, ka, 0, 1e-6, lam_hat=0.0),
                                       rgs.GlobalConfig(mu=1.0 - ka * er60.d_max,
                                                        L=1.0 + ka * er60.d_max)))
    put("er60/ppr/ch_cap", *rgs.chebyshev(rsys.make_ppr_system(er60, 0.2, 3, 1e-8),
                                          rgs.GlobalConfig(max_sweeps=3)))
    for tau in (1.0, 5.0):
        put(f"er500/hk/taylor{tau}", *rgs.hk_taylor_global(rsys.make_hk_system(er500, tau, 0, 1e-5)))
    d["katz_alpha"] = np.float64(ka)
    # degree-generalized signed feature push (src/dynamic.py:199-222)
    from graphdiff import dynamic as rdyn
    rng = np.random.default_rng(5)
    src = rng.standard_normal(er500.n) * (rng.random(er500.n) < 0.05)
    for beta in (0.0, 0.5, 1.0):
        pair, rp = rdyn.beta_push(er500, src, 0.15, beta, 1e-4)
        k = f"er500/betapush{beta}"
        d[f"{k}/p"], d[f"{k}/r"] = pair.p, pair.r
        d[f"{k}/sweeps"] = np.int64(rp.sweeps)
        d[f"{k}/total_ops"] = np.int64(rp.total_ops)
        d[f"{k}/parked"] = np.float64(rp.notes["parked_mass"])
    d["betapush/source"] = src
    np.savez_compressed(os.path.join(HERE, "global.npz"), **d)
    print("wrote global.npz", len(d))


if __name__ == "__main__":
    main()
