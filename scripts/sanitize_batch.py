"""Small runs of every batched kernel for compute-sanitizer (memcheck /
racecheck / synccheck): cora-shape LocalGD (one CTA per seed, the round kernel
in waves and in the streaming form), LocalCH, LocalGS / LocalSOR, heat kernel,
want_r extraction and the exact re-solve; each checked against the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2410_21634_b200.batch import BatchSolver, hk_params  # noqa: E402
from paper_2410_21634_b200.metrics import sample_sources  # noqa: E402
from paper_2410_21634_b200.synth import rmat_graph  # noqa: E402

g = rmat_graph(2708, 5278, seed=0)
seeds = sample_sources(g, 12, seed=0)
ref = O.batch_local_gd(g, 0.1, 1e-5, seeds, 4)
runs = [("cta", {}, {}), ("rounds", {"GDIFF_STREAM": "0"}, {}),
        ("stream", {"GDIFF_STREAM": "1", "GDIFF_COHORT": "2"}, {}),
        ("rounds-want_r", {}, {"want_r": True}), ("rounds-exact", {}, {"resolve": "all"})]
for name, env, kw in runs:
    os.environ.update(env)
    os.environ["GDIFF_BATCH_MODE"] = "cta" if name == "cta" else "rounds"
    s = BatchSolver(g, 0.1, 1e-5, slots=4, **kw)
    out = s.solve(seeds)
    s.close()
    for k in env:
        os.environ.pop(k)
    assert np.array_equal(out.total_ops, ref["total_ops"]), name
    print(name, "ok", int(out.total_ops.sum()))
os.environ["GDIFF_BATCH_MODE"] = "rounds"
ch = BatchSolver(g, 0.1, 1e-5, slots=4, method="local-ch", mu=0.1, L=1.9).solve(seeds)
cref = O.batch_local_ch(g, 0.1, 1e-5, seeds, 4, 0.1, 1.9)
assert np.array_equal(ch.total_ops, cref["total_ops"])
print("local-ch ok")
for om in (1.0, 1.39):
    so = BatchSolver(g, 0.1, 1e-5, slots=4, method="local-sor", omega=om).solve(seeds)
    sref = O.batch_local_gd(g, 0.1, 1e-5, seeds, 4, method="local-sor", omega=om)
    assert np.array_equal(so.total_ops, sref["total_ops"])
    print("local-sor", om, "ok")
hk = BatchSolver(g, 0.1, 1e-4, slots=4, method="local-hk",
                 hk=hk_params(g, 3.0, 1e-4, int(np.argmax(g.degrees)))).solve(seeds[:4])
print("local-hk ok", int(hk.total_ops.sum()))
