"""``bench`` command of the reference CLI with ``--backend cuda``.

Mirrors ``graphdiff bench`` (src/cli.py:150-190, arguments :290-320): the
same graph/eps/alpha/omega/sources arguments, records written with
``write_records_jsonl`` / ``write_records_csv`` and the same one-line
``{"speedup": ..., "sources": ...}`` summary; exit code 0 when every record
converged, 2 otherwise, 1 on usage or input errors (src/cli.py:36-41,
:347-361).  Records carry ``backend: "cuda"``.  Families run on the device:
``gd`` (global GD per source + batched LocalGD), ``gs`` / ``sor`` / ``ch``
(batched local-gs / local-sor / local-ch; their global counterparts stay in
the reference, so their speedup entry is null).

    python -m paper_2410_21634_b200.cli bench --graph g.csr --problem ppr \\
        --methods gd,sor --num-sources 64 --eps 1e-6 --out records.jsonl
"""

from __future__ import annotations

import argparse
import json
import math
import sys

from .graph import GraphFormatError, GraphStructureError, load_csr_cache, load_edge_list
from .metrics import sample_sources
from .records import bench_family, speedup_ratio, write_records_csv, write_records_jsonl
from .systems import SystemError

__all__ = ["main", "build_parser", "resolve_eps"]


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        self.print_usage(sys.stderr)
        sys.stderr.write(f"error: {message}\n")
        raise SystemExit(1)


def _load_graph(path: str):
    if path.endswith(".csr"):
        return load_csr_cache(path)
    with open(path, "r") as fh:
        return load_edge_list(fh)


def resolve_eps(token: str, g) -> float:
    """Literal float or 1/n, 1/m, 1/sqrt n (src/cli.py:50-63)."""
    tok = " ".join(token.strip().lower().replace("(", " ").replace(")", " ").split())
    if tok == "1/n":
        return 1.0 / g.n
    if tok == "1/m":
        return 1.0 / max(g.m, 1)
    if tok in ("1/sqrt n", "1/sqrtn", "1/sqrt"):
        return 1.0 / math.sqrt(g.n)
    try:
        return float(token)
    except ValueError as exc:
        raise SystemError(f"cannot parse eps {token!r}") from exc


def cmd_bench(args) -> int:
    from .local_solvers import optimal_omega
    from .systems import default_katz_alpha

    g = _load_graph(args.graph)
    eps = resolve_eps(args.eps, g)
    if args.problem == "katz" and args.alpha is None:
        args.alpha = default_katz_alpha(g)
    omega = optimal_omega(args.alpha) if args.omega == "auto" else float(args.omega)
    sources = sample_sources(g, args.num_sources, seed=args.seed)
    families = [f.strip() for f in args.methods.split(",") if f.strip()]
    for fam in families:
        if fam not in ("gs", "sor", "gd", "ch"):
            raise SystemError(f"unknown method family {fam}")
    records = []
    for fam in families:
        records += bench_family(g, args.graph, fam, sources, args.alpha, eps, problem=args.problem,
                                omega=omega, max_sweeps=args.max_sweeps)
    (write_records_csv if args.format == "csv" else write_records_jsonl)(records, args.out,
                                                                          timing=args.timing)
    by_method: dict = {}
    for rec in records:
        by_method.setdefault(rec.method, []).append(rec)
    summary = {}
    for fam in families:
        try:
            summary[f"{fam}/local-{fam}"] = speedup_ratio(by_method[fam], by_method[f"local-{fam}"])
        except (KeyError, ValueError):
            summary[f"{fam}/local-{fam}"] = None
    print(json.dumps({"speedup": summary, "sources": len(sources), "backend": args.backend},
                     sort_keys=True))
    return 0 if all(r.converged for r in records) else 2


def build_parser() -> argparse.ArgumentParser:
    parser = _Parser(prog="graphdiff-b200", description="B200 local diffusion solvers")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("bench", help="paired global/local benchmark sweep on the device")
    p.add_argument("--graph", required=True, help="edge list or .csr cache path")
    p.add_argument("--eps", default="1/n", help="float or 1/n, 1/m, '1/sqrt n'")
    p.add_argument("--alpha", type=float, default=None)
    p.add_argument("--omega", default="1.0", help="float or 'auto' for omega*")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--max-sweeps", type=int, default=None)
    p.add_argument("--out", default="report.json")
    p.add_argument("--format", choices=["json", "csv"], default="json")
    p.add_argument("--timing", action="store_true", help="include wall-clock fields")
    p.add_argument("--problem", choices=["ppr", "katz"], required=True)
    p.add_argument("--methods", default="gd", help="comma list of gd, gs, sor, ch")
    p.add_argument("--num-sources", type=int, default=50)
    p.add_argument("--backend", choices=["cuda"], default="cuda")
    p.set_defaults(func=cmd_bench)
    return parser


def main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as exc:
        return exc.code if isinstance(exc.code, int) else 1
    if args.alpha is None and args.problem == "ppr":
        args.alpha = 0.1
    try:
        return args.func(args)
    except (GraphFormatError, GraphStructureError, SystemError, ValueError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
