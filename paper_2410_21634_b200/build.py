"""Build libgdiff.so (sm_100a) in-tree with nvcc.

    python -m paper_2410_21634_b200.build [-v]

Objects go to paper_2410_21634_b200/build/, the shared library next to
this file so it travels with the source tree to the GPU box.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libgdiff.so")
BUILD = os.path.join(HERE, "build")
INCLUDE = os.path.abspath(os.path.join(HERE, "..", "include"))

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", f"-I{INCLUDE}"]
SOURCES = ["graph.cu", "exact.cu", "fifo.cu", "fifo_batch.cu", "global.cu", "batch.cu", "batch_cta.cu",
           "sor_win.cu",
           "batch_signed.cu",
           "generate.cu", "graph_edit.cu", "hk.cu",
           "feature_push.cu"]


def _deps_newer(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    dep = [src, os.path.join(CSRC, "common.cuh"), os.path.join(CSRC, "window.cuh"),
           os.path.join(INCLUDE, "gdiff.h")]
    return any(os.path.getmtime(d) > t for d in dep)


def _compile(src: str, verbose: bool, checked: bool = False) -> str:
    bdir = BUILD + ("_checked" if checked else "")
    obj = os.path.join(bdir, os.path.splitext(src)[0] + ".o")
    path = os.path.join(CSRC, src)
    if _deps_newer(obj, path):
        cmd = [NVCC, *ARCH, *FLAGS, *(["-DGD_CHECKED"] if checked else []), "-c", path, "-o", obj]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{p.stderr}")
        if verbose:
            sys.stderr.write(p.stderr)
    return obj


def build(verbose: bool = False, checked: bool = False) -> str:
    """checked=True: libgdiff_checked.so with the device-side GD_DCHECK bounds
    checks compiled in (csrc/common.cuh), for debugging runs via GDIFF_LIB."""
    os.makedirs(BUILD + ("_checked" if checked else ""), exist_ok=True)
    out = OUT.replace("libgdiff.so", "libgdiff_checked.so") if checked else OUT
    with ThreadPoolExecutor(max_workers=min(8, len(SOURCES))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, checked), SOURCES))
    if not os.path.exists(out) or any(os.path.getmtime(o) > os.path.getmtime(out) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", out, *objs, "-lcudart"]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"link failed:\n{p.stderr}")
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, checked="--checked" in sys.argv))
