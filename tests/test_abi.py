"""The C-ABI library builds for sm_100a, loads without a GPU, and exports
every entry point include/gdiff.h declares (no compute calls here)."""

import ctypes
import os
import re
import subprocess

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "gdiff.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gd_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("gd_graph_create", "gd_local_gd", "gd_local_ch", "gd_push_kernel", "gd_hk_push",
                 "gd_gradient_descent", "gd_batch_create", "gd_batch_solve_device",
                 "gd_batch_solve_host", "gd_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2410_21634_b200.build import build
    path = build()
    lib = ctypes.CDLL(path)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.gd_version() == 1


def test_python_binding_covers_header():
    from paper_2410_21634_b200 import _lib
    assert set(_declared()) == set(_lib.SIGNATURES)


def test_library_is_sm100a_only():
    from paper_2410_21634_b200.build import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build()],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs
