"""R-MAT graphs of the configs' OGB shapes, generated and CSR-built on the GPU.

Candidate edges come from the device kernel ``gd_rmat_keys_device`` (same
counter-based stream as ``synth.rmat_edges``); deduplication ("first m
distinct undirected edges in generation order") and canonical CSR assembly
use device sorts.  The result is identical to ``synth.rmat_graph`` -- the
host builder the tests compare against -- but takes seconds instead of
minutes at the products shape (the reference's host builder took 435 s).
"""

from __future__ import annotations

import ctypes as C
import math

from . import _lib as gdl
from .synth import RMAT_SHAPES

__all__ = ["rmat_csr_device", "RMAT_SHAPES"]


def rmat_csr_device(n: int, m: int, seed: int = 0, abc=(0.57, 0.19, 0.19), device: int = 0):
    """Return (row_ptr int64[n+1], col int32[2m]) as CUDA tensors."""
    import torch

    lib = gdl.load()
    dev = torch.device("cuda", device)
    scale = max(1, int(math.ceil(math.log2(max(n, 2)))))
    chunk = max(1024, int(m * 1.25) + 1024)
    st = torch.cuda.current_stream(dev).cuda_stream
    keys = torch.empty(0, dtype=torch.int64, device=dev)
    first = torch.empty(0, dtype=torch.int64, device=dev)
    drawn = 0
    while True:
        buf = torch.empty(chunk, dtype=torch.int64, device=dev)
        gdl.check(lib.gd_rmat_keys_device(scale, n, drawn, chunk, seed, abc[0], abc[1], abc[2],
                                          C.c_void_p(buf.data_ptr()), C.c_void_p(st)))
        ok = buf >= 0
        idx = torch.arange(drawn, drawn + chunk, dtype=torch.int64, device=dev)[ok]
        keys = torch.cat([keys, buf[ok]])
        first = torch.cat([first, idx])
        del buf, ok, idx
        drawn += chunk
        sk, perm = torch.sort(keys, stable=True)
        head = torch.ones_like(sk, dtype=torch.bool)
        head[1:] = sk[1:] != sk[:-1]
        keys, first = sk[head], first[perm][head]
        del sk, perm, head
        if keys.numel() >= m:
            order = torch.argsort(first)[:m]
            sel = keys[order]
            break
    del keys, first
    lo, hi = sel // n, sel % n
    arc = torch.sort(torch.cat([lo * n + hi, hi * n + lo])).values
    del lo, hi, sel
    src = arc // n
    col = (arc % n).to(torch.int32)
    del arc
    row = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    row[1:] = torch.cumsum(torch.bincount(src, minlength=n), 0)
    return row, col


def relabel_by_degree(row, col):
    """Renumber nodes by descending degree (ties by id) on the device.

    Returns (row2, col2, perm, inv) with perm[old] = new, inv[new] = old.
    Hubs -- which receive most residual contributions -- end up in a
    contiguous low-id block, so per-seed residual updates share 32 B sectors
    and stay in L2.  Frontier sets, sweeps and operation counts are
    invariant under the renumbering.
    """
    import torch

    n = row.numel() - 1
    deg = row[1:] - row[:-1]
    key = (deg.max() - deg) * n + torch.arange(n, device=row.device)
    inv = torch.argsort(key)
    perm = torch.empty_like(inv)
    perm[inv] = torch.arange(n, device=row.device)
    src = torch.repeat_interleave(torch.arange(n, device=row.device), deg)
    akey = perm[src] * n + perm[col.long()]
    akey = torch.sort(akey).values
    col2 = (akey % n).to(torch.int32)
    row2 = torch.zeros(n + 1, dtype=torch.int64, device=row.device)
    row2[1:] = torch.cumsum(deg[inv], 0)
    return row2, col2, perm, inv
