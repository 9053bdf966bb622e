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


def rmat_csr_device_big(n: int, m: int, seed: int = 0, abc=(0.57, 0.19, 0.19), device: int = 0,
                        buckets: int = 16, chunk: int = 1 << 28):
    """Same graph as rmat_csr_device for shapes beyond one device sort
    (torch.sort is limited to INT_MAX elements): candidates are partitioned
    by their low endpoint into `buckets` id ranges (a duplicate always lands
    in the same bucket), deduplicated per bucket keeping the first
    occurrence, the first m distinct edges by generation index are selected
    with an exact global threshold (binary search on the index, no global
    sort), and arcs are sorted per source-range bucket."""
    import torch

    lib = gdl.load()
    dev = torch.device("cuda", device)
    scale = max(1, int(math.ceil(math.log2(max(n, 2)))))
    st = torch.cuda.current_stream(dev).cuda_stream
    width = (n + buckets - 1) // buckets
    bk = [torch.empty(0, dtype=torch.int64, device=dev) for _ in range(buckets)]
    bi = [torch.empty(0, dtype=torch.int64, device=dev) for _ in range(buckets)]
    drawn = 0
    target = int(m * 1.25) + 1024

    def dedupe(b):
        sk, perm = torch.sort(bk[b], stable=True)
        head = torch.ones_like(sk, dtype=torch.bool)
        head[1:] = sk[1:] != sk[:-1]
        bk[b], bi[b] = sk[head], bi[b][perm][head]

    while True:
        while drawn < target:
            c = min(chunk, target - drawn)
            buf = torch.empty(c, dtype=torch.int64, device=dev)
            gdl.check(lib.gd_rmat_keys_device(scale, n, drawn, c, seed, abc[0], abc[1], abc[2],
                                              C.c_void_p(buf.data_ptr()), C.c_void_p(st)))
            ok = buf >= 0
            keys = buf[ok]
            idx = torch.arange(drawn, drawn + c, dtype=torch.int64, device=dev)[ok]
            del buf, ok
            part = torch.div(keys // n, width, rounding_mode="floor")
            for b in range(buckets):
                sel = part == b
                bk[b] = torch.cat([bk[b], keys[sel]])
                bi[b] = torch.cat([bi[b], idx[sel]])
            del keys, idx, part
            drawn += c
        for b in range(buckets):
            dedupe(b)
        if sum(int(x.numel()) for x in bk) >= m:
            break
        target = drawn + max(1 << 24, int(0.1 * m))
    # exact threshold T: #distinct edges whose first index < T equals m
    lo_t, hi_t = 0, drawn
    while lo_t < hi_t:
        mid = (lo_t + hi_t) // 2
        cnt = sum(int((x < mid).sum()) for x in bi)
        if cnt >= m:
            hi_t = mid
        else:
            lo_t = mid + 1
    T = lo_t
    sel_keys = []
    for b in range(buckets):
        sel_keys.append(bk[b][bi[b] < T])
        bk[b] = bi[b] = None
    torch.cuda.empty_cache()
    # arcs per source bucket: forward (lo -> hi) already bucketed by lo;
    # reverse (hi -> lo) re-bucketed by hi
    rev = [[] for _ in range(buckets)]
    for b in range(buckets):
        k = sel_keys[b]
        hi = k % n
        part = torch.div(hi, width, rounding_mode="floor")
        rk = hi * n + k // n
        for b2 in range(buckets):
            rev[b2].append(rk[part == b2])
        del hi, part, rk
    row = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    cols = []
    for b in range(buckets):
        arcs = torch.sort(torch.cat([sel_keys[b]] + rev[b])).values
        sel_keys[b] = None
        rev[b] = None
        src = arcs // n
        lo_id = b * width
        cnt = torch.bincount(src - lo_id, minlength=min(width, n - lo_id))
        row[lo_id + 1:lo_id + 1 + cnt.numel()] = cnt
        cols.append((arcs % n).to(torch.int32))
        del arcs, src
    col = torch.cat(cols)
    del cols
    row = torch.cumsum(row, 0)
    return row, col
