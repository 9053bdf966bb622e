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

__all__ = ["rmat_csr_device", "rmat_csr_device_big", "rmat_keys_torch", "RMAT_SHAPES"]


def _s64(c: int) -> int:
    """A uint64 constant as the int64 with the same bits."""
    return c - (1 << 64) if c >= 1 << 63 else c


def _srl(z, s: int):
    """Logical right shift of int64 tensors holding uint64 bits."""
    return (z >> s) & ((1 << (64 - s)) - 1)


def _splitmix64_t(z):
    z = z + _s64(0x9E3779B97F4A7C15)
    z = (z ^ _srl(z, 30)) * _s64(0xBF58476D1CE4E5B9)
    z = (z ^ _srl(z, 27)) * _s64(0x94D049BB133111EB)
    return z ^ _srl(z, 31)


def rmat_keys_torch(scale: int, n: int, first: int, count: int, seed: int, abc, dev,
                    chunk: int = 1 << 24):
    """The candidate keys of gd_rmat_keys_device (csrc/generate.cu) with torch
    tensor ops only: no libgdiff.  Same counter-based stream as
    synth.rmat_edges + permute_ids (int64 arithmetic wraps like uint64);
    used by bench.py's reference arm so that arm never loads the product
    library.  Returns int64 keys min*n+max, -1 for dropped candidates."""
    import torch

    ta = int(round(abc[0] * 65536))
    tb = ta + int(round(abc[1] * 65536))
    tc = tb + int(round(abc[2] * 65536))
    base = _s64((seed * 0x632BE59BD9B4E019) & 0xFFFFFFFFFFFFFFFF)
    z = (seed ^ 0x5EED) + 0x9E3779B97F4A7C15 & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    pkey = z ^ (z >> 31)
    mask = (1 << scale) - 1
    sh = max(1, scale // 2)
    nchunks = (scale + 3) // 4
    out = torch.empty(count, dtype=torch.int64, device=dev)
    for c0 in range(0, count, chunk):
        e = torch.arange(first + c0, first + min(count, c0 + chunk), dtype=torch.int64, device=dev)
        u = torch.zeros_like(e)
        v = torch.zeros_like(e)
        for k in range(nchunks):
            h = _splitmix64_t(base ^ (e * nchunks + k))
            for q in range(4):
                lvl = 4 * k + q
                if lvl >= scale:
                    break
                f = (h >> (16 * q)) & 0xFFFF
                bit = scale - 1 - lvl
                u |= (f >= tb).to(torch.int64) << bit
                v |= (((f >= ta) & (f < tb)) | (f >= tc)).to(torch.int64) << bit
        for rnd in range(3):
            mult = ((pkey >> (rnd * 16)) & 0xFFFF) * 2 + 0x9E37 * 2 + 1
            u = (u * mult) & mask
            u = u ^ (u >> sh)
            v = (v * mult) & mask
            v = v ^ (v >> sh)
        ok = (u < n) & (v < n) & (u != v)
        key = torch.minimum(u, v) * n + torch.maximum(u, v)
        out[c0:c0 + e.numel()] = torch.where(ok, key, torch.full_like(key, -1))
    return out


def _keys(native: bool, scale, n, first, count, seed, abc, dev):
    import torch

    if not native:
        return rmat_keys_torch(scale, n, first, count, seed, abc, dev)
    lib = gdl.load()
    st = torch.cuda.current_stream(dev).cuda_stream
    buf = torch.empty(count, dtype=torch.int64, device=dev)
    gdl.check(lib.gd_rmat_keys_device(scale, n, first, count, seed, abc[0], abc[1], abc[2],
                                      C.c_void_p(buf.data_ptr()), C.c_void_p(st)))
    return buf


def rmat_csr_device(n: int, m: int, seed: int = 0, abc=(0.57, 0.19, 0.19), device: int = 0,
                    native: bool = True):
    """Return (row_ptr int64[n+1], col int32[2m]) as CUDA tensors.  native=False
    draws the candidates with torch ops instead of the library kernel (the
    same graph)."""
    import torch

    dev = torch.device("cuda", device) if torch.cuda.is_available() else torch.device("cpu")
    scale = max(1, int(math.ceil(math.log2(max(n, 2)))))
    chunk = max(1024, int(m * 1.25) + 1024)
    keys = torch.empty(0, dtype=torch.int64, device=dev)
    first = torch.empty(0, dtype=torch.int64, device=dev)
    drawn = 0
    while True:
        buf = _keys(native, scale, n, drawn, chunk, seed, abc, dev)
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
                        buckets: int = 16, chunk: int = 1 << 28, native: bool = True):
    """Same graph as rmat_csr_device for shapes beyond one device sort
    (torch.sort is limited to INT_MAX elements): candidates are partitioned
    by their low endpoint into `buckets` id ranges (a duplicate always lands
    in the same bucket), deduplicated per bucket keeping the first
    occurrence, the first m distinct edges by generation index are selected
    with an exact global threshold (binary search on the index, no global
    sort), and arcs are sorted per source-range bucket."""
    import torch

    dev = torch.device("cuda", device)
    scale = max(1, int(math.ceil(math.log2(max(n, 2)))))
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
            buf = _keys(native, scale, n, drawn, c, seed, abc, dev)
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
