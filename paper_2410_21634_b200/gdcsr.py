"""GDCSR v1 files straight into (and out of) device graphs.

The reference's binary CSR cache (src/graph.py:298-321): the magic ``GDCSR``,
a version byte (1), little-endian int64 ``n`` and ``arcs``, then int64
``offsets[n+1]`` and int64 ``targets[arcs]``.  ``load_csr_cache`` reads both
arrays into host memory and runs ``CsrGraph.validate`` -- an interpreted
O(sum d) loop (src/graph.py:105-123) that dominates loading at the
products / papers100M shapes.

Here the file is memory-mapped, streamed to HBM in chunks through one pinned
staging buffer (targets narrowed to the device graph's int32 on the GPU), and
validated on the device with the reference's checks and error types:
offsets start at 0, nondecreasing and covering targets; targets in range,
no self loops, strictly ascending inside each row, every arc's reverse
present.  ``save_device_graph`` writes the same bytes ``save_csr_cache``
writes for the same graph.
"""

from __future__ import annotations

import struct

import numpy as np

from .graph import GraphFormatError, GraphStructureError, _MAGIC, _VERSION

__all__ = ["read_gdcsr_header", "load_device_graph", "save_device_graph"]

_HDR = len(_MAGIC) + 1 + 16
_CHUNK = 1 << 25  # int64 words per staging copy (256 MB)


def read_gdcsr_header(path) -> tuple[int, int]:
    """(n, arcs) of a GDCSR v1 file, with the reference's format errors."""
    with open(path, "rb") as fh:
        if fh.read(len(_MAGIC)) != _MAGIC:
            raise GraphFormatError("not a CSR cache file")
        (ver,) = struct.unpack("<B", fh.read(1))
        if ver != _VERSION:
            raise GraphFormatError(f"unsupported cache version {ver}")
        raw = fh.read(16)
        if len(raw) != 16:
            raise GraphFormatError("truncated CSR cache header")
        n, arcs = struct.unpack("<qq", raw)
        fh.seek(0, 2)
        size = fh.tell()
    if n < 0 or arcs < 0:
        raise GraphFormatError("negative sizes in CSR cache header")
    if size < _HDR + 8 * (n + 1 + arcs):
        raise GraphFormatError("truncated CSR cache file")
    return n, arcs


def _upload(mm: np.ndarray, out, dtype, torch, stage):
    """Copy a memory-mapped little-endian int64 array into ``out`` (a device
    tensor of ``dtype``) in staging-buffer chunks."""
    total = mm.shape[0]
    for a in range(0, total, _CHUNK):
        b = min(total, a + _CHUNK)
        h = stage[: b - a]
        h.numpy()[:] = mm[a:b]
        d = h.to(out.device, non_blocking=False)
        out[a:b] = d if dtype == torch.int64 else d.to(dtype)


def _validate_device(n: int, row_ptr, col, torch, chunk: int = 1 << 26) -> None:
    """The checks of CsrGraph.validate (src/graph.py:105-123) on the GPU, in
    row ranges of about `chunk` arcs so the temporaries stay O(chunk) (a few GB
    at most) whatever the graph size: self loops and strictly sorted rows per
    range, symmetry by a vectorised binary search of every arc's reverse in its
    target's (sorted) row."""
    arcs = col.numel()
    if int(row_ptr[0]) != 0:
        raise GraphStructureError("bad offsets array")
    if int(row_ptr[-1]) != arcs:
        raise GraphStructureError("offsets do not cover targets")
    deg = row_ptr[1:] - row_ptr[:-1]
    if n and bool((deg < 0).any()):
        raise GraphStructureError("offsets not nondecreasing")
    if arcs == 0:
        return
    if int(col.min()) < 0 or int(col.max()) >= n:
        raise GraphStructureError("target id out of range")
    dmax = int(deg.max())
    steps = max(1, dmax.bit_length())
    r0 = 0
    while r0 < n:
        # rows [r0, r1) holding at most `chunk` arcs (at least one row)
        lim = int(row_ptr[r0]) + chunk
        r1 = int(torch.searchsorted(row_ptr, torch.tensor([lim], device=row_ptr.device),
                                    right=True)[0]) - 1
        r1 = min(n, max(r0 + 1, r1))
        a0, a1 = int(row_ptr[r0]), int(row_ptr[r1])
        if a1 > a0:
            src = torch.repeat_interleave(
                torch.arange(r0, r1, device=col.device, dtype=torch.int64), deg[r0:r1])
            t = col[a0:a1].to(torch.int64)
            if bool((src == t).any()):
                raise GraphStructureError("self-loop present")
            same = src[1:] == src[:-1]
            if bool((same & (t[1:] <= t[:-1])).any()):
                raise GraphStructureError("row targets not strictly sorted")
            # reverse arc (t -> src): binary search for src in row t
            lo, hi = row_ptr[t], row_ptr[t + 1]
            end = hi.clone()
            for _ in range(steps + 1):
                act = lo < hi
                mid = torch.where(act, (lo + hi) >> 1, lo)
                go = act & (col[mid.clamp(max=arcs - 1)].to(torch.int64) < src)
                lo = torch.where(go, mid + 1, lo)
                hi = torch.where(act & ~go, mid, hi)
            found = (lo < end) & (col[lo.clamp(max=arcs - 1)].to(torch.int64) == src)
            if not bool(found.all()):
                raise GraphStructureError("missing reverse arc")
            del src, t, lo, hi, end, mid, go, act, found
        r0 = r1


def load_device_graph(path, device: int = 0, validate: bool = True):
    """A DeviceGraph from a GDCSR v1 file (the reference's load_csr_cache,
    src/graph.py:308-321), without building the host CsrGraph."""
    import torch

    from .device import DeviceGraph

    n, arcs = read_gdcsr_header(path)
    if n >= 2**31 - 1:
        raise GraphStructureError("node ids must fit int32 on the device")
    mm = np.memmap(path, dtype="<i8", mode="r", offset=_HDR, shape=(n + 1 + arcs,))
    dev = torch.device("cuda", device)
    stage = torch.empty(min(_CHUNK, n + 1 + arcs), dtype=torch.int64, pin_memory=True)
    row_ptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    col = torch.empty(arcs, dtype=torch.int32, device=dev)
    _upload(mm[: n + 1], row_ptr, torch.int64, torch, stage)
    if arcs:
        t64 = mm[n + 1:]
        # the int64 range is checked per chunk before narrowing to int32
        lo_hi = []
        for a in range(0, arcs, _CHUNK):
            b = min(arcs, a + _CHUNK)
            h = stage[: b - a]
            h.numpy()[:] = t64[a:b]
            d = h.to(dev)
            lo_hi.append(torch.stack([d.min(), d.max()]))
            col[a:b] = d.to(torch.int32)
        mm_all = torch.stack(lo_hi)
        if validate and (int(mm_all[:, 0].min()) < 0 or int(mm_all[:, 1].max()) >= n):
            raise GraphStructureError("target id out of range")
    del mm
    if validate:
        _validate_device(n, row_ptr, col, torch)
    dg = DeviceGraph.from_device(n, row_ptr, col, device)
    torch.cuda.synchronize(dev)
    return dg


def save_device_graph(dg, path) -> None:
    """Write a DeviceGraph as GDCSR v1: the bytes save_csr_cache
    (src/graph.py:298-305) writes for the same graph."""
    g = dg.to_host()
    with open(path, "wb") as fh:
        fh.write(_MAGIC + struct.pack("<B", _VERSION) + struct.pack("<qq", g.n, g.targets.shape[0]))
        fh.write(np.asarray(g.offsets, dtype="<i8").tobytes())
        fh.write(np.asarray(g.targets, dtype="<i8").tobytes())
