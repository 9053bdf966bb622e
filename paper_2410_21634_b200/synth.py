"""Seeded graph generators.

Small fixtures (path / complete / star / Erdos-Renyi / preferential
attachment) reproduce the reference generators (src/synth.py:18-79) draw for
draw, so a seed names the same graph on both sides.

``rmat_edges`` is the benchmark generator for the configs' OGB shapes.  Its
random stream is a counter-based integer hash (splitmix64 of
(seed, edge index, level chunk)), so the host version here and the device
version (``gd_rmat_edges`` in csrc/generate.cu) emit the same candidate edge
list bit for bit; ``rmat_graph`` then keeps the first ``m`` distinct
undirected edges in generation order and builds canonical CSR.  Graph
identity between the CPU oracle and the device run is therefore by
construction, and is additionally checked by hashing offsets/targets.
"""

from __future__ import annotations

import numpy as np

from .graph import CsrGraph, csr_from_pairs, from_edges

__all__ = [
    "path_graph", "complete_graph", "star_graph", "erdos_renyi",
    "preferential_attachment", "rmat_edges", "rmat_graph", "rmat_edge_order", "RMAT_SHAPES",
    "splitmix64", "permute_ids", "csr_hash",
]

# (n, undirected edges) of the configs in BASELINE.json
RMAT_SHAPES = {
    "cora": (2_708, 5_278),
    "arxiv": (169_343, 1_166_243),
    "products": (2_385_902, 61_859_140),
    "papers100M": (111_059_433, 1_615_685_872),
}

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def path_graph(n: int) -> CsrGraph:
    return from_edges(n, [(i, i + 1) for i in range(n - 1)])


def complete_graph(n: int) -> CsrGraph:
    return from_edges(n, [(i, j) for i in range(n) for j in range(i + 1, n)])


def star_graph(n: int) -> CsrGraph:
    return from_edges(n, [(0, i) for i in range(1, n)])


def erdos_renyi(n: int, p: float, seed: int, ensure_connected_source: int | None = 0) -> CsrGraph:
    """G(n, p); same random draws as the reference generator."""
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n, k=1)
    keep = rng.random(iu.shape[0]) < p
    a, b = iu[keep], ju[keep]
    pairs = np.stack([a, b], axis=1).astype(np.int64)
    s = ensure_connected_source
    if s is not None and not np.any((a == s) | (b == s)):
        t = int(rng.integers(0, n - 1))
        t = t + 1 if t >= s else t
        pairs = np.concatenate([pairs, np.array([[min(s, t), max(s, t)]], dtype=np.int64)])
    return csr_from_pairs(n, pairs)


def preferential_attachment(n: int, m_per_node: int, seed: int) -> CsrGraph:
    """Degree-proportional attachment; same draws as the reference generator."""
    if n <= m_per_node:
        raise ValueError("need n > m_per_node")
    rng = np.random.default_rng(seed)
    pool = np.empty(2 * n * m_per_node, dtype=np.int64)
    plen = 0
    edges = []
    for v in range(m_per_node):
        edges.append((v, m_per_node))
        pool[plen], pool[plen + 1] = v, m_per_node
        plen += 2
    for v in range(m_per_node + 1, n):
        chosen: set[int] = set()
        while len(chosen) < m_per_node:
            chosen.add(int(pool[rng.integers(0, plen)]))
        for u in chosen:
            edges.append((u, v))
            pool[plen], pool[plen + 1] = u, v
            plen += 2
    return from_edges(n, edges)


# --------------------------------------------------------------------------
# counter-based R-MAT (identical on host and device)
# --------------------------------------------------------------------------

def splitmix64(x: np.ndarray) -> np.ndarray:
    z = (x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)) & _M64
    with np.errstate(over="ignore"):
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
    return z ^ (z >> np.uint64(31))


def permute_ids(x: np.ndarray, scale: int, seed: int) -> np.ndarray:
    """Bijection on [0, 2^scale): three rounds of odd-multiply + xorshift."""
    mask = np.uint64((1 << scale) - 1)
    z = x.astype(np.uint64)
    key = int(splitmix64(np.array([seed ^ 0x5EED], dtype=np.uint64))[0])
    sh = np.uint64(max(1, scale // 2))
    with np.errstate(over="ignore"):
        for rnd in range(3):
            mult = np.uint64(((key >> (rnd * 16)) & 0xFFFF) * 2 + 0x9E37 * 2 + 1)
            z = (z * mult) & mask
            z = z ^ (z >> sh)
    return z


def _thresholds(a: float, b: float, c: float) -> tuple[int, int, int]:
    ta = int(round(a * 65536))
    tb = ta + int(round(b * 65536))
    tc = tb + int(round(c * 65536))
    return ta, tb, tc


def rmat_edges(scale: int, first: int, count: int, seed: int,
               abc: tuple[float, float, float] = (0.57, 0.19, 0.19)) -> np.ndarray:
    """Candidate edges [first, first+count) as int64 (count, 2), ids < 2^scale,
    before id permutation.  Each 64-bit hash drives four levels (16 bits each)."""
    ta, tb, tc = (np.uint64(t) for t in _thresholds(*abc))
    e = np.arange(first, first + count, dtype=np.uint64)
    u = np.zeros(count, dtype=np.uint64)
    v = np.zeros(count, dtype=np.uint64)
    nchunks = (scale + 3) // 4
    base = np.uint64((seed * 0x632BE59BD9B4E019) & 0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        for k in range(nchunks):
            h = splitmix64((base ^ (e * np.uint64(nchunks) + np.uint64(k))) & _M64)
            for q in range(4):
                lvl = 4 * k + q
                if lvl >= scale:
                    break
                f = (h >> np.uint64(16 * q)) & np.uint64(0xFFFF)
                bit = np.uint64(scale - 1 - lvl)
                ub = (f >= tb).astype(np.uint64)             # quadrants c, d
                vb = (((f >= ta) & (f < tb)) | (f >= tc)).astype(np.uint64)  # b, d
                u |= ub << bit
                v |= vb << bit
    return np.stack([u.astype(np.int64), v.astype(np.int64)], axis=1)


def rmat_graph(n: int, m: int, seed: int = 0, abc=(0.57, 0.19, 0.19),
               chunk: int | None = None) -> CsrGraph:
    """R-MAT graph with exactly ``m`` undirected edges on ``n`` nodes (host).

    Scale = ceil(log2 n); ids are permuted, ids >= n and self loops dropped,
    and candidates are drawn in chunks until m distinct edges exist; the
    first m distinct edges (by first appearance) are kept.
    """
    sel = rmat_edge_order(n, m, seed, abc, chunk)
    pairs = np.stack([sel // n, sel % n], axis=1)
    return csr_from_pairs(n, pairs)


def rmat_edge_order(n: int, m: int, seed: int = 0, abc=(0.57, 0.19, 0.19),
                    chunk: int | None = None) -> np.ndarray:
    """The m edges of rmat_graph as undirected keys min*n+max in generation
    (first appearance) order -- the order config 5 splits into snapshots."""
    scale = max(1, int(np.ceil(np.log2(max(n, 2)))))
    chunk = chunk or max(1024, int(m * 1.25) + 1024)
    keys = np.empty(0, dtype=np.int64)
    first = np.empty(0, dtype=np.int64)
    drawn = 0
    while True:
        cand = rmat_edges(scale, drawn, chunk, seed, abc)
        a = permute_ids(cand[:, 0], scale, seed).astype(np.int64)
        b = permute_ids(cand[:, 1], scale, seed).astype(np.int64)
        idx = np.arange(drawn, drawn + chunk, dtype=np.int64)
        ok = (a < n) & (b < n) & (a != b)
        k = np.minimum(a[ok], b[ok]) * n + np.maximum(a[ok], b[ok])
        keys = np.concatenate([keys, k])
        first = np.concatenate([first, idx[ok]])
        drawn += chunk
        uk, pos = np.unique(keys, return_index=True)
        if uk.shape[0] >= m:
            return uk[np.argsort(first[pos], kind="stable")[:m]]
        keys, first = uk, first[pos]


def csr_hash(g) -> str:
    """Short content hash of (n, offsets, targets) for identity checks."""
    import hashlib

    h = hashlib.sha256()
    h.update(np.int64(g.n).tobytes())
    h.update(np.ascontiguousarray(g.offsets, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(g.targets, dtype=np.int64).tobytes())
    return h.hexdigest()[:16]
