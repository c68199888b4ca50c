"""CPU oracle for the DRGraph layout path -- TEST INFRASTRUCTURE, NOT THE PRODUCT.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline /
``--impl reference`` leg may import this module.  The GPU product
(``paper_2008_07799_b200``) never routes through it.

Every function restates one function of the reference package ``drgraph``
(``/root/reference/pkg/src/drgraph``) and cites the ``file:line`` it follows.
The heavy loops (BFS, perplexity bisection, coarsening, the splitmix64 SGD
step loop, Vose) live in ``oracle.c`` (built by ``make -C oracle`` into
``oracle/_build/liboracle.so``); the numpy glue reproduces the reference's
array arithmetic.  The restatement is pinned by ``tests/test_oracle_golden.py``
against vectors the reference itself produced (``tests/golden/``).

The node-parallel (expected-gradient) iteration, the level aggregation, the KL
evaluator and the neighbour cap are NOT in the reference; they are restated from
SURVEY.md §8(a) A12 / §8(c) and built only from pinned pieces.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

# seed tags, optimizer.py:26-29
HIERARCHY_TAG = 1
INIT_TAG = 2
JITTER_TAG = 3
EPOCH_TAG = 4


def build() -> str:
    """Compile oracle.c (gcc) into oracle/_build/liboracle.so."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or (
                os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "oracle.c"))):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64, i32, f64, u64 = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_uint64
        L.orc_khop_count.argtypes = [P, P, i64, i32, i64, P, i32]
        L.orc_khop_fill.argtypes = [P, P, i64, i32, i64, P, P, P, i32]
        L.orc_sigma_rows.argtypes = [P, i64, i32, f64, f64, i32, f64, f64, P, P, i32]
        L.orc_search_sigma.argtypes = [P, P, i32, i64, f64, f64, i32, f64, f64]
        L.orc_search_sigma.restype = f64
        L.orc_fsum.argtypes = [P, i64]
        L.orc_fsum.restype = f64
        L.orc_coarsen_with_order.argtypes = [P, P, i64, P, P]
        L.orc_coarsen_with_order.restype = i64
        L.orc_build_alias.argtypes = [P, i64, f64, P, P]
        L.orc_sgd_steps.argtypes = [P, P, i64, P, P, i64, P, i32, i64, i32, i32,
                                    f64, f64, f64, f64, u64]
        L.orc_sgd_steps.restype = i64
        L.orc_sgd_epoch_threads.argtypes = [P, P, i64, P, P, i64, P, i32, P, P, i32, i32,
                                            i32, f64, f64, f64, f64]
        L.orc_sgd_epoch_threads.restype = i64
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _threads(threads: int | None) -> int:
    return threads if threads else (os.cpu_count() or 1)


# --------------------------------------------------------------------------
# Graph (graph.py:27-125)
# --------------------------------------------------------------------------

@dataclass(frozen=True, eq=False)
class Graph:
    """CSR graph, graph.py:27-77."""
    indptr: np.ndarray   # int64 [n+1]
    indices: np.ndarray  # int32 [2E]

    @property
    def node_count(self) -> int:
        return len(self.indptr) - 1

    @property
    def edge_count(self) -> int:
        return len(self.indices) // 2

    @property
    def degrees(self) -> np.ndarray:
        return np.diff(self.indptr)

    def edge_array(self) -> np.ndarray:
        u = np.repeat(np.arange(self.node_count, dtype=np.int32), self.degrees)
        keep = u < self.indices
        return np.column_stack([u[keep], self.indices[keep]])


def from_edges(pairs, node_count: int | None = None) -> Graph:
    """graph.py:80-125 (without sparse-id remapping)."""
    pairs = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    if node_count is None:
        node_count = int(pairs.max()) + 1 if pairs.size else 0
    pairs = pairs[pairs[:, 0] != pairs[:, 1]]
    if pairs.size:
        lo = np.minimum(pairs[:, 0], pairs[:, 1])
        hi = np.maximum(pairs[:, 0], pairs[:, 1])
        keys = np.unique(lo * np.int64(node_count) + hi)
        lo = keys // node_count
        hi = keys % node_count
        src = np.concatenate([lo, hi])
        dst = np.concatenate([hi, lo])
    else:
        src = np.empty(0, dtype=np.int64)
        dst = np.empty(0, dtype=np.int64)
    order = np.lexsort((dst, src))
    src = src[order]
    dst = dst[order]
    indptr = np.zeros(node_count + 1, dtype=np.int64)
    np.add.at(indptr, src + 1, 1)
    np.cumsum(indptr, out=indptr)
    return Graph(indptr=indptr, indices=dst.astype(np.int32))


# ---------------------------------------------------------------------------
# Text parsers (graph.py:128-243), restated for the parse parity tests
# ---------------------------------------------------------------------------

class OracleParseError(ValueError):
    """graph.py:17-24: message prefixed with 'line N: ' when the line is known."""

    def __init__(self, message, line=None):
        self.line = line
        super().__init__(message if line is None else f"line {line}: {message}")


def _source_lines(source):
    """graph.py:128-131: a str splits by str.splitlines, anything else iterates."""
    return source.splitlines() if isinstance(source, str) else list(source)


def _as_int(tok):
    try:
        return int(tok)
    except ValueError:
        return None


def remap_node_count(pairs):
    """Node count and (possibly compacted) pairs of from_edges(remap_sparse_ids=True)
    (graph.py:90-103)."""
    if pairs.size == 0:
        return 0, pairs
    ids = np.unique(pairs)
    if ids[-1] > 2 * len(ids):
        if ids[-1] == np.iinfo(np.int64).max:   # numpy cannot size the lookup table
            raise ValueError("Maximum allowed dimension exceeded")
        return len(ids), np.searchsorted(ids, pairs)
    return int(ids[-1]) + 1, pairs


def parse_edge_list(source) -> Graph:
    """graph.py:134-167."""
    ids = []
    for k, raw in enumerate(_source_lines(source)):
        body = raw.strip()
        if body == "" or body[0] == "#" or body[0] == "%":
            continue
        toks = body.split()
        if len(toks) != 2:
            raise OracleParseError(f"expected two ids, got {len(toks)} tokens", k + 1)
        a, b = _as_int(toks[0]), _as_int(toks[1])
        if a is None or b is None:
            raise OracleParseError(f"malformed integer in {toks!r}", k + 1)
        if min(a, b) < 0:
            raise OracleParseError(f"negative node id in {toks!r}", k + 1)
        ids += (a, b)
    if not ids:
        return Graph(np.zeros(1, dtype=np.int64), np.empty(0, dtype=np.int32))
    pairs = np.array(ids, dtype=np.int64).reshape(-1, 2)
    n, pairs = remap_node_count(pairs)
    return from_edges(pairs, n)


def parse_matrix_market(source) -> Graph:
    """graph.py:170-243."""
    lines = _source_lines(source)
    if not lines:
        raise OracleParseError("empty file, missing MatrixMarket header")
    head = lines[0].strip().split()
    if len(head) < 5 or head[0] != "%%MatrixMarket":
        raise OracleParseError("missing '%%MatrixMarket' header", 1)
    obj, fmt, fld, sym = (t.lower() for t in head[1:5])
    if (obj, fmt) != ("matrix", "coordinate"):
        raise OracleParseError(f"unsupported MatrixMarket type '{obj} {fmt}'"
                               " (need 'matrix coordinate')", 1)
    if fld not in ("pattern", "real", "integer", "complex"):
        raise OracleParseError(f"unsupported field '{fld}'", 1)
    if sym not in ("general", "symmetric", "skew-symmetric", "hermitian"):
        raise OracleParseError(f"unsupported symmetry '{sym}'", 1)
    k, size = 1, None
    while k < len(lines):
        body = lines[k].strip()
        k += 1
        if body == "" or body.startswith("%"):
            continue
        parts = body.split()
        if len(parts) != 3:
            raise OracleParseError("size line must be 'rows cols nnz'", k)
        size = [_as_int(p) for p in parts]
        if None in size:
            raise OracleParseError(f"malformed size line {body!r}", k)
        break
    if size is None:
        raise OracleParseError("missing size line")
    rows, cols, declared = size
    if rows != cols:
        raise OracleParseError(f"adjacency matrix must be square, got {rows}x{cols}", k)
    if rows < 0 or declared < 0:
        raise OracleParseError("negative dimension in size line", k)
    ids = []
    for j in range(k, len(lines)):
        body = lines[j].strip()
        if body == "" or body.startswith("%"):
            continue
        if len(ids) // 2 >= declared:
            raise OracleParseError(f"more than the declared {declared} entries", j + 1)
        parts = body.split()
        if len(parts) < 2:
            raise OracleParseError("coordinate entry needs at least 'i j'", j + 1)
        a, b = _as_int(parts[0]), _as_int(parts[1])
        if a is None or b is None:
            raise OracleParseError(f"malformed coordinate entry {body!r}", j + 1)
        if not (1 <= a <= rows and 1 <= b <= cols):
            raise OracleParseError(f"index ({a}, {b}) outside declared {rows}x{cols}", j + 1)
        ids += (a - 1, b - 1)
    if len(ids) // 2 != declared:
        raise OracleParseError(f"declared {declared} entries but found {len(ids) // 2}")
    return from_edges(np.array(ids, dtype=np.int64).reshape(-1, 2), rows)


# ---------------------------------------------------------------------------
# Output formats (output.py:12-108, graph.py:246-250), restated for the tests
# ---------------------------------------------------------------------------

def write_coords(positions) -> str:
    """output.py:12-17."""
    pos = np.asarray(positions, dtype=np.float64).reshape(-1, 2)
    return "".join([f"#nodes {len(pos)}\n"] + [f"{x:.6f} {y:.6f}\n" for x, y in pos])


def format_edge_list(g: Graph) -> str:
    """graph.py:246-250 (edges u < v in CSR order)."""
    src = np.repeat(np.arange(g.node_count), np.diff(g.indptr))
    keep = src < g.indices
    return "".join(f"{u} {v}\n" for u, v in zip(src[keep].tolist(), g.indices[keep].tolist()))


def _svg_color(t: float) -> str:
    """_edge_color (output.py:44-51)."""
    if t <= 0.5:
        u = 2.0 * t
        rgb = (1.0 - u, u, 0.0)
    else:
        u = 2.0 * t - 1.0
        rgb = (0.0, 1.0 - u, u)
    return "#" + "".join(f"{int(round(255 * c)):02x}" for c in rgb)


def write_svg(g: Graph, positions, canvas=1000, margin=20.0, node_radius=2.0, edge_width=1.0,
              edge_cap=600_000, seed=0) -> str:
    """output.py:56-108."""
    pos = np.asarray(positions, dtype=np.float64).reshape(-1, 2)
    size = float(canvas)
    inner = size - 2.0 * margin
    xs = ys = np.empty(0)
    if len(pos):
        lo = pos.min(axis=0)
        spans = pos.max(axis=0) - lo
        span = float(spans.max())
        scale = inner / span if span > 0 else 0.0
        off = margin + (inner - spans * scale) / 2.0
        xs = off[0] + (pos[:, 0] - lo[0]) * scale
        ys = size - (off[1] + (pos[:, 1] - lo[1]) * scale)
    src = np.repeat(np.arange(g.node_count), np.diff(g.indptr))
    keep = src < g.indices
    edges = np.column_stack([src[keep], g.indices[keep]])
    if len(edges) > edge_cap:
        pick = np.sort(np.random.default_rng(seed).choice(len(edges), size=edge_cap,
                                                          replace=False))
        edges = edges[pick]
    out = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{canvas}" height="{canvas}" '
           f'viewBox="0 0 {canvas} {canvas}">', f'<rect width="{canvas}" height="{canvas}" fill="white"/>']
    if len(edges):
        a, b = edges[:, 0], edges[:, 1]
        du, dv = xs[a] - xs[b], ys[a] - ys[b]
        ln = np.sqrt(du * du + dv * dv)
        lmin, lrange = float(ln.min()), float(ln.max()) - float(ln.min())
        for (u, v), L in zip(edges.tolist(), ln):
            t = (L - lmin) / lrange if lrange > 0 else 0.0
            out.append(f'<line x1="{xs[u]:.2f}" y1="{ys[u]:.2f}" x2="{xs[v]:.2f}" '
                       f'y2="{ys[v]:.2f}" stroke="{_svg_color(t)}" stroke-width="{edge_width}"/>')
    out += [f'<circle cx="{x:.2f}" cy="{y:.2f}" r="{node_radius}" fill="black"/>'
            for x, y in zip(xs, ys)]
    out.append("</svg>")
    return "\n".join(out) + "\n"


def connected_components(g: Graph) -> int:
    """Component count (graph.py:369-388), via scipy's C implementation."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components as cc
    n = g.node_count
    if n == 0:
        return 0
    m = csr_matrix((np.ones(len(g.indices)), g.indices, g.indptr), shape=(n, n))
    return int(cc(m, directed=False)[0])


# --------------------------------------------------------------------------
# k-hop neighbourhoods (graph.py:252-366)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class NeighborDistances:
    indptr: np.ndarray
    ids: np.ndarray
    dists: np.ndarray
    k: int

    @property
    def node_count(self) -> int:
        return len(self.indptr) - 1


def all_k_neighborhoods(g: Graph, k: int, cap: int = 0,
                        threads: int | None = None) -> NeighborDistances:
    """graph.py:308-366; k=1 copies the adjacency (graph.py:318-323).
    ``cap`` > 0: (dist,id)-sorted prefix of each row (BASELINE C3 extension)."""
    if k < 1:
        raise ValueError("k must be >= 1")
    n = g.node_count
    indptr = np.ascontiguousarray(g.indptr, dtype=np.int64)
    indices = np.ascontiguousarray(g.indices, dtype=np.int32)
    if k == 1 and cap <= 0:
        return NeighborDistances(indptr.copy(), indices.copy(),
                                 np.ones(len(indices), dtype=np.int32), 1)
    L = lib()
    counts = np.zeros(n, dtype=np.int64)
    L.orc_khop_count(_p(indptr), _p(indices), n, k, cap, _p(counts), _threads(threads))
    out_indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=out_indptr[1:])
    nnz = int(out_indptr[-1])
    ids = np.empty(nnz, dtype=np.int32)
    dists = np.empty(nnz, dtype=np.int32)
    L.orc_khop_fill(_p(indptr), _p(indices), n, k, cap, _p(out_indptr), _p(ids), _p(dists),
                    _threads(threads))
    return NeighborDistances(out_indptr, ids, dists, k)


def bfs_k_neighborhood(g: Graph, source: int, k: int) -> list[tuple[int, int]]:
    """graph.py:280-305 (pure Python, for tiny cases)."""
    from collections import deque
    dist = {source: 0}
    q = deque([source])
    out = []
    while q:
        v = q.popleft()
        d = dist[v]
        if d == k:
            break
        for u in g.indices[g.indptr[v]:g.indptr[v + 1]]:
            u = int(u)
            if u not in dist:
                dist[u] = d + 1
                out.append((u, d + 1))
                q.append(u)
    out.sort(key=lambda e: (e[1], e[0]))
    return out


# --------------------------------------------------------------------------
# Similarity (similarity.py:56-278)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class SparseSimilarity:
    indptr: np.ndarray
    targets: np.ndarray
    weights: np.ndarray
    total_mass: float
    sigma: np.ndarray
    k: int

    @property
    def node_count(self) -> int:
        return len(self.indptr) - 1

    @property
    def entry_count(self) -> int:
        return len(self.targets)

    def sources(self) -> np.ndarray:
        return np.repeat(np.arange(self.node_count, dtype=np.int32), np.diff(self.indptr))

    def row_masses(self) -> np.ndarray:
        """similarity.py:84-91."""
        if self.node_count == 0 or len(self.weights) == 0:
            return np.zeros(self.node_count, dtype=np.float64)
        return np.add.reduceat(np.append(self.weights, 0.0),
                               self.indptr[:-1]) * (np.diff(self.indptr) > 0)


def row_histograms(nd: NeighborDistances) -> np.ndarray:
    """Per-row count of entries at each hop distance 1..k (rows are sorted by
    distance, graph.py:262-263)."""
    n = nd.node_count
    k = nd.k
    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(nd.indptr))
    hist = np.zeros(n * k, dtype=np.int64)
    np.add.at(hist, src * k + (nd.dists.astype(np.int64) - 1), 1)
    return hist.reshape(n, k)


def search_sigma(counts, dvals, n_row, target, tol=1e-5, max_iter=64,
                 sigma_min=1e-5, sigma_max=1e5) -> float:
    """similarity.py:167-199 over a row's distance histogram."""
    counts = np.ascontiguousarray(counts, dtype=np.int64)
    dvals = np.ascontiguousarray(dvals, dtype=np.float64)
    return float(lib().orc_search_sigma(_p(counts), _p(dvals), len(counts), int(n_row),
                                        float(target), tol, max_iter, sigma_min, sigma_max))


def conditional_table(nd: NeighborDistances, perplexity="auto", tol=1e-5, max_iter=64,
                      sigma_min=1e-5, sigma_max=1e5, threads=None):
    """Per-node sigma and p_{j|i} per hop distance (similarity.py:246-262)."""
    n, k = nd.node_count, nd.k
    hist = np.ascontiguousarray(row_histograms(nd))
    sigma = np.ones(n, dtype=np.float64)
    pcond = np.zeros((n, k), dtype=np.float64)
    perp = -1.0 if perplexity == "auto" else float(perplexity)
    lib().orc_sigma_rows(_p(hist), n, k, perp, tol, max_iter, sigma_min, sigma_max,
                         _p(sigma), _p(pcond), _threads(threads))
    return sigma, pcond, hist


def build_sparse_similarity(nd: NeighborDistances, perplexity="auto", tol=1e-5,
                            max_iter=64, sigma_min=1e-5, sigma_max=1e5,
                            threads=None) -> SparseSimilarity:
    """similarity.py:216-278.  Rows must be mirror-complete (uncapped BFS);
    see ``build_capped_similarity`` for the union-symmetrised cap extension."""
    n = nd.node_count
    if len(nd.dists) == 0:
        return SparseSimilarity(nd.indptr.copy(), nd.ids.copy(), np.empty(0), 0.0,
                                np.ones(n), nd.k)
    counts = np.diff(nd.indptr)
    src = np.repeat(np.arange(n, dtype=np.int64), counts)
    n_ne = int((counts > 0).sum())
    if nd.k == 1 or int(nd.dists.max()) == 1:
        # closed form, similarity.py:202-213
        inv = np.zeros(n, dtype=np.float64)
        nz = counts > 0
        inv[nz] = 1.0 / counts[nz]
        weights = (inv[src] + inv[nd.ids]) / (2.0 * max(n_ne, 1))
        sigma = np.ones(n, dtype=np.float64)
    else:
        sigma, pcond, _ = conditional_table(nd, perplexity, tol, max_iter, sigma_min,
                                            sigma_max, threads)
        d = nd.dists.astype(np.int64) - 1
        cond = pcond[src, d]
        mirror = pcond[nd.ids.astype(np.int64), d]   # p_{i|j}: same hop distance
        weights = (cond + mirror) / (2.0 * n_ne)
    total = fsum(weights)
    return SparseSimilarity(nd.indptr.copy(), nd.ids.copy(), weights, total, sigma, nd.k)


def build_capped_similarity(nd_capped: NeighborDistances, perplexity="auto", tol=1e-5,
                            max_iter=64, sigma_min=1e-5, sigma_max=1e5,
                            threads=None) -> SparseSimilarity:
    """BASELINE C3 extension (not in the reference): conditional rows over the
    capped rows (the reference's per-row search, similarity.py:246-262), then
    union symmetrisation P_ij = (p_{j|i} + p_{i|j}) / (2 N_ne) with a missing
    mirror counting 0."""
    n = nd_capped.node_count
    if len(nd_capped.dists) == 0:
        return SparseSimilarity(nd_capped.indptr.copy(), nd_capped.ids.copy(), np.empty(0),
                                0.0, np.ones(n), nd_capped.k)
    counts = np.diff(nd_capped.indptr)
    src = np.repeat(np.arange(n, dtype=np.int64), counts)
    n_ne = int((counts > 0).sum())
    if nd_capped.k == 1 or int(nd_capped.dists.max()) == 1:
        inv = np.zeros(n)
        inv[counts > 0] = 1.0 / counts[counts > 0]
        cond = inv[src]
        sigma = np.ones(n)
    else:
        sigma, pcond, _ = conditional_table(nd_capped, perplexity, tol, max_iter, sigma_min,
                                            sigma_max, threads)
        cond = pcond[src, nd_capped.dists.astype(np.int64) - 1]
    dst = nd_capped.ids.astype(np.int64)
    keys = np.concatenate([src * n + dst, dst * n + src])
    vals = np.concatenate([cond, cond])
    # one or two contributions per key: their sum does not depend on their order
    # (IEEE addition commutes), so any sort will do
    order = np.argsort(keys)
    keys = keys[order]
    vals = vals[order]
    start = np.flatnonzero(np.concatenate([[True], keys[1:] != keys[:-1]]))
    uniq = keys[start]
    w = np.add.reduceat(vals, start) / (2.0 * n_ne)
    rows = uniq // n
    tgt = (uniq % n).astype(np.int32)
    indptr = np.zeros(n + 1, dtype=np.int64)
    indptr[1:] = np.cumsum(np.bincount(rows, minlength=n))
    total = fsum(w)
    return SparseSimilarity(indptr, tgt, w, total, sigma, nd_capped.k)


def fsum(x) -> float:
    """math.fsum of a float64 array (C restatement of CPython's algorithm)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    return float(lib().orc_fsum(_p(x), len(x)))


# --------------------------------------------------------------------------
# Hierarchy (multilevel.py:19-138)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class Hierarchy:
    levels: list
    maps: list
    rho: float
    min_size: int

    @property
    def depth(self) -> int:
        return len(self.levels) - 1


def coarsen_with_order(g: Graph, order: np.ndarray):
    """multilevel.py:48-79."""
    n = g.node_count
    indptr = np.ascontiguousarray(g.indptr, dtype=np.int64)
    indices = np.ascontiguousarray(g.indices, dtype=np.int32)
    order = np.ascontiguousarray(order, dtype=np.int64)
    parent = np.empty(n, dtype=np.int32)
    nc = int(lib().orc_coarsen_with_order(_p(indptr), _p(indices), n, _p(order), _p(parent)))
    edges = g.edge_array()
    if edges.size:
        cu = parent[edges[:, 0]]
        cv = parent[edges[:, 1]]
        keep = cu != cv
        ce = np.column_stack([cu[keep], cv[keep]])
    else:
        ce = np.empty((0, 2), dtype=np.int64)
    return from_edges(ce, node_count=nc), parent


def coarsen_once(g: Graph, seed: int):
    """multilevel.py:82-92."""
    order = np.random.default_rng(seed).permutation(g.node_count)
    return coarsen_with_order(g, order)


def build_hierarchy(g: Graph, rho=0.8, min_size=16, seed=0, max_levels: int | None = None,
                    force_levels: int | None = None) -> Hierarchy:
    """multilevel.py:95-113.  ``max_levels`` (total level count cap) and
    ``force_levels`` (skip the rho test until that many levels exist) are the
    BASELINE C2-C5 extensions (SURVEY §7 hard part 5)."""
    rng = np.random.default_rng(seed)
    levels = [g]
    maps = []
    while levels[-1].node_count > min_size:
        if max_levels is not None and len(levels) >= max_levels:
            break
        level_seed = int(rng.integers(0, 2**63 - 1))
        coarse, parent = coarsen_once(levels[-1], level_seed)
        forced = force_levels is not None and len(levels) < force_levels
        if not forced and coarse.node_count > rho * levels[-1].node_count:
            break
        if coarse.node_count == levels[-1].node_count:
            break
        levels.append(coarse)
        maps.append(parent)
    return Hierarchy(levels, maps, rho, min_size)


def compose_maps(h: Hierarchy, level: int) -> np.ndarray:
    """multilevel.py:116-123."""
    flat = np.arange(h.levels[0].node_count, dtype=np.int32)
    for m in h.maps[:level]:
        flat = m[flat]
    return flat


def prolong(coarse_positions, cmap, jitter_scale, seed):
    """multilevel.py:126-138."""
    fine = coarse_positions[cmap].astype(np.float64, copy=True)
    if jitter_scale > 0:
        rng = np.random.default_rng(seed)
        fine += rng.normal(0.0, jitter_scale, size=fine.shape)
    return fine


# --------------------------------------------------------------------------
# Samplers (optimizer.py:85-300)
# --------------------------------------------------------------------------

def derive_seed(seed: int, *tags: int) -> int:
    """optimizer.py:32-34."""
    return int(np.random.SeedSequence([seed, *tags]).generate_state(1, np.uint64)[0])


def build_alias_table(weights):
    """optimizer.py:111-139 (Vose, same stack order).  Returns (prob, alias)."""
    w = np.ascontiguousarray(weights, dtype=np.float64)
    if len(w) == 0:
        raise ValueError("cannot build an alias table over zero items")
    if w.min() < 0:
        raise ValueError("negative weight")
    total = float(w.sum())
    if total <= 0:
        raise ValueError("all weights are zero")
    prob = np.empty(len(w), dtype=np.float64)
    alias = np.empty(len(w), dtype=np.int32)
    lib().orc_build_alias(_p(w), len(w), total, _p(prob), _p(alias))
    return prob, alias


def negative_weights(row_mass: np.ndarray, power: float = 0.75) -> np.ndarray:
    """optimizer.py:243-259 (weights before the alias build)."""
    mass = row_mass
    with np.errstate(invalid="ignore"):
        w = np.where(mass > 0, mass, 0.0) ** power
    if power == 0:
        w = np.ones_like(mass)
    top = float(w.max()) if len(w) else 0.0
    if top <= 0.0:
        w = np.ones_like(mass)
        top = 1.0
    return np.where(w > 0, w, 1e-8 * top)


@dataclass
class Samplers:
    """optimizer.py:270-300."""
    pos_rec: np.ndarray
    pair_rec: np.ndarray
    neg_rec: np.ndarray
    _maps: dict = field(default_factory=dict)

    def level_map(self, h: Hierarchy, level: int) -> np.ndarray:
        if level not in self._maps:
            self._maps[level] = compose_maps(h, level)
        return self._maps[level]


def build_samplers(ns: SparseSimilarity, neg_power=0.75) -> Samplers:
    src = ns.sources()
    canon = src < ns.targets
    if ns.entry_count == 0 or float(ns.weights.sum()) <= 0.0:
        raise ValueError("similarity carries no mass; nothing to sample")
    pprob, palias = build_alias_table(ns.weights[canon])
    nprob, nalias = build_alias_table(negative_weights(ns.row_masses(), neg_power))
    pos_rec = np.empty((len(pprob), 2)); pos_rec[:, 0] = pprob; pos_rec[:, 1] = palias
    neg_rec = np.empty((len(nprob), 2)); neg_rec[:, 0] = nprob; neg_rec[:, 1] = nalias
    pair_rec = np.empty((len(pprob), 2), dtype=np.int32)
    pair_rec[:, 0] = src[canon]
    pair_rec[:, 1] = ns.targets[canon]
    return Samplers(pos_rec, pair_rec, neg_rec)


# --------------------------------------------------------------------------
# SGD (optimizer.py:142-203, _kernels.py:48-141, optimizer.py:310-413)
# --------------------------------------------------------------------------

@dataclass
class OptimizerParams:
    """optimizer.py:37-74 defaults, plus the BASELINE `init` extension."""
    neg_samples: int = 5
    gamma: float = 0.1
    gamma_coarsest: float = 0.01
    iters: int = 400
    b: int = 2
    lr0: float = 1.0
    grad_clip: float = 5.0
    eps: float = 1e-3
    neg_power: float = 0.75
    init_scale: float = 1e-4
    jitter_rel: float = 1e-3
    seed: int = 0
    threads: int = 1


def sgd_steps(pos, samplers: Samplers, node_map, mapped, n_steps, neg_count, b, gamma, eps,
              clip, lr, seed) -> int:
    """_kernels.py:48-141, bit-exact twin (fp64, splitmix64)."""
    assert pos.dtype == np.float64 and pos.flags.c_contiguous
    nm = np.ascontiguousarray(node_map, dtype=np.int32)
    return int(lib().orc_sgd_steps(
        _p(pos), _p(samplers.pos_rec), len(samplers.pos_rec), _p(samplers.pair_rec),
        _p(samplers.neg_rec), len(samplers.neg_rec), _p(nm), int(bool(mapped)), int(n_steps),
        int(neg_count), int(b), float(gamma), float(eps), float(clip), float(lr),
        ctypes.c_uint64(int(seed))))


def _infer_level(h: Hierarchy, n: int) -> int:
    for level, g in enumerate(h.levels):
        if g.node_count == n:
            return level
    raise ValueError(f"no hierarchy level has {n} nodes")


def sgd_epoch(positions, h: Hierarchy, samplers: Samplers, params: OptimizerParams, t: int,
              stats=None, level: int | None = None, threads: int | None = None):
    """optimizer.py:310-353 (threads > 1: Hogwild workers over the C step loop)."""
    n = len(positions)
    if level is None:
        level = _infer_level(h, n)
    gamma = params.gamma_coarsest if level == h.depth else params.gamma
    lr = max(params.lr0 * (1.0 - t / params.iters), 0.0)
    node_map = np.ascontiguousarray(samplers.level_map(h, level), dtype=np.int32)
    nthreads = threads if threads is not None else params.threads
    workers = min(nthreads, n) if nthreads > 1 else 1
    counts = np.array([n // workers + (1 if w < n % workers else 0) for w in range(workers)],
                      dtype=np.int64)
    seeds = np.array([derive_seed(params.seed, EPOCH_TAG, level, t, w) for w in range(workers)],
                     dtype=np.uint64)
    evals = int(lib().orc_sgd_epoch_threads(
        _p(positions), _p(samplers.pos_rec), len(samplers.pos_rec), _p(samplers.pair_rec),
        _p(samplers.neg_rec), len(samplers.neg_rec), _p(node_map), int(level > 0), _p(counts),
        _p(seeds), workers, params.neg_samples, params.b, gamma, params.eps, params.grad_clip,
        lr))
    if not np.isfinite(positions).all():
        raise FloatingPointError(f"non-finite coordinate after epoch {t} at level {level}")
    if stats is not None:
        stats["gradient_steps"] = stats.get("gradient_steps", 0) + n
        stats["distance_evals"] = stats.get("distance_evals", 0) + evals
    return positions


def layout_radius(positions) -> float:
    """optimizer.py:356-358."""
    center = positions.mean(axis=0)
    return float(np.sqrt(((positions - center) ** 2).sum(axis=1)).max())


def layout_graph(g: Graph, k=1, perplexity="auto", params: OptimizerParams | None = None,
                 rho=0.8, min_size=16, max_levels=None, force_levels=None, init=None,
                 neighbor_cap=0):
    """optimizer.py:361-413.  With the defaults and threads=1 it reproduces the
    reference bit for bit (pinned by tests/test_oracle_golden.py).  ``init``:
    optional (n_coarsest, 2) initial positions (BASELINE C1 uniform init)."""
    opt = params or OptimizerParams()
    nd = all_k_neighborhoods(g, k, cap=neighbor_cap)
    ns = (build_capped_similarity(nd, perplexity) if neighbor_cap > 0
          else build_sparse_similarity(nd, perplexity))
    h = build_hierarchy(g, rho=rho, min_size=min_size, seed=derive_seed(opt.seed, HIERARCHY_TAG),
                        max_levels=max_levels, force_levels=force_levels)
    stats = {"levels": [lv.node_count for lv in h.levels], "gradient_steps": 0,
             "distance_evals": 0}
    if init is None:
        rng = np.random.default_rng(derive_seed(opt.seed, INIT_TAG))
        positions = rng.normal(0.0, opt.init_scale, size=(h.levels[-1].node_count, 2))
    elif callable(init):   # init(n_coarsest) -> positions
        positions = np.array(init(h.levels[-1].node_count), dtype=np.float64)
    else:
        positions = np.array(init, dtype=np.float64)
    if ns.entry_count == 0:
        stats["skipped_optimization"] = True
        return prolong(positions, compose_maps(h, h.depth), 0.0, 0), stats, ns, h
    samplers = build_samplers(ns, opt.neg_power)
    for level in range(h.depth, -1, -1):
        for t in range(opt.iters):
            sgd_epoch(positions, h, samplers, opt, t, stats, level=level)
        if level > 0:
            radius = layout_radius(positions)
            jitter = opt.jitter_rel * radius if radius > 0 else opt.init_scale
            positions = prolong(positions, h.maps[level - 1], jitter,
                                derive_seed(opt.seed, JITTER_TAG, level))
    return positions, stats, ns, h


# --------------------------------------------------------------------------
# Node-parallel expected-gradient iteration -- the math the
# GPU kernel K7 implements, restated in fp64 from the reference's per-
# interaction gradients (optimizer.py:174-203) with the kernel's clip
# (_kernels.py:94-101, 126-135).
# --------------------------------------------------------------------------

def _ipow(x, n):
    r = np.ones_like(x)
    for _ in range(n):
        r = r * x
    return r


def clipped_attractive(d, b, clip):
    """Per-row attractive gradient wrt y_i of pairs with displacement d=(y_i-y_j),
    clipped per component (_kernels.py:88-101); zero at ld2 == 0."""
    ld2 = (d * d).sum(axis=1)
    pw = _ipow(ld2, b - 1)
    with np.errstate(divide="ignore", invalid="ignore"):
        coef = np.where(ld2 > 0, -2.0 * float(b) * pw / (1.0 + pw * ld2), 0.0)
    return np.clip(coef[:, None] * d, -clip, clip)


def clipped_repulsive(d, b, gamma, eps, clip):
    """optimizer.py:189-203 with the kernel's clip (_kernels.py:118-135)."""
    ld2 = (d * d).sum(axis=1)
    pw = _ipow(ld2, b - 1)
    with np.errstate(divide="ignore", invalid="ignore"):
        coef = np.where(ld2 + eps > 0, gamma * 2.0 * float(b) / ((ld2 + eps) * (1.0 + pw * ld2)),
                        0.0)
    return np.clip(coef[:, None] * d, -clip, clip)


def drawn_steps(pos, draws, lr, gamma, eps, clip, b):
    """The reference step loop (_kernels.py:82-140) on steps whose draws are given:
    draws[f, s] = source i (f = 0), target j (f = 1; j == i: collapsed pair, no
    attraction), negative m (f = 2 + m; -1 = every attempt hit i or j, skipped as
    at _kernels.py:118-119).  Sequential, fp64, updates ``pos`` in place."""
    bf = float(b)
    for s in range(draws.shape[1]):
        i, j = int(draws[0, s]), int(draws[1, s])
        if i != j:                                   # _kernels.py:82-105
            dx = pos[i, 0] - pos[j, 0]
            dy = pos[i, 1] - pos[j, 1]
            ld2 = dx * dx + dy * dy
            if ld2 > 0.0:
                pw = ld2 ** (b - 1)
                coef = -2.0 * bf * pw / (1.0 + pw * ld2)
                gx = min(max(coef * dx, -clip), clip)
                gy = min(max(coef * dy, -clip), clip)
                pos[i] += (lr * gx, lr * gy)
                pos[j] -= (lr * gx, lr * gy)
        for m in range(2, draws.shape[0]):           # _kernels.py:106-140
            t = int(draws[m, s])
            if t < 0:
                continue
            dx = pos[i, 0] - pos[t, 0]
            dy = pos[i, 1] - pos[t, 1]
            ld2 = dx * dx + dy * dy
            if ld2 + eps > 0.0:
                pw = ld2 ** (b - 1)
                coef = gamma * 2.0 * bf / ((ld2 + eps) * (1.0 + pw * ld2))
                gx = min(max(coef * dx, -clip), clip)
                gy = min(max(coef * dy, -clip), clip)
                pos[i] += (lr * gx, lr * gy)
                pos[t] -= (lr * gx, lr * gy)
    return pos


def deferred_drawn_epoch(pos, draws, lr, gamma, eps, clip, b, snap=None, fold=True,
                         defer=True):
    """The multi-GPU epoch of paper_2008_07799_b200/shard.py on given draws, as a
    sequential fp64 restatement: the reference step (_kernels.py:82-140) with the
    source and the attraction partner read and moved in place, each negative read
    from the epoch-start snapshot (plus this step's own earlier reactions on it) and
    its reaction deferred into a delta added at the epoch end.  ``snap``: an older
    snapshot to read the negatives from; ``fold=False`` returns (pos, delta)
    without adding the delta.  ``defer=False``: the 1-GPU snapshot form
    (DRG_SAMPLED_SNAPSHOT) -- the negatives are still read from the snapshot, but
    their reactions move ``pos`` at once, like every other update."""
    snap = pos.copy() if snap is None else snap
    delta = np.zeros_like(pos)
    bf = float(b)
    M = draws.shape[0] - 2
    for s in range(draws.shape[1]):
        i, j = int(draws[0, s]), int(draws[1, s])
        yi = pos[i].copy()
        gi = np.zeros(2)
        if i != j:
            dx, dy = yi[0] - pos[j, 0], yi[1] - pos[j, 1]
            ld2 = dx * dx + dy * dy
            if ld2 > 0.0:
                pw = ld2 ** (b - 1)
                coef = -2.0 * bf * pw / (1.0 + pw * ld2)
                g = np.array([min(max(coef * dx, -clip), clip),
                              min(max(coef * dy, -clip), clip)]) * lr
                pos[j] -= g
                yi += g
                gi += g
        own = {}
        for m in range(M):
            t = int(draws[2 + m, s])
            if t < 0:
                continue
            yc = snap[t] + own.get(t, 0.0)
            dx, dy = yi[0] - yc[0], yi[1] - yc[1]
            ld2 = dx * dx + dy * dy
            if ld2 + eps > 0.0:
                pw = ld2 ** (b - 1)
                coef = gamma * 2.0 * bf / ((ld2 + eps) * (1.0 + pw * ld2))
                g = np.array([min(max(coef * dx, -clip), clip),
                              min(max(coef * dy, -clip), clip)]) * lr
                if defer:
                    delta[t] -= g
                else:
                    pos[t] -= g
                own[t] = own.get(t, 0.0) - g
                yi += g
                gi += g
        pos[i] += gi
    if not fold:
        return pos, delta
    pos += delta
    return pos


def periodic_drawn_epochs(pos, draws_per_epoch, lrs, gamma, eps, clip, b, every):
    """drg_shard_run with exchange_every = r: the negatives read the snapshot taken at
    the last exchange, their reactions accumulate until it; exchanges after every r-th
    epoch and after the last."""
    pos = np.array(pos, dtype=np.float64)
    snap = pos.copy()
    delta = np.zeros_like(pos)
    n = len(draws_per_epoch)
    for j in range(n):
        pos, d = deferred_drawn_epoch(pos, draws_per_epoch[j], lrs[j], gamma, eps, clip, b,
                                      snap=snap, fold=False)
        delta += d
        if (j + 1) % every == 0 or j + 1 == n:
            pos += delta
            delta[:] = 0.0
            snap = pos.copy()
    return pos


def lagged_drawn_epochs(pos, draws_per_epoch, lrs, gamma, eps, clip, b):
    """drg_shard_run with DRG_SHARD_LAGGED as its emulation runs it (the worst case of
    the overlapped exchange): epoch j reads the negatives from the snapshot taken at
    the end of epoch j - 2 and its reactions are folded in after epoch j + 1."""
    pos = np.array(pos, dtype=np.float64)
    snaps = [pos.copy(), pos.copy()]
    deltas = [np.zeros_like(pos), np.zeros_like(pos)]
    n = len(draws_per_epoch)
    for j in range(n):
        pos, deltas[j & 1] = deferred_drawn_epoch(pos, draws_per_epoch[j], lrs[j], gamma, eps,
                                                  clip, b, snap=snaps[j & 1], fold=False)
        pos += deltas[(j + 1) & 1]
        deltas[(j + 1) & 1] = np.zeros_like(pos)
        snaps[j & 1] = pos.copy()
    pos += deltas[(n - 1) & 1]
    return pos


def node_parallel_iteration(indptr, targets, W, V, y, neg_idx, lr, gamma, eps, clip, b):
    """One Jacobi iteration of K7 in fp64:
    y_a' = y_a + lr * (sum_b W_ab clip(g_att(y_a, y_b)) + V_a sum_m clip(g_rep(y_a, y_cm)))
    with neg_idx[a, m] = -1 meaning "no negative" (all redraws collided)."""
    y = np.asarray(y, dtype=np.float64)
    n = len(y)
    src = np.repeat(np.arange(n), np.diff(indptr))
    d = y[src] - y[np.asarray(targets, dtype=np.int64)]
    g = clipped_attractive(d, b, clip) * np.asarray(W, dtype=np.float64)[:, None]
    att = np.zeros((n, 2))
    np.add.at(att, src, g)
    rep = np.zeros((n, 2))
    if neg_idx is not None and neg_idx.size:
        M = neg_idx.shape[1]
        a = np.repeat(np.arange(n), M)
        c = neg_idx.reshape(-1).astype(np.int64)
        ok = c >= 0
        dr = y[a[ok]] - y[c[ok]]
        gr = clipped_repulsive(dr, b, gamma, eps, clip)
        np.add.at(rep, a[ok], gr)
    return y + lr * (att + np.asarray(V, dtype=np.float64)[:, None] * rep)


def level_data(ns: SparseSimilarity, h: Hierarchy, level: int, neg_power=0.75):
    """P^l, R^l, Q^l of SURVEY §8(a) A10/A12 by pulling level-0 quantities
    through compose_maps: P^l_ab = sum of P_ij over i->a, j->b, a != b;
    R^l_a = sum of level-0 row masses; Q^l_a = sum of normalised negative weights."""
    cmap = compose_maps(h, level).astype(np.int64)
    n_l = h.levels[level].node_count
    src = ns.sources().astype(np.int64)
    a = cmap[src]
    bb = cmap[ns.targets.astype(np.int64)]
    keep = a != bb
    keys = a[keep] * n_l + bb[keep]
    w = ns.weights[keep]
    uniq, inv = np.unique(keys, return_inverse=True)
    P = np.zeros(len(uniq))
    np.add.at(P, inv, w)
    rows = uniq // n_l
    indptr = np.zeros(n_l + 1, dtype=np.int64)
    np.add.at(indptr, rows + 1, 1)
    np.cumsum(indptr, out=indptr)
    r = ns.row_masses()
    wneg = negative_weights(r, neg_power)
    R = np.zeros(n_l); np.add.at(R, cmap, r)
    Q = np.zeros(n_l); np.add.at(Q, cmap, wneg / wneg.sum())
    return indptr, (uniq % n_l).astype(np.int32), P, R, Q


# --------------------------------------------------------------------------
# Quality evaluators (metrics.py:77-145)
# --------------------------------------------------------------------------

def kl_divergence(ns: SparseSimilarity, y, b=2, z_pairs: int | None = None, seed=0) -> float:
    """KL(P||Q) = sum P log P + sum P log(1 + d^{2b}) + log Z,
    Z = sum_{i != j} 1/(1 + d^{2b}) (exact, or a seeded Monte-Carlo estimate
    over ``z_pairs`` uniform ordered pairs)."""
    y = np.asarray(y, dtype=np.float64)
    n = len(y)
    src = ns.sources().astype(np.int64)
    w = ns.weights
    keep = w > 0
    d2 = ((y[src[keep]] - y[ns.targets[keep]]) ** 2).sum(axis=1)
    term = float((w[keep] * np.log(w[keep])).sum() + (w[keep] * np.log1p(d2 ** b)).sum())
    if z_pairs is None:
        Z = 0.0
        chunk = max(1, 4_000_000 // max(n, 1))
        for lo in range(0, n, chunk):
            hi = min(lo + chunk, n)
            dd = ((y[lo:hi, None, :] - y[None, :, :]) ** 2).sum(axis=2)
            q = 1.0 / (1.0 + dd ** b)
            q[np.arange(hi - lo), np.arange(lo, hi)] = 0.0
            Z += float(q.sum())
    else:
        rng = np.random.default_rng(seed)
        i = rng.integers(0, n, z_pairs)
        j = rng.integers(0, n - 1, z_pairs)
        j = j + (j >= i)
        dd = ((y[i] - y[j]) ** 2).sum(axis=1)
        Z = float((1.0 / (1.0 + dd ** b)).mean()) * n * (n - 1)
    return term / max(float(w.sum()), 1e-300) + math.log(Z)


def neighborhood_preservation(g: Graph, y, k_eval=2, sample: np.ndarray | None = None) -> float:
    """metrics.py:114-145: mean Jaccard between each node's k_eval-hop set and its
    equally sized layout k-NN (ties by id).  ``sample``: evaluate on these nodes
    only (for n > 200k)."""
    from scipy.spatial import cKDTree
    y = np.asarray(y, dtype=np.float64)
    n = g.node_count
    nd = all_k_neighborhoods(g, k_eval)
    kp = np.diff(nd.indptr)
    nodes = np.arange(n) if sample is None else np.asarray(sample)
    tree = cKDTree(y)
    total = 0.0
    kmax = int(kp[nodes].max()) if len(nodes) else 0
    _, idx = tree.query(y[nodes], k=min(kmax + 1, n))
    idx = np.atleast_2d(idx)
    for r, i in enumerate(nodes):
        ki = int(kp[i])
        if ki == 0:
            total += 1.0
            continue
        row = idx[r]
        row = row[row != i][:ki]
        gs = set(nd.ids[nd.indptr[i]:nd.indptr[i + 1]].tolist())
        ls = set(row.tolist())
        total += len(gs & ls) / len(gs | ls)
    return total / len(nodes)
