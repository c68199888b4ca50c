"""Coarsening hierarchy and prolongation (drop-in for drgraph.multilevel).

The visiting permutation of each level is drawn exactly as the reference does
(numpy PCG64 ``default_rng(level_seed).permutation(n)``, multilevel.py:91, with
level seeds from ``default_rng(seed).integers(0, 2**63-1)``, multilevel.py:104-107)
-- that is seeding, not compute -- and the greedy pass itself runs as the K4
LFMIS kernel (drg_coarsen), bit-exact with coarsen_with_order.  The coarse CSR
is the deduplicated image of the fine edges (drg_coarse_graph).
"""

from __future__ import annotations

import concurrent.futures
import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .graph import DeviceGraph, Graph


@dataclass(frozen=True)
class Hierarchy:
    """Graphs G0..GL and child->parent maps (multilevel.py:19-45)."""

    levels: list
    maps: list
    rho: float
    min_size: int
    device_levels: list = field(default=None, repr=False, compare=False)
    device_maps: list = field(default=None, repr=False, compare=False)

    @property
    def depth(self) -> int:
        return len(self.levels) - 1

    def nbytes(self) -> int:
        return (sum(g.nbytes() for g in self.levels) + sum(m.nbytes for m in self.maps))

    def dump_text(self) -> str:
        lines = [f"{g.node_count} {g.edge_count}" for g in self.levels]
        for m in self.maps:
            lines.append(" ".join(str(int(p)) for p in m))
        return "\n".join(lines) + "\n"


@dataclass
class DeviceHierarchy:
    """The hierarchy resident in HBM: level graphs and int32 parent maps."""

    levels: list          # DeviceGraph per level
    maps: list            # torch int32, maps[l]: level l -> level l+1
    rho: float
    min_size: int
    rounds: list = field(default_factory=list)   # MIS rounds per coarsening

    @property
    def depth(self) -> int:
        return len(self.levels) - 1

    @property
    def sizes(self) -> list:
        return [g.node_count for g in self.levels]

    def nbytes(self) -> int:
        return sum(g.nbytes() for g in self.levels) + sum(m.numel() * 4 for m in self.maps)

    def to_host(self) -> Hierarchy:
        return Hierarchy([g.to_host() for g in self.levels], [m.cpu().numpy() for m in self.maps],
                         self.rho, self.min_size, self.levels, self.maps)


def device_parents(dg: DeviceGraph, order: torch.Tensor):
    """K4's greedy pass with an explicit visiting order (device int64): (parent
    int32, coarse node count, MIS rounds)."""
    n = dg.node_count
    if n < 1:
        raise ValueError("cannot coarsen an empty graph")
    parent = torch.empty(n, dtype=torch.int32, device=dg.indptr.device)
    nc = _lib.out_i64()
    rounds = ctypes.c_int32(0)
    _lib.call("drg_coarsen", _lib.ptr(dg.indptr), _lib.ptr(dg.indices), n, _lib.ptr(order),
              _lib.ptr(parent), _lib.byref(nc), _lib.byref(rounds), _lib.stream_ptr())
    return parent, nc.value, rounds.value


def device_coarse_graph(dg: DeviceGraph, parent: torch.Tensor, n_c: int) -> DeviceGraph:
    """The coarse CSR: the deduplicated image of the fine edges under ``parent``."""
    dev = dg.indptr.device
    indptr = torch.empty(n_c + 1, dtype=torch.int64, device=dev)
    cols = torch.empty(max(dg.nnz, 1), dtype=torch.int32, device=dev)
    nnz = _lib.out_i64()
    _lib.call("drg_coarse_graph", _lib.ptr(dg.indptr), _lib.ptr(dg.indices), dg.node_count,
              _lib.ptr(parent), n_c, _lib.ptr(indptr), _lib.ptr(cols), _lib.byref(nnz),
              _lib.stream_ptr())
    return DeviceGraph(indptr, cols[:nnz.value].clone())


def device_coarsen(dg: DeviceGraph, order: torch.Tensor):
    """K4 with an explicit visiting order (device int64).  Returns
    (coarse DeviceGraph, parent int32, MIS rounds)."""
    parent, n_c, rounds = device_parents(dg, order)
    return device_coarse_graph(dg, parent, n_c), parent, rounds


def level_order(n: int, seed: int) -> np.ndarray:
    """The reference's visiting order for one level (multilevel.py:91):
    ``np.random.default_rng(seed).permutation(n)`` bit for bit, as int32, by the
    library's host routine drg_pcg64_permutation (numpy's Fisher-Yates on the same
    PCG64 stream, draws and swaps pipelined on two threads)."""
    st = np.random.default_rng(seed).bit_generator.state
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    m64 = (1 << 64) - 1
    out = np.empty(n, dtype=np.int32)
    _lib.call_host("drg_pcg64_permutation", s >> 64, s & m64, inc >> 64, inc & m64,
              int(st["has_uint32"]), int(st["uinteger"]), n, out.ctypes.data)
    return out


def device_build_hierarchy(dg: DeviceGraph, rho: float = 0.8, min_size: int = 16, seed: int = 0,
                           max_levels: int | None = None, force_levels: int | None = None,
                           level0_relabel: torch.Tensor | None = None,
                           first_order=None) -> DeviceHierarchy:
    """build_hierarchy (multilevel.py:95-113) on a resident graph.  Extensions for
    the BASELINE configs: ``max_levels`` caps the total level count; ``force_levels``
    keeps coarsening past the rho test until that many levels exist.
    ``level0_relabel`` (old id -> new id): ``dg`` is the input graph relabelled; the
    reference's level-0 visiting order (drawn over the original ids) is translated,
    so the coarse levels are exactly the reference's.  ``first_order``: a
    concurrent.futures.Future of that level-0 order, drawn ahead (see
    first_level_order) so the host permutation overlaps device work."""
    if not 0.0 < rho < 1.0:
        raise ValueError("rho must be in (0, 1)")
    if min_size < 1:
        raise ValueError("min_size must be >= 1")
    rng = np.random.default_rng(seed)
    h = DeviceHierarchy([dg], [], rho, min_size)
    ahead = None   # (seed, future) of the next level's visiting order, drawn early
    while h.levels[-1].node_count > min_size:
        if max_levels is not None and len(h.levels) >= max_levels:
            break
        top = h.levels[-1]
        if ahead is not None:
            level_seed, fut = ahead
            host_order = fut.result()
            ahead = None
        else:
            level_seed = int(rng.integers(0, 2**63 - 1))
            if first_order is not None and len(h.levels) == 1:
                host_order = first_order.result()
            else:
                host_order = level_order(top.node_count, level_seed)
        order = torch.from_numpy(host_order).to(top.indptr.device).to(torch.int64)
        if level0_relabel is not None and len(h.levels) == 1:
            order = level0_relabel.to(torch.int64)[order]
        parent, n_c, rounds = device_parents(top, order)
        forced = force_levels is not None and len(h.levels) < force_levels
        if not forced and n_c > rho * top.node_count:
            break
        if n_c == top.node_count:
            break
        # the next level's host permutation (its size is n_c, its seed the next draw of
        # the same stream) runs on a host thread while the device builds this coarse CSR
        if n_c > min_size and (max_levels is None or len(h.levels) + 1 < max_levels):
            nxt = int(rng.integers(0, 2**63 - 1))
            ahead = (nxt, _AHEAD_POOL.submit(level_order, n_c, nxt))
        h.levels.append(device_coarse_graph(top, parent, n_c))
        h.maps.append(parent)
        h.rounds.append(rounds)
    return h


def coarsen_with_order(g: Graph, order: np.ndarray):
    """multilevel.py:48-79 on the GPU (bit-exact parents and coarse CSR)."""
    _lib.load()
    dg = DeviceGraph.from_host(g)
    coarse, parent, _ = device_coarsen(
        dg, torch.from_numpy(np.ascontiguousarray(order, dtype=np.int64)).cuda())
    return coarse.to_host(), parent.cpu().numpy()


def coarsen_once(g: Graph, seed: int):
    """multilevel.py:82-92."""
    if g.node_count < 1:
        raise ValueError("cannot coarsen an empty graph")
    return coarsen_with_order(g, level_order(g.node_count, seed))


def build_hierarchy(g: Graph, rho: float = 0.8, min_size: int = 16, seed: int = 0,
                    max_levels: int | None = None, force_levels: int | None = None) -> Hierarchy:
    """multilevel.py:95-113 (level 0 is the input graph by reference)."""
    if not 0.0 < rho < 1.0:
        raise ValueError("rho must be in (0, 1)")
    if min_size < 1:
        raise ValueError("min_size must be >= 1")
    if g.node_count <= min_size:
        return Hierarchy([g], [], rho, min_size)
    _lib.load()
    dh = device_build_hierarchy(DeviceGraph.from_host(g), rho, min_size, seed, max_levels,
                                force_levels)
    host = dh.to_host()
    return Hierarchy([g] + host.levels[1:], host.maps, rho, min_size, dh.levels, dh.maps)


def compose_maps(h: Hierarchy, level: int) -> np.ndarray:
    """Flat map from level-0 ids to level-``level`` ancestors (multilevel.py:116-123)."""
    if not 0 <= level <= h.depth:
        raise ValueError(f"level {level} outside hierarchy of depth {h.depth}")
    n0 = h.levels[0].node_count
    if level == 0:
        return np.arange(n0, dtype=np.int32)
    _lib.load()
    st = _lib.stream_ptr()
    flat = torch.empty(n0, dtype=torch.int32, device="cuda")
    nxt = torch.empty_like(flat)
    dmaps = h.device_maps or [torch.from_numpy(np.ascontiguousarray(m, dtype=np.int32)).cuda()
                              for m in h.maps]
    _lib.call("drg_compose_maps", None, None, n0, _lib.ptr(flat), st)
    for m in dmaps[:level]:
        _lib.call("drg_compose_maps", _lib.ptr(flat), _lib.ptr(m), n0, _lib.ptr(nxt), st)
        flat, nxt = nxt, flat
    return flat.cpu().numpy()


def device_prolong(y_coarse: torch.Tensor, parent: torch.Tensor, jitter: float, seed: int
                   ) -> torch.Tensor:
    """K6: y_fine = y_coarse[parent] + N(0, jitter) (Philox Box-Muller)."""
    n = parent.numel()
    out = torch.empty((n, 2), dtype=torch.float32, device=y_coarse.device)
    _lib.call("drg_prolong", _lib.ptr(y_coarse), _lib.ptr(parent), n, float(jitter),
              int(seed) & 0xFFFFFFFFFFFFFFFF, _lib.ptr(out), _lib.stream_ptr())
    return out


def prolong(coarse_positions: np.ndarray, cmap: np.ndarray, jitter_scale: float,
            seed: int) -> np.ndarray:
    """multilevel.py:126-138 on the GPU.  Zero jitter copies parents exactly; the
    jitter is a counter-based normal stream (statistically the reference's
    N(0, jitter_scale), not numpy's bit stream).  Positions are fp32 on device."""
    _lib.load()
    yc = torch.from_numpy(np.ascontiguousarray(coarse_positions, dtype=np.float32)).cuda()
    pm = torch.from_numpy(np.ascontiguousarray(cmap, dtype=np.int32)).cuda()
    return device_prolong(yc, pm, jitter_scale, seed).cpu().numpy().astype(np.float64)


def isolated_last(dg: DeviceGraph, min_fraction: float = 0.01):
    """Relabelling that moves isolated nodes behind all others (relative order kept).
    Isolated nodes are never gathered as neighbours, so the gathered part of Y
    becomes one dense prefix (L2-resident where the whole Y would not be, e.g.
    R-MAT).  Returns (relabelled graph, old -> new id) or (dg, None)."""
    deg = dg.indptr[1:] - dg.indptr[:-1]
    iso = deg == 0
    n = deg.numel()
    if n == 0 or float(iso.float().mean()) < min_fraction:
        return dg, None
    order = torch.argsort(iso.to(torch.int8), stable=True)           # new -> old
    rel = torch.empty_like(order)
    rel[order] = torch.arange(n, device=order.device)
    indptr = torch.zeros(n + 1, dtype=torch.int64, device=order.device)
    indptr[1:] = torch.cumsum(deg[order], 0)
    # neighbours are never isolated and keep their relative order: rows stay sorted
    indices = rel.to(torch.int32)[dg.indices.to(torch.int64)]
    return DeviceGraph(indptr, indices), rel.to(torch.int32)


def relabel_coarse_levels(dh: DeviceHierarchy) -> list:
    """Isolated-last relabelling of every coarse level of a built hierarchy (maps
    and level graphs rewritten).  Returns the per-level old -> new maps (None =
    identity); level 0 is left to the caller."""
    rels = [None]
    for l in range(1, dh.depth + 1):
        g2, rel = isolated_last(dh.levels[l])
        rels.append(rel)
        if rel is None:
            continue
        dh.levels[l] = g2
        dh.maps[l - 1] = rel[dh.maps[l - 1].to(torch.int64)]
        if l < dh.depth:
            m = torch.empty_like(dh.maps[l])
            m[rel.to(torch.int64)] = dh.maps[l]
            dh.maps[l] = m
    return rels


_AHEAD_POOL = concurrent.futures.ThreadPoolExecutor(1)


def first_level_order(n: int, seed: int, executor):
    """Future of the reference's level-0 visiting order (multilevel.py:91 with the
    first seed of build_hierarchy's stream, multilevel.py:104-107), computed on a
    host thread while the device runs the k-hop / similarity kernels."""
    def draw():
        level_seed = int(np.random.default_rng(seed).integers(0, 2**63 - 1))
        return level_order(n, level_seed)
    return executor.submit(draw)
