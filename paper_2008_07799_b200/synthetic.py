"""Seeded synthetic graphs of the BASELINE.json configs (inputs, not the path).

The reference ships no generators for these families (SURVEY §8(c) "Datasets"),
so these are the builder's own, shared by the GPU arm, the CPU arms and the
tests.  Large CSRs are produced on the device and canonicalised by
drg_from_edges, so they match the reference's from_edges (graph.py:80-125)
bit for bit.

  C1 grid(100, 100)            4-neighbour grid, 10,000 nodes
  C2 rgg(200_000, seed)        unit-square random geometric graph, mean degree 10
  C3 barabasi_albert(1e6, 4)   preferential attachment, m = 4
  C4 mesh3d(120)               26-neighbour 3-D mesh, 1,728,000 nodes
  C5 rmat(24, 16)              R-MAT (.57, .19, .19, .05), symmetrised, deduplicated
"""

from __future__ import annotations

import math

import numpy as np
import torch

from .graph import DeviceGraph, Graph, device_from_edges


def _finish(dg: DeviceGraph, device) -> DeviceGraph | Graph:
    return dg if device == "cuda" else dg.to_host()


def grid(w: int, h: int, device="cuda"):
    """w x h 4-neighbour grid (row-major ids), as the reference tests' grid_graph."""
    idx = torch.arange(w * h, dtype=torch.int64, device="cuda").reshape(h, w)
    e = torch.cat([torch.stack([idx[:, :-1].reshape(-1), idx[:, 1:].reshape(-1)], 1),
                   torch.stack([idx[:-1, :].reshape(-1), idx[1:, :].reshape(-1)], 1)])
    return _finish(device_from_edges(e, w * h), device)


def mesh3d(side: int = 120, device="cuda"):
    """side^3 nodes, 26-neighbourhood, id = (x*side + y)*side + z.  Built directly
    as a canonical CSR: offsets in lexicographic (dx, dy, dz) order are in
    increasing id order, so masked rows come out sorted."""
    dev = "cuda"
    n = side ** 3
    ids = torch.arange(n, dtype=torch.int64, device=dev)
    x, y, z = ids // (side * side), (ids // side) % side, ids % side
    offs = [(dx, dy, dz) for dx in (-1, 0, 1) for dy in (-1, 0, 1) for dz in (-1, 0, 1)
            if (dx, dy, dz) != (0, 0, 0)]
    cols, masks = [], []
    for dx, dy, dz in offs:
        ok = ((x + dx >= 0) & (x + dx < side) & (y + dy >= 0) & (y + dy < side)
              & (z + dz >= 0) & (z + dz < side))
        cols.append(ids + (dx * side * side + dy * side + dz))
        masks.append(ok)
    col = torch.stack(cols, 1)
    mask = torch.stack(masks, 1)
    indices = col[mask].to(torch.int32)
    indptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    indptr[1:] = torch.cumsum(mask.sum(1), 0)
    return _finish(DeviceGraph(indptr, indices.contiguous()), device)


def rgg(n: int = 200_000, seed: int = 0, mean_degree: float = 10.0, device="cuda"):
    """n points U[0,1]^2 (numpy PCG64 seed), edge iff distance < r with
    r = sqrt(mean_degree / (pi n))."""
    from scipy.spatial import cKDTree
    pts = np.random.default_rng(seed).random((n, 2))
    r = math.sqrt(mean_degree / (math.pi * n))
    pairs = cKDTree(pts).query_pairs(r, output_type="ndarray")
    e = torch.from_numpy(pairs.astype(np.int64)).cuda()
    return _finish(device_from_edges(e, n), device)


def barabasi_albert(n: int = 1_000_000, m: int = 4, seed: int = 0, device="cuda"):
    """Preferential attachment, m edges per new node, in the linearised-chord-
    diagram form (Bollobas-Riordan): edge e of node e // m gets endpoint slots 2e
    (itself) and 2e+1, which copies a uniform slot r in [0, 2e+1] -- i.e. a node
    chosen proportionally to its current degree.  Copy chains are resolved on the
    device by pointer jumping; loops and repeated edges are dropped by
    drg_from_edges.  Power-law degrees (exponent 3)."""
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    E = m * n
    e = torch.arange(E, dtype=torch.int64, device="cuda")
    span = (2 * e + 2).to(torch.float64)
    r = torch.minimum((torch.rand(E, dtype=torch.float64, device="cuda", generator=gen)
                       * span).to(torch.int64), 2 * e + 1)
    ptr = r.clone()
    for _ in range(256):
        odd = (ptr & 1) == 1
        if not bool(odd.any()):
            break
        ptr = torch.where(odd, r[torch.clamp((ptr - 1) // 2, min=0)], ptr)
    pairs = torch.stack([e // m, (ptr // 2) // m], 1)
    return _finish(device_from_edges(pairs, n), device)


# R-MAT quadrant draws from a counter-based hash (splitmix64 of (seed, edge, level)):
# the same edges from torch on the device (the bench) and from numpy on any host
# (the CPU reference arm of the C5 parity runs, scripts/quality_c5.py)
_SM_GAMMA = 0x9E3779B97F4A7C15
_SM_M1 = 0xBF58476D1CE4E5B9
_SM_M2 = 0x94D049BB133111EB
_SEED_MIX = 0xD1B54A32D192ED03


def _s64(c: int) -> int:   # uint64 constant as the int64 torch holds
    return c - (1 << 64) if c >= 1 << 63 else c


def _rmat_uniform_torch(x: torch.Tensor) -> torch.Tensor:
    """splitmix64(x) -> float64 in [0, 1) (53 bits); int64 tensors wrap like uint64,
    right shifts made logical by masking."""
    def srl(z, k):
        return (z >> k) & ((1 << (64 - k)) - 1)
    z = x + _s64(_SM_GAMMA)
    z = (z ^ srl(z, 30)) * _s64(_SM_M1)
    z = (z ^ srl(z, 27)) * _s64(_SM_M2)
    z = z ^ srl(z, 31)
    return srl(z, 11).to(torch.float64) * (1.0 / (1 << 53))


def _rmat_uniform_numpy(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(_SM_GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_SM_M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_SM_M2)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53))


def rmat_edges(scale: int, edge_factor: int = 16, a=0.57, b=0.19, c=0.19, seed: int = 0,
               lo: int = 0, hi: int | None = None, device="cuda"):
    """Draws [lo, hi) of R-MAT(2^scale, edge_factor * 2^scale): level l of draw e takes
    quadrant a / b / c / d from u = splitmix64(seed * K + 32 e + l) -- an int64 [m, 2]
    torch tensor (``device``), or a numpy array for device="numpy"."""
    m = edge_factor << scale
    hi = m if hi is None else min(hi, m)
    ab, abc = a + b, a + b + c
    base = (seed * _SEED_MIX) & ((1 << 64) - 1)
    if device == "numpy":
        e = np.arange(lo, hi, dtype=np.uint64)
        u = np.zeros(hi - lo, dtype=np.int64)
        v = np.zeros(hi - lo, dtype=np.int64)
        with np.errstate(over="ignore"):
            key = e * np.uint64(32) + np.uint64(base)
        for lev in range(scale):
            with np.errstate(over="ignore"):
                r = _rmat_uniform_numpy(key + np.uint64(lev))
            u = (u << 1) | (r >= ab)
            v = (v << 1) | (((r >= a) & (r < ab)) | (r >= abc))
        return np.stack([u, v], 1)
    e = torch.arange(lo, hi, dtype=torch.int64, device=device)
    key = e * 32 + _s64(base)
    u = torch.zeros(hi - lo, dtype=torch.int64, device=device)
    v = torch.zeros(hi - lo, dtype=torch.int64, device=device)
    for lev in range(scale):
        r = _rmat_uniform_torch(key + lev)
        u = (u << 1) | (r >= ab).to(torch.int64)                          # quadrants c, d
        v = (v << 1) | (((r >= a) & (r < ab)) | (r >= abc)).to(torch.int64)  # b, d
    return torch.stack([u, v], 1)


def rmat(scale: int = 24, edge_factor: int = 16, a=0.57, b=0.19, c=0.19, seed: int = 0,
         device="cuda", chunk: int = 1 << 26):
    """R-MAT with 2^scale nodes and edge_factor * 2^scale draws (rmat_edges; no
    relabelling), symmetrised, self-loops and duplicates removed by drg_from_edges."""
    n = 1 << scale
    m = edge_factor * n
    parts = [rmat_edges(scale, edge_factor, a, b, c, seed, lo, lo + chunk, device="cuda")
             for lo in range(0, m, chunk)]
    e = torch.cat(parts)
    del parts
    return _finish(device_from_edges(e, n), device)
