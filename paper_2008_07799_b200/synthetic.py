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


def rmat(scale: int = 24, edge_factor: int = 16, a=0.57, b=0.19, c=0.19, seed: int = 0,
         device="cuda", chunk: int = 1 << 26):
    """R-MAT with 2^scale nodes and edge_factor * 2^scale draws (no relabelling),
    symmetrised, self-loops and duplicates removed by drg_from_edges."""
    n = 1 << scale
    m = edge_factor * n
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    parts = []
    for lo in range(0, m, chunk):
        cnt = min(chunk, m - lo)
        u = torch.zeros(cnt, dtype=torch.int64, device="cuda")
        v = torch.zeros(cnt, dtype=torch.int64, device="cuda")
        for _ in range(scale):
            r = torch.rand(cnt, device="cuda", generator=g)
            bit_u = (r >= a + b).to(torch.int64)                    # quadrants c, d
            bit_v = (((r >= a) & (r < a + b)) | (r >= a + b + c)).to(torch.int64)  # b, d
            u = (u << 1) | bit_u
            v = (v << 1) | bit_v
        parts.append(torch.stack([u, v], 1))
    e = torch.cat(parts)
    return _finish(device_from_edges(e, n), device)
