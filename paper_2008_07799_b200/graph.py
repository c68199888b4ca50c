"""Graph types and the K1 k-hop kernel (drop-in for drgraph.graph).

Host types keep the reference's layout and methods (graph.py:27-77, 252-277) so
callers see numpy arrays exactly as before; every computation runs on the GPU
through libdrgraph_b200.so.  ``DeviceGraph`` / ``DeviceNeighborDistances`` are
the HBM-resident forms the pipeline passes between kernels without host trips.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterator

import numpy as np
import torch

from . import _lib


class ParseError(ValueError):
    """Malformed graph input (graph.py:17-24)."""

    def __init__(self, message: str, line: int | None = None):
        self.line = line
        if line is not None:
            message = f"line {line}: {message}"
        super().__init__(message)


@dataclass(frozen=True, eq=False)
class Graph:
    """Undirected simple graph in compressed-row layout (graph.py:27-77).

    ``indices[indptr[i]:indptr[i+1]]`` holds the sorted neighbour ids of node i;
    every edge appears in both rows.
    """

    indptr: np.ndarray   # int64, node_count + 1
    indices: np.ndarray  # int32, 2 * edge_count

    @property
    def node_count(self) -> int:
        return len(self.indptr) - 1

    @property
    def edge_count(self) -> int:
        return len(self.indices) // 2

    @property
    def degrees(self) -> np.ndarray:
        return np.diff(self.indptr)

    def neighbors(self, i: int) -> np.ndarray:
        return self.indices[self.indptr[i]:self.indptr[i + 1]]

    def degree(self, i: int) -> int:
        return int(self.indptr[i + 1] - self.indptr[i])

    def edge_array(self) -> np.ndarray:
        u = np.repeat(np.arange(self.node_count, dtype=np.int32), self.degrees)
        keep = u < self.indices
        return np.column_stack([u[keep], self.indices[keep]])

    def edges(self) -> Iterator[tuple[int, int]]:
        for u, v in self.edge_array():
            yield int(u), int(v)

    def nbytes(self) -> int:
        return self.indptr.nbytes + self.indices.nbytes

    def __eq__(self, other: object) -> bool:
        if not isinstance(other, Graph):
            return NotImplemented
        return (np.array_equal(self.indptr, other.indptr)
                and np.array_equal(self.indices, other.indices))

    def __repr__(self) -> str:
        return f"Graph(nodes={self.node_count}, edges={self.edge_count})"


@dataclass
class DeviceGraph:
    """A Graph resident in HBM: indptr int64[n+1], indices int32[2E]."""

    indptr: torch.Tensor
    indices: torch.Tensor

    @property
    def node_count(self) -> int:
        return self.indptr.numel() - 1

    @property
    def nnz(self) -> int:
        return self.indices.numel()

    @staticmethod
    def from_host(g: Graph, device="cuda", non_blocking: bool = False) -> "DeviceGraph":
        ip = torch.from_numpy(np.ascontiguousarray(g.indptr, dtype=np.int64))
        ix = torch.from_numpy(np.ascontiguousarray(g.indices, dtype=np.int32))
        return DeviceGraph(ip.to(device, non_blocking=non_blocking),
                           ix.to(device, non_blocking=non_blocking))

    def to_host(self) -> Graph:
        return Graph(indptr=self.indptr.cpu().numpy(), indices=self.indices.cpu().numpy())

    def nbytes(self) -> int:
        return self.indptr.numel() * 8 + self.indices.numel() * 4


def device_from_edges(pairs: torch.Tensor, node_count: int) -> DeviceGraph:
    """from_edges on device (graph.py:80-125): drg_from_edges."""
    pairs = pairs.to(torch.int64).contiguous()
    m = pairs.numel() // 2
    indptr = torch.empty(node_count + 1, dtype=torch.int64, device=pairs.device)
    out = torch.empty(max(2 * m, 1), dtype=torch.int32, device=pairs.device)
    nnz = _lib.out_i64()
    _lib.call("drg_from_edges", _lib.ptr(pairs), m, node_count, _lib.ptr(indptr), _lib.ptr(out),
              _lib.byref(nnz), _lib.stream_ptr())
    return DeviceGraph(indptr, out[:nnz.value].clone())


def from_edges(pairs, node_count: int | None = None, remap_sparse_ids: bool = False) -> Graph:
    """Canonical CSR from (u, v) pairs (graph.py:80-125), built on the GPU.

    Self-loops are dropped, duplicate and reversed edges collapse.  With
    ``remap_sparse_ids`` ids are compacted when the max id exceeds twice the
    distinct-id count (graph.py:94-100)."""
    pairs = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    if pairs.size and pairs.min() < 0:
        raise ParseError("negative node id")
    if node_count is None:
        if pairs.size == 0:
            node_count = 0
        else:
            distinct = np.unique(pairs)
            max_id = int(distinct[-1])
            if remap_sparse_ids and max_id > 2 * len(distinct):
                lookup = np.full(max_id + 1, -1, dtype=np.int64)
                lookup[distinct] = np.arange(len(distinct))
                pairs = lookup[pairs]
                node_count = len(distinct)
            else:
                node_count = max_id + 1
    _lib.load()
    dg = device_from_edges(torch.from_numpy(np.ascontiguousarray(pairs)).cuda(), node_count)
    return dg.to_host()


@dataclass(frozen=True)
class NeighborDistances:
    """Neighbours within k hops with exact hop distances (graph.py:252-277).
    Rows sorted by (distance, id); symmetric relation."""

    indptr: np.ndarray  # int64, node_count + 1
    ids: np.ndarray     # int32
    dists: np.ndarray   # int32, 1..k
    k: int

    @property
    def node_count(self) -> int:
        return len(self.indptr) - 1

    def row(self, i: int) -> tuple[np.ndarray, np.ndarray]:
        lo, hi = self.indptr[i], self.indptr[i + 1]
        return self.ids[lo:hi], self.dists[lo:hi]

    def row_size(self, i: int) -> int:
        return int(self.indptr[i + 1] - self.indptr[i])

    def nbytes(self) -> int:
        return self.indptr.nbytes + self.ids.nbytes + self.dists.nbytes


@dataclass
class DeviceNeighborDistances:
    indptr: torch.Tensor  # int64
    ids: torch.Tensor     # int32
    dists: torch.Tensor   # int32
    k: int
    cap: int = 0

    @property
    def node_count(self) -> int:
        return self.indptr.numel() - 1

    @property
    def nnz(self) -> int:
        return self.ids.numel()

    def to_host(self) -> NeighborDistances:
        return NeighborDistances(self.indptr.cpu().numpy(), self.ids.cpu().numpy(),
                                 self.dists.cpu().numpy(), self.k)

    @staticmethod
    def from_host(nd: NeighborDistances) -> "DeviceNeighborDistances":
        return DeviceNeighborDistances(
            torch.from_numpy(np.ascontiguousarray(nd.indptr, dtype=np.int64)).cuda(),
            torch.from_numpy(np.ascontiguousarray(nd.ids, dtype=np.int32)).cuda(),
            torch.from_numpy(np.ascontiguousarray(nd.dists, dtype=np.int32)).cuda(), nd.k)


def device_k_neighborhoods(dg: DeviceGraph, k: int, cap: int | None = None
                           ) -> DeviceNeighborDistances:
    """K1 on a resident graph: drg_khop_count + drg_khop_fill."""
    if k < 1:
        raise ValueError("k must be >= 1")
    n = dg.node_count
    capv = int(cap) if cap else 0
    dev = dg.indptr.device
    indptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    nnz = _lib.out_i64()
    st = _lib.stream_ptr()
    _lib.call("drg_khop_count", _lib.ptr(dg.indptr), _lib.ptr(dg.indices), n, k, capv,
              _lib.ptr(indptr), _lib.byref(nnz), st)
    ids = torch.empty(max(nnz.value, 1), dtype=torch.int32, device=dev)
    dists = torch.empty(max(nnz.value, 1), dtype=torch.int32, device=dev)
    _lib.call("drg_khop_fill", _lib.ptr(dg.indptr), _lib.ptr(dg.indices), n, k, capv,
              _lib.ptr(indptr), _lib.ptr(ids), _lib.ptr(dists), st)
    return DeviceNeighborDistances(indptr, ids[:nnz.value], dists[:nnz.value], k, capv)


def all_k_neighborhoods(g: Graph, k: int, with_stats: bool = False,
                        cap: int | None = None):
    """graph.py:308-366 on the GPU (bit-exact rows).  ``with_stats`` also returns
    the number of queue pushes, which for a BFS equals the entry count
    (test_graph.py:261-266).  ``cap``: BASELINE C3 neighbour-cap extension."""
    if k < 1:
        raise ValueError("k must be >= 1")
    _lib.load()
    nd = device_k_neighborhoods(DeviceGraph.from_host(g), k, cap).to_host()
    return (nd, len(nd.ids)) if with_stats else nd


def device_components(dg: DeviceGraph, labels: bool = False):
    n = dg.node_count
    out = torch.empty(max(n, 1), dtype=torch.int32, device=dg.indptr.device) if labels else None
    cnt = _lib.out_i64()
    _lib.call("drg_components", _lib.ptr(dg.indptr), _lib.ptr(dg.indices), n, _lib.ptr(out),
              _lib.byref(cnt), _lib.stream_ptr())
    return (cnt.value, out[:n]) if labels else cnt.value


def connected_components(g: Graph) -> np.ndarray:
    """Component labels 0..C-1 in first-seen order (graph.py:369-388)."""
    _lib.load()
    if g.node_count == 0:
        return np.zeros(0, dtype=np.int32)
    _, lab = device_components(DeviceGraph.from_host(g), labels=True)
    return lab.cpu().numpy()
