"""Graph types and the K1 k-hop kernel (drop-in for drgraph.graph).

Host types keep the reference's layout and methods (graph.py:27-77, 252-277) so
callers see numpy arrays exactly as before; every computation runs on the GPU
through libdrgraph_b200.so.  ``DeviceGraph`` / ``DeviceNeighborDistances`` are
the HBM-resident forms the pipeline passes between kernels without host trips.
"""

from __future__ import annotations

import warnings
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


def device_remap_ids(pairs: torch.Tensor, remap_sparse_ids: bool) -> int:
    """node_count of from_edges without an explicit count (graph.py:90-103), on the
    device: distinct ids by radix sort + unique; with ``remap_sparse_ids`` and
    max id > 2 * distinct the ids are compacted in place (lower bound in the
    distinct ids == the reference's lookup table).  Raises on a negative id."""
    n = _lib.out_i64()
    try:
        _lib.call("drg_id_remap", _lib.ptr(pairs), pairs.numel() // 2, int(remap_sparse_ids),
                  _lib.byref(n), _lib.stream_ptr())
    except ValueError as e:
        if "negative node id" in str(e):
            raise ParseError("negative node id") from None
        if "Maximum allowed dimension exceeded" in str(e):
            raise ValueError("Maximum allowed dimension exceeded") from None
        raise
    return n.value


def from_edges(pairs, node_count: int | None = None, remap_sparse_ids: bool = False) -> Graph:
    """Canonical CSR from (u, v) pairs (graph.py:80-125), built on the GPU.

    Self-loops are dropped, duplicate and reversed edges collapse.  With
    ``remap_sparse_ids`` ids are compacted when the max id exceeds twice the
    distinct-id count (graph.py:94-100)."""
    pairs = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    if pairs.size == 0:
        n = 0 if node_count is None else node_count
        return Graph(np.zeros(n + 1, dtype=np.int64), np.empty(0, dtype=np.int32))
    _lib.load()
    dp = torch.from_numpy(np.ascontiguousarray(pairs)).cuda()
    if node_count is None:
        node_count = device_remap_ids(dp, remap_sparse_ids)
    elif pairs.min() < 0:
        raise ParseError("negative node id")
    return device_from_edges(dp, node_count).to_host()


# ------------------------------------------------------------------ text ingestion
# graph.py:128-243 on the device (ingest.cu): the bytes go to HBM once, line
# splitting, tokenising and int() run there; the host only formats the message of
# the first failing line, and (MatrixMarket) reads the header and size lines.

_MM_FIELDS = {"pattern", "real", "integer", "complex"}
_MM_SYMMETRIES = {"general", "symmetric", "skew-symmetric", "hermitian"}
_SPLITLINES, _NEWLINE_ONLY = 0, 1
_SPLITLINES_CHECKED = 2   # raw file bytes: strict UTF-8 first, as open(encoding="utf-8")


def _text_source(source):
    """(UTF-8 bytes, line mode, explicit line starts or None) for the reference's
    source kinds (graph.py:128-131): a str is split by str.splitlines, a text stream
    by its "\n" line iteration, any other iterable element-wise.  ``bytes`` (the
    raw contents of a UTF-8 file, as cli.py:194 reads them) split like the str."""
    if isinstance(source, (bytes, bytearray, memoryview)):
        return np.frombuffer(bytes(source), dtype=np.uint8), _SPLITLINES_CHECKED, None
    if isinstance(source, np.ndarray) and source.dtype == np.uint8:
        return np.ascontiguousarray(source).reshape(-1), _SPLITLINES_CHECKED, None
    if isinstance(source, str):
        return np.frombuffer(source.encode("utf-8", "surrogatepass"), np.uint8), _SPLITLINES, None
    if hasattr(source, "read"):
        text = source.read()
        return np.frombuffer(text.encode("utf-8", "surrogatepass"), np.uint8), _NEWLINE_ONLY, None
    parts = [str(x).encode("utf-8", "surrogatepass") for x in source]
    starts = np.zeros(len(parts), dtype=np.int64)
    if parts:
        np.cumsum(np.fromiter(map(len, parts[:-1]), dtype=np.int64, count=len(parts) - 1),
                  out=starts[1:])
    return np.frombuffer(b"".join(parts), dtype=np.uint8), None, starts


class _DeviceText:
    """Text bytes in HBM with their line starts (drg_text_lines)."""

    def __init__(self, data: np.ndarray, mode, starts):
        _lib.load()
        self.host = data
        self.n = int(data.size)
        with warnings.catch_warnings():   # read-only bytes: only copied from, never written
            warnings.simplefilter("ignore", UserWarning)
            host = torch.from_numpy(data) if data.size else torch.empty(0, dtype=torch.uint8)
        if data.size:
            host = host.pin_memory() if torch.cuda.is_available() else host
        self.dev = host.to("cuda", non_blocking=True) if data.size else \
            torch.empty(1, dtype=torch.uint8, device="cuda")
        if starts is not None:
            self.starts = torch.from_numpy(starts).cuda()
            return
        count, bad = _lib.out_i64(), _lib.out_i64()
        check = mode == _SPLITLINES_CHECKED
        mode = _SPLITLINES if check else mode
        _lib.call("drg_text_lines", _lib.ptr(self.dev), self.n, mode, None, _lib.byref(count),
                  _lib.byref(bad) if check else None, _lib.stream_ptr())
        if check and bad.value >= 0:
            p = bad.value
            try:   # the codec's own verdict on the sequence at the first invalid byte
                bytes(data[p:p + 4]).decode("utf-8")
                start, end, reason = 0, 1, "invalid continuation byte"
            except UnicodeDecodeError as e:
                start, end, reason = e.start, e.end, e.reason
            raise UnicodeDecodeError("utf-8", bytes(data), p + start, p + end, reason)
        self.starts = torch.empty(max(count.value, 1), dtype=torch.int64, device="cuda")
        if count.value:
            _lib.call("drg_text_lines", _lib.ptr(self.dev), self.n, mode, _lib.ptr(self.starts),
                      _lib.byref(count), None, _lib.stream_ptr())
        self.starts = self.starts[:count.value]

    @property
    def n_lines(self) -> int:
        return int(self.starts.numel())

    def lines(self, lo: int, hi: int) -> list[str]:
        """Decoded text of lines lo..hi-1 (host, for headers and messages)."""
        hi = min(hi, self.n_lines)
        if hi <= lo:
            return []
        st = self.starts[lo:min(hi + 1, self.n_lines)].cpu().numpy().tolist()
        if len(st) == hi - lo:
            st.append(self.n)
        return [bytes(self.host[a:b]).decode("utf-8", "surrogatepass") for a, b in zip(st[:-1], st[1:])]

    def parse(self, first: int, kind: int, rows: int = 0, declared: int = 0):
        """drg_parse_lines over lines first..: (device pairs [m, 2], error line index or
        -1, status, overflow)."""
        n_lines = self.n_lines - first
        pairs = torch.empty((max(n_lines, 1), 2), dtype=torch.int64, device="cuda")
        m, err, status, over = _lib.out_i64(), _lib.out_i64(), _lib.out_i32(), _lib.out_i32()
        starts = self.starts[first:] if n_lines > 0 else self.starts
        _lib.call("drg_parse_lines", _lib.ptr(self.dev), self.n, _lib.ptr(starts), max(n_lines, 0),
                  kind, rows, declared, _lib.ptr(pairs), _lib.byref(m), _lib.byref(err),
                  _lib.byref(status), _lib.byref(over), _lib.stream_ptr())
        e = err.value
        return pairs[:m.value], (first + e if e >= 0 else -1), status.value, over.value


def _graph_from_device_pairs(pairs: torch.Tensor, node_count: int | None,
                             remap_sparse_ids: bool) -> Graph:
    if pairs.numel() == 0:
        n = 0 if node_count is None else node_count
        return Graph(np.zeros(n + 1, dtype=np.int64), np.empty(0, dtype=np.int32))
    pairs = pairs.contiguous()
    if node_count is None:
        node_count = device_remap_ids(pairs, remap_sparse_ids)
    return device_from_edges(pairs, node_count).to_host()


def parse_edge_list(source) -> Graph:
    """Whitespace-separated "u v" edge list (graph.py:134-167): '#'/'%' comments and
    blank lines skipped, exactly two non-negative int() ids per line, sparse id
    spaces remapped.  Same ParseError messages and line numbers."""
    text = _DeviceText(*_text_source(source))
    pairs, err, status, overflow = text.parse(0, 0)
    if err >= 0:
        line = text.lines(err, err + 1)[0].strip()
        tokens = line.split()
        if status == 2:
            raise ParseError(f"expected two ids, got {len(tokens)} tokens", err + 1)
        if status == 3:
            raise ParseError(f"malformed integer in {tokens!r}", err + 1)
        raise ParseError(f"negative node id in {tokens!r}", err + 1)
    if overflow:   # np.asarray(us, dtype=np.int64) on an id >= 2**63 (graph.py:162-163)
        raise OverflowError("Python int too large to convert to C long")
    return _graph_from_device_pairs(pairs, None, True)


def parse_matrix_market(source) -> Graph:
    """MatrixMarket coordinate file as an undirected graph (graph.py:170-243): the
    header and size lines are read on the host, the entry lines on the device."""
    text = _DeviceText(*_text_source(source))
    if text.n_lines == 0:
        raise ParseError("empty file, missing MatrixMarket header")
    header = text.lines(0, 1)[0]
    tokens = header.strip().split()
    if len(tokens) < 5 or tokens[0] != "%%MatrixMarket":
        raise ParseError("missing '%%MatrixMarket' header", 1)
    obj, fmt, fld, sym = (t.lower() for t in tokens[1:5])
    if obj != "matrix" or fmt != "coordinate":
        raise ParseError(f"unsupported MatrixMarket type '{obj} {fmt}' (need 'matrix coordinate')", 1)
    if fld not in _MM_FIELDS:
        raise ParseError(f"unsupported field '{fld}'", 1)
    if sym not in _MM_SYMMETRIES:
        raise ParseError(f"unsupported symmetry '{sym}'", 1)
    rows = cols = declared = None
    idx, chunk = 1, 64
    while rows is None and idx < text.n_lines:
        for raw in text.lines(idx, idx + chunk):
            idx += 1
            line = raw.strip()
            if not line or line.startswith("%"):
                continue
            parts = line.split()
            if len(parts) != 3:
                raise ParseError("size line must be 'rows cols nnz'", idx)
            try:
                rows, cols, declared = (int(p) for p in parts)
            except ValueError:
                raise ParseError(f"malformed size line {line!r}", idx) from None
            break
        chunk *= 2
    if rows is None:
        raise ParseError("missing size line")
    if rows != cols:
        raise ParseError(f"adjacency matrix must be square, got {rows}x{cols}", idx)
    if rows < 0 or declared < 0:
        raise ParseError("negative dimension in size line", idx)
    pairs, err, status, _ = text.parse(idx, 1, rows, declared)
    if err >= 0:
        lineno = err + 1
        if status == 6:
            raise ParseError(f"more than the declared {declared} entries", lineno)
        line = text.lines(err, err + 1)[0].strip()
        parts = line.split()
        if status == 2:
            raise ParseError("coordinate entry needs at least 'i j'", lineno)
        if status == 3:
            raise ParseError(f"malformed coordinate entry {line!r}", lineno)
        i, j = int(parts[0]), int(parts[1])
        raise ParseError(f"index ({i}, {j}) outside declared {rows}x{cols}", lineno)
    if pairs.shape[0] != declared:
        raise ParseError(f"declared {declared} entries but found {pairs.shape[0]}")
    return _graph_from_device_pairs(pairs, rows, False)


def read_graph(path: str, fmt: str = "auto") -> Graph:
    """cli.load_graph (cli.py:185-203) from the file's bytes: format sniffed from the
    extension or a '%%MatrixMarket' head, then the device parser."""
    data = np.fromfile(path, dtype=np.uint8)
    if fmt == "auto":
        head = bytes(data[:1024]).decode("utf-8", "ignore").replace("\r\n", "\n").replace("\r", "\n")
        fmt = "mtx" if path.endswith(".mtx") or head[:128].lstrip().startswith("%%MatrixMarket") \
            else "edgelist"
    return parse_matrix_market(data) if fmt == "mtx" else parse_edge_list(data)


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


def device_k_neighborhood(dg: DeviceGraph, source: int, k: int
                          ) -> tuple[torch.Tensor, torch.Tensor]:
    """One source's (ids, dists) row, (dist, id)-sorted: drg_khop_source (K1's
    global-memory tier on one source)."""
    n = dg.node_count
    cnt = _lib.out_i64()
    st = _lib.stream_ptr()
    _lib.call("drg_khop_source", _lib.ptr(dg.indptr), _lib.ptr(dg.indices), n, k, int(source),
              None, None, 0, _lib.byref(cnt), st)
    m = cnt.value
    ids = torch.empty(max(m, 1), dtype=torch.int32, device=dg.indptr.device)
    dists = torch.empty(max(m, 1), dtype=torch.int32, device=dg.indptr.device)
    if m:
        _lib.call("drg_khop_source", _lib.ptr(dg.indptr), _lib.ptr(dg.indices), n, k, int(source),
                  _lib.ptr(ids), _lib.ptr(dists), m, _lib.byref(cnt), st)
    return ids[:m], dists[:m]


def bfs_k_neighborhood(g: Graph, source: int, k: int) -> list[tuple[int, int]]:
    """All nodes within k hops of ``source`` with their exact hop distance, sorted by
    (distance, id), the source excluded (graph.py:280-305), on the device."""
    if not 0 <= source < g.node_count:
        raise ValueError(f"source {source} out of range for {g.node_count} nodes")
    if k < 1:
        raise ValueError("k must be >= 1")
    _lib.load()
    ids, dists = device_k_neighborhood(DeviceGraph.from_host(g), source, k)
    return [(int(i), int(d)) for i, d in zip(ids.cpu().tolist(), dists.cpu().tolist())]


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
