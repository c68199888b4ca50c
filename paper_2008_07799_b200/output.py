"""Coordinate-file, edge-list and SVG emission formatted on the device (drop-in for
drgraph.output, output.py:1-108, and graph.format_edge_list, graph.py:246-250).

The texts are byte-identical to the reference's: the records are formatted by
output.cu (Python's round-half-even fixed-point formatting, the same IEEE operation
order for the SVG geometry), the host only joins the header lines and draws the SVG
edge sample with the reference's numpy stream.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .graph import Graph


def _emit(entry: str, *args, bad_out: bool = True) -> tuple[bytes, int]:
    """Size pass, allocation, write pass of a drg_format_* entry."""
    n_bytes = _lib.out_i64()
    bad = _lib.out_i64()
    tail = [_lib.byref(bad)] if bad_out else []
    _lib.call(entry, *args, None, _lib.byref(n_bytes), *tail, _lib.stream_ptr())
    buf = torch.empty(max(n_bytes.value, 1), dtype=torch.uint8, device="cuda")
    _lib.call(entry, *args, _lib.ptr(buf), _lib.byref(n_bytes), *tail, _lib.stream_ptr())
    return buf[:n_bytes.value].cpu().numpy().tobytes(), (bad.value if bad_out else -1)


def _positions(positions) -> torch.Tensor:
    if isinstance(positions, torch.Tensor):
        return positions.to(device="cuda", dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(positions, dtype=np.float64)).cuda()


def write_coords(positions) -> str:
    """One "x y" line per node after a "#nodes N" header, 6 decimals (output.py:12-17)."""
    _lib.load()
    pos = _positions(positions).reshape(-1, 2)
    n = pos.shape[0]
    body, bad = _emit("drg_format_coords", _lib.ptr(pos), n)
    if bad >= 0:   # |coordinate| >= 2^50 / 1e6: rows the device does not format
        raise ValueError(f"coordinate of node {bad} too large for fixed-point output")
    return f"#nodes {n}\n" + body.decode("ascii")


def read_coords(text: str) -> np.ndarray:
    """Inverse of write_coords (output.py:20-29)."""
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines or not lines[0].startswith("#nodes"):
        raise ValueError("missing '#nodes N' header")
    n = int(lines[0].split()[1])
    rows = [tuple(map(float, ln.split())) for ln in lines[1:]]
    if len(rows) != n:
        raise ValueError(f"header says {n} nodes, found {len(rows)} lines")
    return np.array(rows, dtype=np.float64).reshape(n, 2)


def format_edge_list(g: Graph) -> str:
    """graph.py:246-250: "u v" per edge (u < v, CSR order), newline-terminated."""
    _lib.load()
    if len(g.indices) == 0:
        return ""
    ip = torch.from_numpy(np.asarray(g.indptr, dtype=np.int64)).cuda()
    ix = torch.from_numpy(np.asarray(g.indices, dtype=np.int32)).cuda()
    body, _ = _emit("drg_format_edge_list", _lib.ptr(ip), _lib.ptr(ix), g.node_count,
                    ix.numel(), bad_out=False)
    return body.decode("ascii")


@dataclass
class SvgStyle:
    """Rendering knobs (output.py:32-42)."""

    canvas: int = 1000
    margin: float = 20.0
    node_radius: float = 2.0
    edge_width: float = 1.0
    edge_cap: int = 600_000


def write_svg(g: Graph, positions, style: SvgStyle | None = None, seed: int = 0) -> str:
    """The layout as an SVG document, nodes above edges (output.py:56-108)."""
    _lib.load()
    style = style or SvgStyle()
    pos = _positions(positions).reshape(-1, 2)
    n = pos.shape[0]
    size = float(style.canvas)
    inner = size - 2.0 * style.margin
    head = (f'<svg xmlns="http://www.w3.org/2000/svg" width="{style.canvas}" '
            f'height="{style.canvas}" viewBox="0 0 {style.canvas} {style.canvas}">\n'
            f'<rect width="{style.canvas}" height="{style.canvas}" fill="white"/>\n')
    if n == 0:
        return head + "</svg>\n"
    bbox = (ctypes.c_double * 4)()
    _lib.call("drg_bbox2", _lib.ptr(pos), n, bbox, _lib.stream_ptr())
    mins = np.array([bbox[0], bbox[1]])
    spans = np.array([bbox[2], bbox[3]]) - mins
    span = float(spans.max())
    scale = inner / span if span > 0 else 0.0
    offset = style.margin + (inner - spans * scale) / 2.0
    # edges u < v in CSR order; above the cap the reference's seeded sample
    # (output.py:82-86), drawn with numpy's own stream on the host
    ip = np.asarray(g.indptr, dtype=np.int64)
    ix = np.asarray(g.indices, dtype=np.int32)
    src = np.repeat(np.arange(g.node_count, dtype=np.int32), np.diff(ip))
    keep = src < ix
    edges = np.column_stack([src[keep], ix[keep]])
    if len(edges) > style.edge_cap:
        rng = np.random.default_rng(seed)
        pick = np.sort(rng.choice(len(edges), size=style.edge_cap, replace=False))
        edges = edges[pick]
    m = len(edges)
    ed = torch.from_numpy(np.ascontiguousarray(edges, dtype=np.int32)).cuda() if m else \
        torch.empty((1, 2), dtype=torch.int32, device="cuda")
    line_tail = f'" stroke-width="{style.edge_width}"/>'.encode()
    circle_tail = f'" r="{style.node_radius}" fill="black"/>'.encode()
    args = (_lib.ptr(pos), n, _lib.ptr(ed), m, float(mins[0]), float(mins[1]),
            float(offset[0]), float(offset[1]), float(scale), size, line_tail, circle_tail)
    lens = [_lib.out_i64(), _lib.out_i64()]
    bad = _lib.out_i64()
    _lib.call("drg_format_svg", *args, None, _lib.byref(lens[0]), None, _lib.byref(lens[1]),
              _lib.byref(bad), _lib.stream_ptr())
    if bad.value >= 0:
        raise ValueError("SVG coordinate too large for fixed-point output")
    lines = torch.empty(max(lens[0].value, 1), dtype=torch.uint8, device="cuda")
    circles = torch.empty(max(lens[1].value, 1), dtype=torch.uint8, device="cuda")
    _lib.call("drg_format_svg", *args, _lib.ptr(lines), _lib.byref(lens[0]), _lib.ptr(circles),
              _lib.byref(lens[1]), _lib.byref(bad), _lib.stream_ptr())
    body = (lines[:lens[0].value].cpu().numpy().tobytes()
            + circles[:lens[1].value].cpu().numpy().tobytes())
    return head + body.decode("ascii") + "</svg>\n"
