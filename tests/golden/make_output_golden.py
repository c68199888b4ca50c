"""Golden texts of the output formats, produced by the REFERENCE package (drgraph).

Run in the build container only (it needs /root/reference, read-only):

    python tests/golden/make_output_golden.py

Writes tests/golden/output_golden.json: positions (float64, exact JSON round trip)
and graphs with the reference's write_coords (output.py:12-17), write_svg
(output.py:56-108, including the capped edge sample) and format_edge_list
(graph.py:246-250) texts.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from drgraph.graph import format_edge_list, from_edges  # noqa: E402
from drgraph.output import SvgStyle, write_coords, write_svg  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "output_golden.json")


def tie_positions():
    """Values at and around the rounding boundaries of %.6f, signs, zeros, specials."""
    vals = [0.0, -0.0, 5e-7, -5e-7, 1.5e-6, 2.5e-6, 0.0000005, 1.0000005, 2.0000025, -3.0000035,
            0.1234565, 0.1234575, 123456.7890125, 1e-300, -1e-300, 7.25, -7.25, 1e8 + 0.5e-6,
            999999.9999995, -999999.9999995, 3.141592653589793, float("nan"), float("inf"),
            float("-inf"), 0.5, 1.5, 2.5, 0.125, 0.375, 4503599.6274, 1e9]
    v = np.array(vals + [0.0] * (len(vals) % 2), dtype=np.float64)
    return v.reshape(-1, 2)


def main():
    rng = np.random.default_rng(11)
    coords = {
        "ties": tie_positions(),
        "normal": rng.normal(0, 50, size=(500, 2)),
        "float32_values": rng.normal(0, 3, size=(300, 2)).astype(np.float32).astype(np.float64),
        "grid_halves": (np.arange(200, dtype=np.float64).reshape(100, 2) / 8.0 - 7.0),
        "empty": np.zeros((0, 2)),
    }
    cases = []
    for name, pos in coords.items():
        cases.append({"kind": "coords", "name": name, "pos": pos.tolist(),
                      "want": write_coords(pos)})
    graphs = {}
    pairs = rng.integers(0, 300, size=(900, 2))
    graphs["r300"] = (from_edges(pairs, 300), rng.normal(0, 10, size=(300, 2)))
    graphs["path"] = (from_edges(np.array([[0, 1], [1, 2], [2, 3]]), 4),
                      np.array([[0.0, 0.0], [1.0, 0.0], [2.0, 0.5], [3.0, 0.25]]))
    graphs["one_edge"] = (from_edges(np.array([[0, 1]]), 2), np.array([[0.0, 0.0], [1.0, 1.0]]))
    graphs["same_point"] = (from_edges(np.array([[0, 1], [1, 2]]), 3), np.ones((3, 2)))
    graphs["single_node"] = (from_edges(np.zeros((0, 2), dtype=np.int64), 1), np.array([[2.0, 3.0]]))
    graphs["tall"] = (from_edges(np.array([[0, 1], [1, 2]]), 3),
                      np.array([[0.0, 0.0], [0.1, 5.0], [0.05, 10.0]]))
    for name, (g, pos) in graphs.items():
        cases.append({"kind": "edges", "name": name, "indptr": g.indptr.tolist(),
                      "indices": g.indices.tolist(), "want": format_edge_list(g)})
        cases.append({"kind": "svg", "name": name, "indptr": g.indptr.tolist(),
                      "indices": g.indices.tolist(), "pos": pos.tolist(), "style": {},
                      "seed": 0, "want": write_svg(g, pos)})
    g, pos = graphs["r300"]
    style = dict(canvas=640, margin=7.5, node_radius=1.5, edge_width=0.5, edge_cap=100)
    for seed in (0, 3):
        cases.append({"kind": "svg", "name": f"r300_capped_seed{seed}", "indptr": g.indptr.tolist(),
                      "indices": g.indices.tolist(), "pos": pos.tolist(), "style": style,
                      "seed": seed, "want": write_svg(g, pos, SvgStyle(**style), seed)})
    with open(OUT, "w") as f:
        json.dump({"generator": "tests/golden/make_output_golden.py", "cases": cases}, f)
    print(OUT, len(cases), "cases")


if __name__ == "__main__":
    main()
