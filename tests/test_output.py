"""Output formats (output.py:12-108, graph.py:246-250).

tests/golden/output_golden.json holds the REFERENCE's texts for write_coords
(rounding ties, signed zeros, nan/inf, large values), format_edge_list and
write_svg (default and capped/sampled styles, degenerate spans).  CPU: the oracle
restatement against them; GPU: the device formatters against them byte for byte,
and against the oracle on a large random layout.
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = json.load(open(os.path.join(HERE, "golden", "output_golden.json")))["cases"]


def _graph(mod, c):
    return mod.Graph(np.array(c["indptr"], dtype=np.int64), np.array(c["indices"], dtype=np.int32))


@pytest.mark.parametrize("case", CASES, ids=[f"{c['kind']}/{c['name']}" for c in CASES])
def test_oracle_output_matches_reference(case):
    if case["kind"] == "coords":
        got = O.write_coords(np.array(case["pos"], dtype=np.float64).reshape(-1, 2))
    elif case["kind"] == "edges":
        got = O.format_edge_list(_graph(O, case))
    else:
        got = O.write_svg(_graph(O, case), np.array(case["pos"]), seed=case["seed"], **case["style"])
    assert got == case["want"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[f"{c['kind']}/{c['name']}" for c in CASES])
def test_device_output_matches_reference(case):
    import paper_2008_07799_b200 as B
    if case["kind"] == "coords":
        got = B.write_coords(np.array(case["pos"], dtype=np.float64).reshape(-1, 2))
    elif case["kind"] == "edges":
        got = B.format_edge_list(_graph(B, case))
    else:
        got = B.write_svg(_graph(B, case), np.array(case["pos"]), B.SvgStyle(**case["style"]),
                          case["seed"])
    assert got == case["want"]


@pytest.mark.gpu
def test_device_output_large_random():
    import paper_2008_07799_b200 as B
    rng = np.random.default_rng(4)
    pos = (rng.normal(0, 30, size=(200_000, 2)).astype(np.float32)).astype(np.float64)
    pos[::97] = np.round(pos[::97] * 8) / 8          # exact binary ties at .2f
    assert B.write_coords(pos) == O.write_coords(pos)
    pairs = rng.integers(0, 200_000, size=(700_000, 2))
    g = O.from_edges(pairs, 200_000)
    bg = B.Graph(g.indptr, g.indices)
    assert B.format_edge_list(bg) == O.format_edge_list(g)
    assert B.write_svg(bg, pos, seed=5) == O.write_svg(g, pos, seed=5)
    assert B.read_coords(B.write_coords(pos)).shape == (200_000, 2)
