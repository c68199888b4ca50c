"""Text ingestion parity (graph.py:128-243).

tests/golden/parse_golden.json holds the REFERENCE's own results (CSR, or exception
type / message / line) for edge-list and MatrixMarket sources given as a str, a text
stream, a list of lines and raw file bytes -- every line-break and whitespace class
of str.splitlines / str.split, Unicode digits and underscores for int(), every
ParseError of the two parsers, UTF-8 errors.  CPU: the oracle restatement against
the golden cases.  GPU: the device parsers against the golden cases and against
the oracle on large random texts.
"""
import base64
import io
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = json.load(open(os.path.join(HERE, "golden", "parse_golden.json")))["cases"]


def _source(case, raw_bytes_ok):
    if case["source"] == "str":
        return case["text"]
    if case["source"] == "stream":
        return io.StringIO(case["text"])
    if case["source"] == "list":
        return list(case["lines"])
    data = base64.b64decode(case["b64"])
    if raw_bytes_ok:
        return data
    # what cli.py:194 hands the parser: the file decoded with universal newlines
    return data.decode("utf-8").replace("\r\n", "\n").replace("\r", "\n")


def _outcome(fn, src, parse_error):
    try:
        g = fn(src)
        return {"indptr": np.asarray(g.indptr).tolist(), "indices": np.asarray(g.indices).tolist()}
    except parse_error as e:
        return {"error": "ParseError", "message": str(e), "line": e.line}
    except (OverflowError, UnicodeDecodeError, ValueError) as e:
        return {"error": type(e).__name__, "message": str(e), "line": None}


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_parsers_match_reference(case):
    fn = O.parse_edge_list if case["kind"] == "el" else O.parse_matrix_market
    try:
        src = _source(case, raw_bytes_ok=False)
    except UnicodeDecodeError as e:
        assert case["want"] == {"error": "UnicodeDecodeError", "message": str(e), "line": None}
        return
    assert _outcome(fn, src, O.OracleParseError) == case["want"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_device_parsers_match_reference(case):
    import paper_2008_07799_b200 as B
    fn = B.parse_edge_list if case["kind"] == "el" else B.parse_matrix_market
    assert _outcome(fn, _source(case, raw_bytes_ok=True), B.ParseError) == case["want"]


def _random_edge_text(rng, lines, id_max, unicode=True):
    ws = [" ", "\t", "  ", " \t "] + (["\u2009", "\u3000", "\x1f"] if unicode else [])
    brk = ["\n", "\r\n", "\r"] + (["\x0b", "\u2028", "\x85"] if unicode else [])
    out = []
    for _ in range(lines):
        r = rng.random()
        if r < 0.03:
            out.append("# c")
        elif r < 0.05:
            out.append(" ")
        else:
            u, v = rng.integers(0, id_max, size=2)
            out.append(ws[rng.integers(len(ws))] + str(u) + ws[rng.integers(len(ws))] + str(v))
        out.append(brk[rng.integers(len(brk))])
    return "".join(out)


@pytest.mark.gpu
@pytest.mark.parametrize("seed,lines,id_max", [(0, 200_000, 50_000), (1, 100_000, 10**9),
                                               (2, 50_000, 300)])
def test_device_edge_list_large_random(seed, lines, id_max):
    import paper_2008_07799_b200 as B
    text = _random_edge_text(np.random.default_rng(seed), lines, id_max)
    want = O.parse_edge_list(text)
    got = B.parse_edge_list(text)
    assert np.array_equal(got.indptr, want.indptr) and np.array_equal(got.indices, want.indices)
    # the same text as raw file bytes (what read_graph streams to the device)
    got_b = B.parse_edge_list(text.encode())
    assert np.array_equal(got_b.indptr, want.indptr) and np.array_equal(got_b.indices, want.indices)


@pytest.mark.gpu
def test_device_error_line_in_large_text():
    import paper_2008_07799_b200 as B
    rng = np.random.default_rng(5)
    rows = [f"{u} {v}" for u, v in rng.integers(0, 1000, size=(100_000, 2))]
    rows[73_123] = "12 x"
    rows[90_000] = "1 2 3"
    with pytest.raises(B.ParseError) as e:
        B.parse_edge_list("\n".join(rows))
    assert e.value.line == 73_124 and str(e.value) == "line 73124: malformed integer in ['12', 'x']"


@pytest.mark.gpu
def test_read_graph_files(tmp_path):
    import paper_2008_07799_b200 as B
    rng = np.random.default_rng(9)
    pairs = rng.integers(0, 5000, size=(30_000, 2))
    el = tmp_path / "g.txt"
    el.write_text("# edges\n" + "\n".join(f"{u}\t{v}" for u, v in pairs) + "\n")
    want = O.parse_edge_list(el.read_text())
    got = B.read_graph(str(el))
    assert np.array_equal(got.indptr, want.indptr) and np.array_equal(got.indices, want.indices)
    mm = tmp_path / "g.mtx"
    mm.write_text("%%MatrixMarket matrix coordinate pattern general\n" + f"5000 5000 {len(pairs)}\n"
                  + "\n".join(f"{u + 1} {v + 1}" for u, v in pairs) + "\n")
    want = O.parse_matrix_market(mm.read_text())
    got = B.read_graph(str(mm))
    assert np.array_equal(got.indptr, want.indptr) and np.array_equal(got.indices, want.indices)
