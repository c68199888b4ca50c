"""Golden cases for the text parsers, produced by the REFERENCE package (drgraph).

Run in the build container only (it needs /root/reference, read-only):

    python tests/golden/make_parse_golden.py

Writes tests/golden/parse_golden.json: every case is a source (str, a text stream,
a list of lines, or raw file bytes read the way cli.py:194 reads them) for
parse_edge_list (graph.py:134-167) or parse_matrix_market (graph.py:170-243) with
the reference's result -- the CSR, or the exception type, message and line.
"""

from __future__ import annotations

import base64
import io
import json
import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from drgraph.graph import ParseError, parse_edge_list, parse_matrix_market  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "parse_golden.json")

EDGE_TEXTS = {
    "basic": "0 1\n1 2",
    "loops_dups": "0 0\n0 1\n1 0\n2 1\n1 2\n",
    "comments": "# header\n% other\n\n0 1\n  # indented comment\n1 2\n",
    "malformed": "0 1\n1 x\n",
    "three_tokens": "0 1 2\n",
    "one_token": "0 1\n5\n",
    "negative": "0 -1\n",
    "negative_zero": "-0 3\n+1 2\n",
    "sparse_ids": "0 1000000\n1000000 2000000\n",
    "dense_ids": "0 3\n3 4\n1 2\n",
    "tabs_spaces": "\t0\t\t1  \n   2 \t 1\t\n",
    "crlf": "0 1\r\n1 2\r\n2 3\r\n",
    "cr_only": "0 1\r1 2\r2 3",
    "vt_ff_breaks": "0 1\x0b1 2\x0c2 3",
    "sep_breaks": "0 1\x1c1 2\x1d2 3\x1e3 4",
    "unit_sep_space": "0\x1f1\n",
    "unicode_spaces": "0\u00a01\n1\u30002\n2\u20093\n3\u202f4\n",
    "unicode_breaks": "0 1\u20281 2\u20292 3\u00853 4",
    "fullwidth_digits": "\uff11 \uff12\n\uff12 \uff13\n",
    "arabic_digits": "\u0663 \u0664\n\u0661\u0662 3\n",
    "underscores": "1_0 2_0\n1_000 10\n",
    "double_underscore": "1__0 2\n",
    "leading_underscore": "_1 2\n",
    "trailing_underscore": "1_ 2\n",
    "sign_alone": "+ 1\n",
    "big_positive": "99999999999999999999 1\n",
    "big_negative": "-99999999999999999999 1\n",
    "int64_max": "9223372036854775807 0\n",
    "empty": "",
    "only_comments": "# nothing\n% here\n",
    "only_blank": "\n\n   \n",
    "bom": "\ufeff0 1\n1 2\n",
    "hash_inside": "0 1 # trailing comment\n",
    "error_after_blanks": "0 1\n\n\n2 x\n",
    "leading_zeros": "007 010\n",
    "first_error_wins": "0 1 2\n1 x\n",
    "non_ascii_token": "0 1\n\u00e9 2\n",
    "hex": "0x1 2\n",
    "float": "1.0 2\n",
    "trailing_break_pair": "0 1\n\r\n",
}

MM_TEXTS = {
    "pattern_symmetric": "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 2\n2 1\n3 2\n",
    "real_general_diag": ("%%MatrixMarket matrix coordinate real general\n% note\n4 4 5\n"
                          "1 1 2.5\n1 2 1.0\n2 3 -1\n4 4 0.5\n3 4 7e3\n"),
    "complex_columns": "%%MatrixMarket matrix coordinate complex hermitian\n2 2 1\n2 1 0.5 -0.5\n",
    "uppercase_header": "%%MatrixMarket MATRIX Coordinate Pattern General\n2 2 1\n1 2\n",
    "missing_header": "3 3 2\n2 1\n3 2\n",
    "array_object": "%%MatrixMarket matrix array real general\n3 3 1\n1 2\n",
    "bad_field": "%%MatrixMarket matrix coordinate text general\n2 2 1\n1 2\n",
    "bad_symmetry": "%%MatrixMarket matrix coordinate pattern lower\n2 2 1\n1 2\n",
    "short_header": "%%MatrixMarket matrix coordinate\n2 2 1\n1 2\n",
    "blank_first_line": "\n%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 2\n",
    "out_of_range": "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n4 1\n",
    "zero_index": "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n0 1\n",
    "huge_index": "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n99999999999999999999 1\n",
    "fewer_entries": "%%MatrixMarket matrix coordinate pattern general\n3 3 2\n1 2\n",
    "more_entries": "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n1 2\n2 3\n",
    "more_and_malformed": "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n1 2\n1 x\n",
    "size_two_parts": "%%MatrixMarket matrix coordinate pattern general\n3 3\n1 2\n",
    "size_malformed": "%%MatrixMarket matrix coordinate pattern general\n3 x 2\n1 2\n",
    "non_square": "%%MatrixMarket matrix coordinate pattern general\n3 4 1\n1 2\n",
    "negative_dims": "%%MatrixMarket matrix coordinate pattern general\n-1 -1 0\n",
    "entry_one_part": "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n2\n",
    "entry_malformed": "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n1 x\n",
    "empty_file": "",
    "header_only": "%%MatrixMarket matrix coordinate pattern general\n% c\n",
    "comments_between": ("%%MatrixMarket matrix coordinate pattern general\r\n% a\r\n\r\n"
                         "3 3 2\r\n% b\r\n1 2\r\n\r\n2 3\r\n"),
    "unicode_digits": "%%MatrixMarket matrix coordinate pattern general\n3 3 2\n\uff11 \uff12\n2_0 3\n",
    "empty_matrix": "%%MatrixMarket matrix coordinate pattern general\n0 0 0\n",
    "underscore_size": "%%MatrixMarket matrix coordinate pattern general\n1_0 1_0 1\n10 1\n",
}

RAW_FILES = {   # bytes of a file, read as cli.py:194 reads it
    "el_crlf_file": ("el", b"0 1\r\n1 2\r\n# c\r\n2 3"),
    "el_utf8_file": ("el", "0 1\n\uff12 \uff13\n\u0663\u3000\u0661\u2028".encode()),
    "el_invalid_utf8": ("el", b"0 1\n1 \xff2\n"),
    "el_truncated_utf8": ("el", b"0 1\n1 2\xe2\x80"),
    "el_overlong": ("el", b"0 1\n\xc0\xb1 2\n"),
    "el_surrogate": ("el", b"0 1\n\xed\xa0\x80 2\n"),
    "mm_file": ("mm", b"%%MatrixMarket matrix coordinate pattern general\r\n3 3 2\r\n1 2\r\n2 3\r\n"),
}


def run(fn, src):
    try:
        g = fn(src)
        return {"indptr": g.indptr.tolist(), "indices": g.indices.tolist()}
    except ParseError as e:
        return {"error": "ParseError", "message": str(e), "line": e.line}
    except (OverflowError, UnicodeDecodeError, ValueError) as e:
        return {"error": type(e).__name__, "message": str(e), "line": None}


def random_edge_text(seed, lines=3000):
    rng = np.random.default_rng(seed)
    ws = [" ", "\t", "  ", "\u2009", "\u3000", " \t", "\xa0"]
    out = []
    for _ in range(lines):
        r = rng.random()
        if r < 0.05:
            out.append("# comment " + str(int(rng.integers(0, 99))))
        elif r < 0.08:
            out.append("   ")
        else:
            u, v = rng.integers(0, 400, size=2)
            a = ws[int(rng.integers(0, len(ws)))]
            b = ws[int(rng.integers(0, len(ws)))]
            out.append(f"{a}{u}{b}{v}")
    brk = ["\n", "\r\n", "\r", "\n"]
    return "".join(line + brk[int(rng.integers(0, len(brk)))] for line in out)


def main():
    cases = []
    for name, text in EDGE_TEXTS.items():
        cases.append({"name": f"el/{name}/str", "kind": "el", "source": "str", "text": text,
                      "want": run(parse_edge_list, text)})
        cases.append({"name": f"el/{name}/stream", "kind": "el", "source": "stream",
                      "text": text, "want": run(parse_edge_list, io.StringIO(text))})
        lines = text.split("\n")
        cases.append({"name": f"el/{name}/list", "kind": "el", "source": "list", "lines": lines,
                      "want": run(parse_edge_list, lines)})
    for name, text in MM_TEXTS.items():
        cases.append({"name": f"mm/{name}/str", "kind": "mm", "source": "str", "text": text,
                      "want": run(parse_matrix_market, text)})
        cases.append({"name": f"mm/{name}/stream", "kind": "mm", "source": "stream",
                      "text": text, "want": run(parse_matrix_market, io.StringIO(text))})
    for seed in range(3):
        text = random_edge_text(seed)
        cases.append({"name": f"el/random{seed}/str", "kind": "el", "source": "str",
                      "text": text, "want": run(parse_edge_list, text)})
    with tempfile.TemporaryDirectory() as d:
        for name, (kind, data) in RAW_FILES.items():
            path = os.path.join(d, "g.txt")
            with open(path, "wb") as f:
                f.write(data)
            fn = parse_edge_list if kind == "el" else parse_matrix_market

            def from_file(_, path=path, fn=fn):
                with open(path, "r", encoding="utf-8") as fh:   # cli.py:194
                    return fn(fh.read())
            cases.append({"name": f"{kind}/{name}/bytes", "kind": kind, "source": "bytes",
                          "b64": base64.b64encode(data).decode(), "want": run(from_file, None)})
    with open(OUT, "w") as f:
        json.dump({"generator": "tests/golden/make_parse_golden.py", "cases": cases}, f,
                  ensure_ascii=True, indent=0)
    print(OUT, len(cases), "cases")


if __name__ == "__main__":
    main()
