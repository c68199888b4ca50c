"""CPU checks of the drop-in boundary: the C-ABI library loads and exports every
symbol include/drgraph_b200.h declares (no compute calls -- no GPU here), the
Python binding covers the same set, and the host-side parameter validation
matches the reference (similarity.py:44-53, optimizer.py:60-74)."""

from __future__ import annotations

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "drgraph_b200.h")
LIB = os.path.join(ROOT, "paper_2008_07799_b200", "libdrgraph_b200.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(drg_\w+)\s*\(", text, re.M)))


def test_header_declares_the_path():
    syms = declared_symbols()
    for name in ("drg_khop_count", "drg_khop_fill", "drg_similarity", "drg_coarsen",
                 "drg_coarse_graph", "drg_aggregate_pairs", "drg_alias_build",
                 "drg_layout_iters", "drg_prolong", "drg_layout_radius", "drg_from_edges"):
        assert name in syms


@pytest.mark.skipif(not os.path.exists(LIB), reason="extension not built")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.drg_abi_version() == 1
    lib.drg_last_error.restype = ctypes.c_char_p
    assert isinstance(lib.drg_last_error(), bytes)


def test_python_binding_covers_header():
    from paper_2008_07799_b200 import _lib
    assert set(_lib.SIGNATURES) == set(declared_symbols())


def test_python_constants_equal_the_header_macros():
    """Every DRG_SAMPLED_* flag and DRG_ERR_* status the binding uses has the value
    the header defines (a flag renumbered on one side only would silently select
    another kernel)."""
    from paper_2008_07799_b200 import _lib
    macros = {m.group(1): int(m.group(2), 0) for m in
              re.finditer(r"^#define\s+(DRG_(?:SAMPLED|ERR)_\w+)\s+\(?(-?\d+)\)?\s*$",
                          open(HEADER).read(), re.M)}
    flags = {k: v for k, v in macros.items() if k.startswith("DRG_SAMPLED_")}
    assert len(flags) >= 7 and len(set(flags.values())) == len(flags)
    assert all(v & (v - 1) == 0 for v in flags.values())   # single bits
    for name, value in macros.items():
        if hasattr(_lib, name):
            assert getattr(_lib, name) == value, name
    for name in flags:
        assert hasattr(_lib, name), name


def test_params_validation_matches_reference():
    from paper_2008_07799_b200 import OptimizerParams, SimilarityParams
    for bad in (dict(k=0), dict(k=7), dict(perplexity=0.5)):
        with pytest.raises(ValueError):
            SimilarityParams(**bad)
    for bad in (dict(gamma=-1), dict(iters=0), dict(b=0), dict(threads=0), dict(neg_samples=-1),
                dict(lr0=0), dict(seed=-1), dict(init="x"), dict(update="y")):
        with pytest.raises(ValueError):
            OptimizerParams(**bad)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2008_07799_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "oracle" not in src.replace("oracle/", ""), fn


def test_no_cpu_device_path():
    """Without a CUDA device the product raises instead of computing on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    from paper_2008_07799_b200 import Graph, all_k_neighborhoods
    g = Graph(np.array([0, 1, 2]), np.array([1, 0], dtype=np.int32))
    with pytest.raises(RuntimeError):
        all_k_neighborhoods(g, 2)


@pytest.mark.parametrize("n", [0, 1, 2, 3, 17, 1000, 65537, 300_001])
def test_level_order_is_numpy_permutation(n):
    """drg_pcg64_permutation (host routine behind multilevel.level_order) reproduces
    numpy's Generator(PCG64).permutation bit for bit -- the reference's visiting
    order (multilevel.py:91) -- including a buffered 32-bit half-word state."""
    import numpy as np
    from paper_2008_07799_b200 import _lib
    from paper_2008_07799_b200.multilevel import level_order
    for seed in (0, 7, 2**62 + 3):
        got = level_order(n, seed)
        assert got.dtype == np.int32
        assert np.array_equal(got, np.random.default_rng(seed).permutation(n))
    g = np.random.default_rng(11)
    g.integers(0, 2**32 - 1, dtype=np.uint32)   # leaves a buffered half-word
    st = g.bit_generator.state
    assert st["has_uint32"] == 1
    out = np.empty(n, dtype=np.int32)
    s, inc, m = st["state"]["state"], st["state"]["inc"], (1 << 64) - 1
    _lib.call_host("drg_pcg64_permutation", s >> 64, s & m, inc >> 64, inc & m, 1,
                   st["uinteger"], n, out.ctypes.data)
    assert np.array_equal(out, g.permutation(n))


# The reference's metrics module is out of scope except the metric the
# parity protocol uses (neighborhood_preservation, exported as the device instrument).
OUT_OF_SCOPE = {"MetricsReport", "MetricError", "stress", "count_crossings", "crosslessness",
                "minimum_angle", "compute_metrics"}


def test_public_names_and_parameters_match_the_reference():
    """Every public name of drgraph (__init__.py:57-70; tests/golden/reference_api.json,
    written by make_api_golden.py from the reference itself) on the path is exported,
    and every callable / parameter dataclass takes the reference's parameters, in the
    reference's order (B200 extensions only after them, as keyword-only or defaulted)."""
    import inspect
    import json

    import paper_2008_07799_b200 as B
    ref = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                      "reference_api.json")))
    missing = [n for n in ref["__all__"] if n not in OUT_OF_SCOPE and n not in B.__all__]
    assert not missing, missing
    for name, params in ref["params"].items():
        if name in OUT_OF_SCOPE:
            continue
        obj = getattr(B, name)
        if inspect.isclass(obj):
            ours = list(obj.__dataclass_fields__)
        else:
            ours = [p.name for p in inspect.signature(obj).parameters.values()]
        assert ours[:len(params)] == params, (name, ours, params)
