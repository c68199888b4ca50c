"""Shared fixtures.  The `gpu` marker gates tests that need a B200 (run with -m gpu)."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


def golden_graph(golden, name):
    from oracle.oracle import Graph
    return Graph(golden[f"g/{name}/indptr"], golden[f"g/{name}/indices"])


GRAPH_NAMES = ["p5", "star4", "iso", "grid17", "r60", "r200", "r500", "dense80"]
