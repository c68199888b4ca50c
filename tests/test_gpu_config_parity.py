"""Kernel parity on the BASELINE configurations' own graphs (not only the small
golden graphs): K1 rows and hop distances bit-exact, P within 1e-5 relative and
bitwise symmetric, hierarchy maps bit-exact -- against the oracle (C restatement
of graph.py:308-366, similarity.py:216-278, multilevel.py:95-113, pinned to the
reference by tests/test_oracle_golden.py) on the box's host cores.

C2 RGG 200k k=3 and C4 mesh 120^3 k=2 are checked whole; C3 BA 1M with the
neighbour cap 256 (union P) whole; the C5 hierarchy (R-MAT, 5 forced levels) at
scale 22 (4.2 M nodes) -- the oracle's numpy coarse-graph build makes scale 24 a
minutes-long job, run once by scripts/config_parity.py (profiles/r02_config_parity_*).
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

B = pytest.importorskip("paper_2008_07799_b200")


def _graphs(gh):
    return O.Graph(gh.indptr, gh.indices), B.Graph(gh.indptr, gh.indices)


def _check_rows(got, want):
    assert np.array_equal(got.indptr, want.indptr)
    assert np.array_equal(got.ids, want.ids)
    assert np.array_equal(got.dists, want.dists)


def _check_p(got, want):
    assert np.array_equal(got.indptr, want.indptr)
    assert np.array_equal(got.targets, want.targets)
    assert np.all(np.abs(got.weights - want.weights) <= 1e-5 * np.abs(want.weights))
    # stored entries bitwise symmetric: P_ij == P_ji
    src = np.repeat(np.arange(len(got.indptr) - 1), np.diff(got.indptr))
    key = src.astype(np.int64) * (len(got.indptr) - 1) + got.targets
    mirror = got.targets.astype(np.int64) * (len(got.indptr) - 1) + src
    order = np.argsort(key, kind="stable")
    pos = order[np.searchsorted(key[order], mirror)]
    assert np.array_equal(key[pos], mirror)
    assert np.array_equal(got.weights[pos], got.weights)


@pytest.mark.parametrize("name,k,perp", [("rgg", 3, 30.0), ("mesh", 2, 50.0)])
def test_khop_and_similarity_on_config_graph(name, k, perp):
    from paper_2008_07799_b200 import synthetic
    gh = synthetic.rgg(200_000, seed=0, device="host") if name == "rgg" else \
        synthetic.mesh3d(120, device="host")
    og, bg = _graphs(gh)
    want = O.all_k_neighborhoods(og, k)
    got = B.all_k_neighborhoods(bg, k)
    _check_rows(got, want)
    ns_want = O.build_sparse_similarity(want, perp)
    del want
    ns_got = B.build_sparse_similarity(got, B.SimilarityParams(k=k, perplexity=perp))
    _check_p(ns_got, ns_want)
    assert abs(ns_got.total_mass - 1.0) <= 1e-9


def test_capped_union_similarity_on_ba_1m():
    """BASELINE C3: BA 1M (m=4), k=2, cap 256 -- capped rows bit-exact, union P."""
    from paper_2008_07799_b200 import synthetic
    og, bg = _graphs(synthetic.barabasi_albert(1_000_000, 4, seed=0, device="host"))
    want = O.all_k_neighborhoods(og, 2, cap=256)
    got = B.all_k_neighborhoods(bg, 2, cap=256)
    _check_rows(got, want)
    ns_want = O.build_capped_similarity(want, 50.0)
    ns_got = B.build_sparse_similarity(got, B.SimilarityParams(k=2, perplexity=50.0,
                                                               neighbor_cap=256))
    _check_p(ns_got, ns_want)


def test_rmat_forced_hierarchy_maps():
    """BASELINE C5's hierarchy (force_levels=5) on R-MAT scale 22: every level's map
    and coarse CSR bit-exact."""
    from paper_2008_07799_b200 import synthetic
    from paper_2008_07799_b200.optimizer import _HIERARCHY_TAG, _derive_seed
    og, bg = _graphs(synthetic.rmat(22, 16, seed=0, device="host"))
    seed = _derive_seed(0, _HIERARCHY_TAG)
    want = O.build_hierarchy(og, 0.8, 16, seed, max_levels=5, force_levels=5)
    got = B.build_hierarchy(bg, 0.8, 16, seed, max_levels=5, force_levels=5)
    assert len(got.maps) == len(want.maps) == 4
    for a, b in zip(got.maps, want.maps):
        assert np.array_equal(a, b)
    for a, b in zip(got.levels[1:], want.levels[1:]):
        assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
