"""One-off kernel parity on the full-size BASELINE C5 graph (R-MAT scale 24): the
hierarchy with 5 forced levels bit-exact against the oracle (multilevel.py:95-113)
and the k=1 closed-form P within 1e-5.  tests/test_gpu_config_parity.py runs the
same check at scale 22; this is the minutes-long full-size run.

    python scripts/config_parity.py [scale]     -> one JSON line
"""

from __future__ import annotations

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402


def main(scale: int = 24) -> None:
    import paper_2008_07799_b200 as B
    from paper_2008_07799_b200 import synthetic
    from paper_2008_07799_b200.optimizer import _HIERARCHY_TAG, _derive_seed
    gh = synthetic.rmat(scale, 16, seed=0, device="host")
    og, bg = O.Graph(gh.indptr, gh.indices), B.Graph(gh.indptr, gh.indices)
    out = {"workload": f"rmat{scale}", "nodes": og.node_count, "entries": int(len(og.indices))}
    seed = _derive_seed(0, _HIERARCHY_TAG)
    t0 = time.perf_counter()
    want = O.build_hierarchy(og, 0.8, 16, seed, max_levels=5, force_levels=5)
    out["oracle_hierarchy_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    got = B.build_hierarchy(bg, 0.8, 16, seed, max_levels=5, force_levels=5)
    out["gpu_hierarchy_s"] = time.perf_counter() - t0
    out["levels"] = [lv.node_count for lv in want.levels]
    out["maps_equal"] = [bool(np.array_equal(a, b)) for a, b in zip(got.maps, want.maps)]
    out["coarse_csr_equal"] = [bool(np.array_equal(a.indptr, b.indptr)
                                    and np.array_equal(a.indices, b.indices))
                               for a, b in zip(got.levels[1:], want.levels[1:])]
    del want, got
    nd = O.all_k_neighborhoods(og, 1)
    ns_want = O.build_sparse_similarity(nd, "auto")
    ns_got = B.build_sparse_similarity(B.all_k_neighborhoods(bg, 1), B.SimilarityParams(k=1))
    rel = np.abs(ns_got.weights - ns_want.weights) / np.maximum(np.abs(ns_want.weights), 1e-300)
    out["p_targets_equal"] = bool(np.array_equal(ns_got.targets, ns_want.targets))
    out["p_max_rel_err"] = float(rel.max()) if rel.size else 0.0
    out["ok"] = all(out["maps_equal"]) and all(out["coarse_csr_equal"]) and \
        out["p_targets_equal"] and out["p_max_rel_err"] <= 1e-5
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
