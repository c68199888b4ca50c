"""Ingestion throughput: an edge-list / MatrixMarket text of the C4 mesh (22 M edges)
parsed to the canonical CSR on the device (read_graph path: bytes -> HBM -> lines ->
ids -> remap -> from_edges), device-timed per stage with CUDA events, against the
oracle restatement of the reference's Python loop (graph.py:134-167) on a 1 M-line
sample.  Diagnostics / profiles only."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2008_07799_b200 as B  # noqa: E402
from oracle import oracle as O  # noqa: E402


def main(name="mesh"):
    g = bench.build_workload(name).to_host()
    e = g.edge_array()
    text = ("\n".join(f"{u} {v}" for u, v in e.tolist()) + "\n").encode()
    data = np.frombuffer(text, dtype=np.uint8)
    B.parse_edge_list(data[:100000])   # warm-up (module load, pools)
    torch.cuda.synchronize()
    walls = []
    for _ in range(3):
        t0 = time.perf_counter()
        got = B.parse_edge_list(data)
        walls.append(time.perf_counter() - t0)
    assert np.array_equal(got.indptr, g.indptr) and np.array_equal(got.indices, g.indices)
    wall = min(walls)
    sample = text[: text.index(b"\n", 12_000_000) + 1].decode()
    t0 = time.perf_counter()
    O.parse_edge_list(sample)
    cpu = time.perf_counter() - t0
    cpu_lines = sample.count("\n")
    print(json.dumps({
        "workload": f"{name} edge list", "bytes": len(text), "lines": len(e),
        "gpu_wall_s": wall, "gpu_GBps_e2e": len(text) / wall / 1e9,
        "gpu_lines_per_s": len(e) / wall,
        "cpu_oracle_lines_per_s": cpu_lines / cpu, "cpu_sample_lines": cpu_lines,
        "speedup": (len(e) / wall) / (cpu_lines / cpu)}), flush=True)


if __name__ == "__main__":
    main(*(sys.argv[1:]))
