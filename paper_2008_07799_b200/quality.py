"""Layout-quality instruments on the device.

``kl_divergence`` evaluates KL(P || Q) with the reference's unnormalised t-kernel
(lp_kernel, optimizer.py:150-152) in one C-ABI call (drg_kl_terms): exact Z by a
tiled all-pairs kernel (n up to a few million), or a Monte-Carlo Z.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _lib
from .graph import DeviceGraph, Graph, device_k_neighborhoods
from .similarity import DeviceSimilarity, SparseSimilarity


def kl_divergence(ns: SparseSimilarity | DeviceSimilarity, positions, b: int = 2,
                  z_pairs: int | None = None, seed: int = 0) -> float:
    """KL(P || Q) = sum P log P + sum P log(1 + d^(2b)) + log Z (normalised by
    sum P).  ``z_pairs`` None = exact Z."""
    _lib.load()
    if isinstance(ns, SparseSimilarity):
        ip = torch.from_numpy(np.ascontiguousarray(ns.indptr, dtype=np.int64)).cuda()
        tg = torch.from_numpy(np.ascontiguousarray(ns.targets, dtype=np.int32)).cuda()
        w = torch.from_numpy(np.ascontiguousarray(ns.weights, dtype=np.float64)).cuda()
    else:
        ip, tg, w = ns.indptr, ns.targets, ns.weights
    if isinstance(positions, torch.Tensor):
        y = positions.to(device="cuda", dtype=torch.float32).contiguous()
    else:
        y = torch.from_numpy(np.ascontiguousarray(positions, dtype=np.float32)).cuda()
    n = y.shape[0]
    out = (ctypes.c_double * 4)()
    _lib.call("drg_kl_terms", _lib.ptr(ip), _lib.ptr(tg), _lib.ptr(w), n, _lib.ptr(y), int(b),
              int(z_pairs or 0), int(seed), out, _lib.stream_ptr())
    return (out[0] + out[1]) / max(out[2], 1e-300) + math.log(out[3])


def neighborhood_preservation(g: Graph | DeviceGraph, positions, k_eval: int = 2,
                              sample=None) -> float:
    """metrics.py:114-145 on the device: mean Jaccard between each node's
    k_eval-hop set and its equally sized exact layout k-NN (ties to the lower id).
    ``sample``: evaluate on these node ids only."""
    if k_eval < 1:
        raise ValueError("k_eval must be >= 1")
    _lib.load()
    dg = g if isinstance(g, DeviceGraph) else DeviceGraph.from_host(g)
    n = dg.node_count
    if len(positions) != n:   # metrics.py:126-127
        raise ValueError("layout does not cover all nodes")
    if isinstance(positions, torch.Tensor):
        y = positions.to(device="cuda", dtype=torch.float32).contiguous()
    else:
        y = torch.from_numpy(np.ascontiguousarray(positions, dtype=np.float32)).cuda()
    if y.shape[0] != n:
        raise ValueError("layout does not cover all nodes")
    if n < 2:
        return 1.0
    nd = device_k_neighborhoods(dg, k_eval)
    q = None
    nq = n
    if sample is not None:
        q = torch.as_tensor(np.asarray(sample, dtype=np.int32)).cuda()
        nq = q.numel()
    out = torch.empty(max(nq, 1), dtype=torch.float64, device="cuda")
    _lib.call("drg_neighborhood_preservation", _lib.ptr(y), n, _lib.ptr(nd.indptr),
              _lib.ptr(nd.ids), _lib.ptr(q), nq, _lib.ptr(out), _lib.stream_ptr())
    scores = out[:nq]
    if bool((scores < 0).any()):
        raise RuntimeError("a hop set exceeds the device k-NN capacity (3584)")
    return float(scores.mean())
