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
