"""Multi-GPU sampled epochs: one process per GPU, one distributed Y.

The reference runs Hogwild workers over ONE shared position array
(optimizer.py:325-345).  Here that array is partitioned by node range across the
ranks of a process group: rank r owns rows [bounds[r], bounds[r+1]) of a level in
a buffer every peer maps through CUDA IPC (NVLink / NVSwitch), and runs the steps
whose SOURCE it owns -- n_l R(segment) / R of each epoch, sources drawn from its
segment of the level-0 nodes (through the composed parent map on coarse levels,
the reference's draw-then-map, _kernels.py:76-81).  The source and the attraction
partner are read and moved in place through the peer table (a cut edge is a remote
load and remote atomics); the M negatives are read from a replicated snapshot of
the epoch-start positions and their reactions summed into a delta array, which one
reduce-scatter + all-gather per epoch (NCCL over NVLink, inside the library:
drg_shard_exchange) folds in and redistributes.  Only the weak long-range
repulsion of the negatives sees epoch-start positions; attraction -- the local
structure NP measures -- stays live Hogwild on the one array.

One GPU emulates W ranks (``OptimizerParams.virtual_ranks``): all W parts local,
every rank's draws into one buffer and all steps in ONE apply launch -- the same
kernels and addressing, no rank waiting on another (B200_PROFILING.md), and, since
the deferred-negative law does not depend on W, the fidelity emulation of any W.
The CUDA side is the drg_shard_* family of include/drgraph_b200.h.
"""

from __future__ import annotations

import ctypes
import logging
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

MAX_PARTS = 8
log = logging.getLogger("drgraph")


@dataclass
class ShardLayout:
    """Partition of one level over W ranks (host-side plan, CPU-testable)."""

    n: int
    bounds: list            # W + 1 node bounds of the parts (level-l ids)
    perm: torch.Tensor | None   # level-0 ids sorted by their level-l image (None: level 0)
    seg_lo: list            # per rank: first index of its segment (into perm / ids)
    seg_n: list             # per rank: items of its segment
    step_lo: list           # per rank: first global step id of its share of an epoch
    n_steps: list           # per rank: steps per epoch
    seg_mass: list          # per rank: R mass of its segment

    @property
    def world(self) -> int:
        return len(self.bounds) - 1

    @property
    def pad(self) -> int:
        return max(1, max(b - a for a, b in zip(self.bounds, self.bounds[1:])))


def shard_layout(mass_l: torch.Tensor, world: int, mass0: torch.Tensor | None = None,
                 map_l: torch.Tensor | None = None) -> ShardLayout:
    """Node-range parts of a level and each rank's source segment and step share.

    Parts are cut where the prefix of (R_v / R + 1 / n) crosses multiples of 2 / W:
    ranks get equal shares of an epoch's steps (R mass: steps are drawn ~ R) and of
    the exchange (node count: the padded all-gather moves W x the longest part).
    Rank r's sources are the level-0 nodes whose level-l image it owns (level 0:
    its own range); its steps per epoch are n_l times its share of R, rounded on
    the cumulative sum so the shares add up to n_l exactly."""
    if not 1 <= world <= MAX_PARTS:
        raise ValueError(f"world must be in [1, {MAX_PARTS}]")
    n = int(mass_l.numel())
    m = mass_l.to(torch.float64)
    total = float(m.sum())
    if total > 0:
        cost = m / total + 1.0 / max(n, 1)
    else:
        cost = torch.full_like(m, 1.0 / max(n, 1))
    cum = torch.cumsum(cost, 0)
    marks = cum[-1] * torch.arange(1, world, dtype=torch.float64, device=cum.device) / world \
        if n else torch.zeros(world - 1, dtype=torch.float64)
    cuts = torch.searchsorted(cum, marks, right=True).tolist() if n else [0] * (world - 1)
    bounds = [0] + [min(int(c), n) for c in cuts] + [n]
    for r in range(1, world + 1):
        bounds[r] = max(bounds[r], bounds[r - 1])
    m0 = m if mass0 is None else mass0.to(torch.float64)
    perm = None
    if map_l is None:
        seg_lo = bounds[:-1]
        seg_n = [b - a for a, b in zip(bounds, bounds[1:])]
        pm = torch.cumsum(m0, 0)
        edge = [0.0] + [float(pm[b - 1]) if b > 0 else 0.0 for b in bounds[1:]]
    else:
        mp = map_l.to(torch.int64)
        perm = torch.argsort(mp, stable=True)
        smap = mp[perm]
        bt = torch.tensor(bounds, dtype=torch.int64, device=smap.device)
        pos = torch.searchsorted(smap, bt).tolist()
        seg_lo = pos[:-1]
        seg_n = [b - a for a, b in zip(pos, pos[1:])]
        pm = torch.cumsum(m0[perm], 0)
        edge = [0.0] + [float(pm[p - 1]) if p > 0 else 0.0 for p in pos[1:]]
        perm = perm.to(torch.int32)
    tot0 = edge[-1]
    seg_mass = [edge[r + 1] - edge[r] for r in range(world)]
    if tot0 > 0:
        s = [int(round(n * edge[r] / tot0)) for r in range(world + 1)]
    else:
        s = [n * r // world for r in range(world + 1)]
    s[-1] = n
    return ShardLayout(n, bounds, perm, seg_lo, seg_n, s[:-1],
                       [s[r + 1] - s[r] for r in range(world)], seg_mass)


class ShardContext:
    """drg_shard_* context: W part buffers of ``capacity`` nodes (one per process, or
    all W locally when emulating), peers opened through CUDA IPC, an NCCL
    communicator for the epoch exchange when the group's backend is NCCL."""

    def __init__(self, world: int, capacity: int, group=None):
        self.world = world
        self.group = group
        self.capacity = int(capacity)
        self.rank = -1
        if group is not None:
            import torch.distributed as dist
            self.rank = dist.get_rank(group)
        h = ctypes.c_void_p()
        _lib.call("drg_shard_create", world, self.rank, self.capacity, ctypes.byref(h))
        self.ctx = h
        self.nccl = False
        if group is not None:
            self._connect()

    def _connect(self) -> None:
        import torch.distributed as dist
        buf = (ctypes.c_uint8 * 64)()
        _lib.call("drg_shard_ipc_handle", self.ctx, buf)
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(buf), group=self.group)
        for r, hb in enumerate(handles):
            if r != self.rank:
                _lib.call("drg_shard_open_peer", self.ctx, r, (ctypes.c_uint8 * 64)(*hb))
        self.device_collectives = dist.get_backend(self.group) == "nccl"
        if self.device_collectives:
            # the library's own communicator (the exchange inside drg_shard_run);
            # should libnccl not load, torch's NCCL group does the same exchange
            # epoch by epoch (_exchange_host with device tensors)
            uid = (ctypes.c_uint8 * 128)()
            ok = 1
            if self.rank == 0:
                try:
                    _lib.call("drg_nccl_unique_id", uid)
                except (RuntimeError, NotImplementedError) as e:   # pragma: no cover
                    ok = 0
                    log.warning("library NCCL unavailable (%s): torch collectives", e)
            obj = [bytes(uid), ok]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(self.group, 0),
                                       group=self.group)
            if obj[1]:
                _lib.call("drg_shard_nccl_init", self.ctx, (ctypes.c_uint8 * 128)(*obj[0]))
                self.nccl = True

    def close(self) -> None:
        if self.ctx:
            _lib.load().drg_shard_destroy(self.ctx)
            self.ctx = None

    def __del__(self):  # pragma: no cover - interpreter teardown order
        try:
            self.close()
        except Exception:
            pass

    # ---- one level -------------------------------------------------------------
    def level(self, lay: ShardLayout, device) -> None:
        self.layout = lay
        W = self.world
        self.pad = lay.pad
        self.snap = torch.empty((W * self.pad, 2), dtype=torch.float32, device=device)
        self.delta = torch.zeros((W * self.pad, 2), dtype=torch.float32, device=device)
        bounds = (ctypes.c_int64 * (W + 1))(*lay.bounds)
        pad = _lib.out_i64()
        _lib.call("drg_shard_level", self.ctx, lay.n, bounds, _lib.ptr(self.snap),
                  _lib.ptr(self.delta), _lib.byref(pad))

    def load(self, y: torch.Tensor) -> None:
        _lib.call("drg_shard_load", self.ctx, _lib.ptr(y), _lib.stream_ptr())

    def exchange(self) -> None:
        """Epoch end: reactions folded into their owners, snapshots refreshed."""
        if self.rank < 0 or self.nccl or self.world == 1:
            _lib.call("drg_shard_exchange", self.ctx, _lib.stream_ptr())
            return
        self._exchange_host()

    def store(self, y: torch.Tensor) -> torch.Tensor:
        if self.rank < 0 or self.nccl or self.world == 1:
            _lib.call("drg_shard_store", self.ctx, _lib.ptr(y), _lib.stream_ptr())
            return y
        self._gather_host()
        lay = self.layout
        for r in range(self.world):
            a, b = lay.bounds[r], lay.bounds[r + 1]
            y[a:b] = self.snap[r * self.pad:r * self.pad + b - a]
        return y

    # the exchange through torch.distributed (gloo in the CPU tests: host copies; a
    # torch NCCL group without the library's communicator: device tensors)
    def _exchange_host(self) -> None:
        import torch.distributed as dist
        if getattr(self, "device_collectives", False):
            own = torch.empty((self.pad, 2), dtype=torch.float32, device=self.delta.device)
            dist.reduce_scatter_tensor(own, self.delta, group=self.group)
        else:
            d = self.delta.cpu()
            dist.all_reduce(d, group=self.group)
            own = d[self.rank * self.pad:(self.rank + 1) * self.pad].contiguous().cuda()
        _lib.call("drg_shard_fold", self.ctx, _lib.ptr(own), _lib.stream_ptr())
        self.delta.zero_()
        self._gather_host()

    def _gather_host(self) -> None:
        import torch.distributed as dist
        part = torch.empty((self.pad, 2), dtype=torch.float32, device=self.snap.device)
        _lib.call("drg_shard_read_part", self.ctx, _lib.ptr(part), _lib.stream_ptr())
        if getattr(self, "device_collectives", False):
            dist.all_gather_into_tensor(self.snap, part, group=self.group)
            return
        parts = [torch.empty((self.pad, 2), dtype=torch.float32) for _ in range(self.world)]
        dist.all_gather(parts, part.cpu(), group=self.group)
        self.snap.copy_(torch.cat(parts).to(self.snap.device))


_CONTEXTS: dict = {}


def context_for(world: int, capacity: int, group=None) -> ShardContext:
    """A ShardContext for (world, group) with at least ``capacity`` nodes per part,
    kept across layouts (IPC mappings and the NCCL communicator are set up once).
    Every rank asks with the same capacity (the layouts are deterministic), so a
    re-creation is collective."""
    key = (world, None if group is None else id(group))
    c = _CONTEXTS.get(key)
    if c is None or c.capacity < capacity:
        if c is not None:
            c.close()
        c = ShardContext(world, capacity, group)
        _CONTEXTS[key] = c
    return c
