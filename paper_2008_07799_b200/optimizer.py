"""Multilevel layout optimisation on the GPU (drop-in for drgraph.optimizer).

``layout_graph`` keeps the reference signature (optimizer.py:361-413) and returns
the same ``Layout``; everything after ingestion runs on the device:

    K1 k-hop rows -> K2/K3 similarity -> K4 hierarchy -> A10 level aggregation
    -> per-level Vose tables + packed rows -> K7 iterations (K8 scheduler) -> K6
    prolongation, coarsest to finest.

One K7 iteration at level l stands in for one reference epoch (n_l sampled
steps): it applies the epoch's expected displacement.  The
reference's bitwise splitmix64 trajectories are not reproduced (allowed by the
north star); parity is single-step (tests/test_gpu_parity.py) and final-layout
KL / neighbourhood preservation (tests/test_gpu_quality.py).

Multi-GPU: with a torch.distributed process group, levels with at least
``shard_min_nodes`` nodes are partitioned by node range.  update="sampled"
(shard.py): one distributed Y that every rank maps over NVLink, each rank running
the steps whose source it owns, negatives' reactions folded by a reduce-scatter +
all-gather per epoch (drg_shard_run); the gather modes: each rank updates its rows
and an all-gather refreshes the replicated Y every iteration.  Smaller levels run
replicated (an epoch there is shorter than one exchange).
"""

from __future__ import annotations

import concurrent.futures
import ctypes
import logging
import math
import os
from dataclasses import dataclass, field
from typing import Callable

import numpy as np
import torch

from . import _lib
from .graph import DeviceGraph, Graph, device_components, device_k_neighborhoods
from .multilevel import (DeviceHierarchy, Hierarchy, compose_maps, device_build_hierarchy,
                         device_prolong, first_level_order, isolated_last,
                         relabel_coarse_levels)
from .similarity import (DeviceSimilarity, SimilarityParams, SparseSimilarity,
                         device_similarity)

logger = logging.getLogger("drgraph")

_HIERARCHY_TAG = 1
_INIT_TAG = 2
_JITTER_TAG = 3
_EPOCH_TAG = 4
_INT_MAX = 2**31 - 1


def _derive_seed(seed: int, *tags: int) -> int:
    """Deterministic uint64 child seed (optimizer.py:32-34)."""
    return int(np.random.SeedSequence([seed, *tags]).generate_state(1, np.uint64)[0])


@dataclass
class OptimizerParams:
    """optimizer.py:37-74 (same fields, defaults and validation) plus B200
    extensions: ``init`` ("normal" = reference N(0, init_scale); "uniform" =
    U[-init_scale, init_scale], BASELINE config C1) and ``update``:

    * "sampled" (default): the reference's own step (_kernels.py:65-140) run
      Hogwild-style on the GPU -- KL/NP parity with the reference, fastest on one
      GPU; run-to-run nondeterministic like the reference's threads > 1 mode.
      Steps in flight (``sampled_concurrency[_coarse]``, default by graph size,
      ``sampled_divisors``) trade speed for fidelity.  Levels whose busiest node is the source of > HUB_STEPS steps per epoch
      use warp-aggregated atomics; with ``hub_levels="jacobi"`` the levels above
      GATHER_STEPS (R-MAT coarse levels, where same-address atomics serialise) run
      the gather instead -- faster, but not faithful there (KL +77% on R-MAT 18).
    * "jacobi": the node-parallel expected-gradient iteration (SURVEY §8(a) A12,
      CSR gather + M negatives per node) -- bitwise deterministic and node-range
      shardable across GPUs; matches KL, lower NP on multilevel RGG.
    * "inplace": the gather with in-place (Hogwild) updates.
    * "sgather": the gather with S sampled attraction partners (fast, lower NP).

    ``threads`` keeps the reference's contract (optimizer.py:325-345):
    threads = 1 (the default) is bitwise deterministic for a fixed seed -- the
    sampled epochs run as sub-batches of concurrent steps over positions frozen at
    the sub-batch start with fixed-point (order-independent) increments
    (DRG_SAMPLED_DETERMINISTIC); threads > 1 runs them Hogwild, like the reference's
    worker threads: faster, run-to-run nondeterministic."""

    neg_samples: int = 5
    gamma: float = 0.1
    gamma_coarsest: float = 0.01
    iters: int = 400
    b: int = 2
    lr0: float = 1.0
    grad_clip: float = 5.0
    eps: float = 1e-3
    neg_power: float = 0.75
    init_scale: float = 1e-4
    jitter_rel: float = 1e-3
    seed: int = 0
    threads: int = 1
    init: str = "normal"
    update: str = "sampled"
    # multi-GPU: levels of at least this many nodes are partitioned over the ranks;
    # smaller ones run replicated -- their epochs (C4 level 1: 21 us for 142 k
    # nodes) are shorter than one NVLink exchange
    shard_min_nodes: int = 1 << 20
    # update="sampled": n_0 / this many steps in flight on level 0, n_l / the coarse
    # value on coarser levels; None = by graph size (sampled_divisors)
    sampled_concurrency: int | None = None
    sampled_concurrency_coarse: int | None = None
    # update="sampled", threads > 1: steps under per-node locks on the source and the
    # attraction partner (DRG_SAMPLED_LOCKED) on plain (non-hub) levels.  None = by
    # graph size: on for graphs below FAST_CONCURRENCY_NODES nodes, whose Hogwild
    # form is held to n/256 steps in flight by fidelity (locked_divisors)
    sampled_locks: bool | None = None
    # update="sampled", Hogwild levels: the negatives' positions read from a read-only
    # snapshot of y refreshed before every epoch (DRG_SAMPLED_SNAPSHOT).  None = on
    # for plain levels with at least SNAPSHOT_MIN_THREADS steps in flight (the levels
    # bound by random L2 operations: the C4 mesh's level 0)
    sampled_snapshot: bool | None = None
    att_samples: int = 2           # update="sgather": attraction partners drawn per node
    # update="sampled": the update of levels above GATHER_STEPS.  "sampled" (default)
    # keeps the reference's step there too; "jacobi" gathers them -- 3-6x faster on
    # R-MAT but KL +77% on R-MAT scale 18 (profiles/r01_quality_rmat18_*)
    hub_levels: str = "sampled"
    sampled_fused: bool = False    # update="sampled": draw inline (one kernel per epoch)
                                   # instead of the split draw pass + update pass
    # update="sampled": run levels of >= shard_min_nodes nodes as this many ranks
    # emulated on one GPU (the multi-GPU path of shard.py, all parts local) -- the
    # fidelity emulation of a multi-GPU run; 0 = off
    virtual_ranks: int = 0
    # multi-GPU sampled levels: overlap each epoch's exchange with the next epoch
    # (negatives read positions up to two epochs old, reactions fold in one epoch
    # later; DRG_SHARD_LAGGED) instead of exchanging between epochs
    shard_lagged: bool = False
    # multi-GPU sampled levels: exchange after every this-many epochs (1 = every epoch;
    # r > 1 lets negatives read positions up to r epochs old)
    shard_exchange_every: int = 1

    def __post_init__(self) -> None:
        if self.neg_samples < 0:
            raise ValueError("neg_samples must be >= 0")
        if self.gamma <= 0 or self.gamma_coarsest <= 0:
            raise ValueError("gamma must be positive")
        if self.iters < 1:
            raise ValueError("iters must be >= 1")
        if self.b < 1:
            raise ValueError("b must be >= 1")
        if self.lr0 <= 0:
            raise ValueError("lr0 must be positive")
        if self.threads < 1:
            raise ValueError("threads must be >= 1")
        if self.seed < 0:
            raise ValueError("seed must be non-negative")
        for c in (self.sampled_concurrency, self.sampled_concurrency_coarse):
            if c is not None and c < 1:
                raise ValueError("sampled concurrency divisors must be >= 1")
        if self.shard_exchange_every < 1:
            raise ValueError("shard_exchange_every must be >= 1")
        if not 0 <= self.virtual_ranks <= 8:
            raise ValueError("virtual_ranks must be in [0, 8]")
        if self.init not in ("normal", "uniform"):
            raise ValueError("init must be 'normal' or 'uniform'")
        if self.update not in ("jacobi", "inplace", "sampled", "sgather"):
            raise ValueError("update must be 'jacobi', 'inplace', 'sampled' or 'sgather'")
        if self.att_samples < 1 or self.att_samples + self.neg_samples > 32 and \
                self.update == "sgather":
            raise ValueError("sgather needs att_samples >= 1 and att_samples + neg_samples <= 32")


@dataclass
class Layout:
    """2-D position per node plus bookkeeping (optimizer.py:77-82)."""

    positions: np.ndarray
    stats: dict = field(default_factory=dict)


@dataclass(frozen=True)
class AliasTable:
    """Vose table (optimizer.py:85-108): fp32 thresholds as stored on device."""

    prob: np.ndarray
    alias: np.ndarray
    total_weight: float

    def __len__(self) -> int:
        return len(self.prob)

    # host-side draws from a built table, with the caller's numpy generator (the
    # reference's own sampling helpers, optimizer.py:96-108)
    def sample(self, rng: np.random.Generator) -> int:
        u = rng.random(2)
        idx = min(int(u[0] * len(self.prob)), len(self.prob) - 1)
        return idx if u[1] < self.prob[idx] else int(self.alias[idx])

    def sample_many(self, rng: np.random.Generator, size: int) -> np.ndarray:
        idx = np.minimum((rng.random(size) * len(self.prob)).astype(np.int64),
                         len(self.prob) - 1)
        coin = rng.random(size)
        out = idx.copy()
        take = coin >= self.prob[idx]
        out[take] = self.alias[idx[take]]
        return out


@dataclass(frozen=True)
class PositiveSampler:
    """Alias table over the canonical pairs (i < j) of P plus a direction coin
    (optimizer.py:206-229): (i, j) lands with probability P_ij / total."""

    table: AliasTable
    lo: np.ndarray  # int32
    hi: np.ndarray  # int32

    def sample(self, rng: np.random.Generator) -> tuple[int, int]:
        e = self.table.sample(rng)
        if rng.random() < 0.5:
            return int(self.lo[e]), int(self.hi[e])
        return int(self.hi[e]), int(self.lo[e])

    def sample_many(self, rng: np.random.Generator, size: int):
        e = self.table.sample_many(rng, size)
        flip = rng.random(size) >= 0.5
        return (np.where(flip, self.hi[e], self.lo[e]), np.where(flip, self.lo[e], self.hi[e]))


def _alias_device(w: torch.Tensor) -> tuple[torch.Tensor, float]:
    n = w.numel()
    table = torch.empty(n, dtype=torch.int64, device=w.device)
    total = _lib.out_f64()
    _lib.call("drg_alias_build", _lib.ptr(w), n, _lib.ptr(table), _lib.byref(total),
              _lib.stream_ptr())
    return table, total.value


def _unpack_alias(table: torch.Tensor, total: float) -> AliasTable:
    raw = table.cpu().numpy().view(np.uint32).reshape(-1, 2)
    return AliasTable(raw[:, 0].view(np.float32).astype(np.float64),
                      raw[:, 1].astype(np.int32), total)


def build_alias_table(weights) -> AliasTable:
    """optimizer.py:111-139 (built by the library's Vose routine)."""
    w = np.asarray(weights, dtype=np.float64)
    if len(w) == 0:
        raise ValueError("cannot build an alias table over zero items")
    if w.min() < 0:
        raise ValueError("negative weight")
    if not float(w.sum()) > 0:
        raise ValueError("all weights are zero")
    _lib.load()
    table, total = _alias_device(torch.from_numpy(np.ascontiguousarray(w)).cuda())
    return _unpack_alias(table, total)


def device_negative_weights(row_mass: torch.Tensor, power: float) -> torch.Tensor:
    """optimizer.py:243-259 weights on device (drg_negative_weights)."""
    w = torch.empty_like(row_mass)
    _lib.call("drg_negative_weights", _lib.ptr(row_mass), row_mass.numel(), float(power),
              _lib.ptr(w), _lib.stream_ptr())
    return w


def build_positive_sampler(ns: SparseSimilarity) -> PositiveSampler:
    """O(1) sampler of directed pairs proportional to their similarity
    (optimizer.py:232-240): the device Vose table over the canonical pairs."""
    if ns.entry_count == 0 or float(ns.weights.sum()) <= 0.0:
        raise ValueError("similarity carries no mass; nothing to sample")
    src = ns.sources()
    canonical = src < ns.targets
    return PositiveSampler(build_alias_table(ns.weights[canonical]),
                           src[canonical].astype(np.int32),
                           ns.targets[canonical].astype(np.int32))


def _gradients(y_i, y_j, b: int, gamma: float, eps: float, clip: float, kind: int) -> np.ndarray:
    _lib.load()
    a = torch.tensor([[float(y_i[0]), float(y_i[1])]], dtype=torch.float64, device="cuda")
    c = torch.tensor([[float(y_j[0]), float(y_j[1])]], dtype=torch.float64, device="cuda")
    out = torch.empty((1, 2), dtype=torch.float64, device="cuda")
    _lib.call("drg_gradients", _lib.ptr(a), _lib.ptr(c), 1, int(b), float(gamma), float(eps),
              float(clip), kind, _lib.ptr(out), _lib.stream_ptr())
    return out.cpu().numpy()[0]


def attractive_gradient(y_i, y_j, b: int) -> np.ndarray:
    """Gradient of log(1 / (1 + d^(2b))) w.r.t. y_i (optimizer.py:174-186; zero at
    coincident positions, not clipped), by drg_gradients -- the device function the
    layout kernels inline."""
    return _gradients(y_i, y_j, b, 0.0, 0.0, math.inf, 0)


def repulsive_gradient(y_i, y_jm, b: int, gamma: float, eps: float,
                       clip: float = math.inf) -> np.ndarray:
    """Gradient of gamma log(1 - 1/(1 + d^(2b))) w.r.t. y_i with the eps floor, each
    component clamped to +-clip (optimizer.py:189-203), by drg_gradients."""
    return _gradients(y_i, y_jm, b, gamma, eps, clip, 1)


def lp_kernel(ld: float, b: int) -> float:
    """Unnormalised layout-proximity kernel 1 / (1 + ld^(2b)) (optimizer.py:150-152)."""
    x = ld * ld
    r = 1.0
    for _ in range(b):
        r *= x
    return 1.0 / (1.0 + r)


@dataclass(frozen=True)
class GradientSample:
    """One sampled interaction, for tracing (optimizer.py:155-171)."""

    i: int
    j: int
    ld: float
    lp_kernel: float
    kind: str

    @classmethod
    def from_positions(cls, i: int, j: int, y_i, y_j, b: int, kind: str) -> "GradientSample":
        dx = float(y_i[0]) - float(y_j[0])
        dy = float(y_i[1]) - float(y_j[1])
        ld = math.sqrt(dx * dx + dy * dy)
        return cls(i=i, j=j, ld=ld, lp_kernel=lp_kernel(ld, b), kind=kind)


def build_negative_sampler(ns: SparseSimilarity, power: float = 0.75) -> AliasTable:
    """O(1) node sampler by (incident mass)**power, floor 1e-8*max (optimizer.py:243-259)."""
    _lib.load()
    r = torch.from_numpy(np.ascontiguousarray(ns.row_masses())).cuda()
    table, total = _alias_device(device_negative_weights(r, power))
    return _unpack_alias(table, total)


# ---------------------------------------------------------------------------
# per-level device data
# ---------------------------------------------------------------------------

@dataclass
class LevelData:
    """What K7 reads at one level: CSR row offsets, packed {target, W} records,
    per-node repulsion weight V, and the level's Vose table over Q^l."""

    n: int
    nnz: int
    indptr: torch.Tensor   # int64 [n+1]
    rec: torch.Tensor      # int64 [nnz]  (int32 target | fp32 W << 32)
    V: torch.Tensor        # fp32 [n]
    alias: torch.Tensor    # int64 [n]    (fp32 prob | int32 alias << 32)
    heavy: dict | None = None   # heavy-row split tensors (rows > HEAVY_ROW entries)
    sampled: "SampledTables | None" = None   # update="sampled" tables of this level
    # rows [n_active, n) have no P entries (the isolated nodes isolated_last puts
    # last): the gather leaves them frozen, as the reference effectively does -- they
    # are never sources and are drawn as negatives with ~1e-8 of the mass
    # (optimizer.py:256-258).  None = all rows active.
    n_active: int | None = None

    @property
    def active(self) -> int:
        return self.n if self.n_active is None else self.n_active

    def algorithmic_bytes(self, M: int) -> int:
        """16 B per P entry + (24 + 16 M) B per updated node (level 0)
        -- col 4 + W 4 + y_j 8 per entry; rowptr 4 + y_a 8 + y_a' 8 + V 4 and per
        negative an 8 B alias record + 8 B y_c per node."""
        return 16 * self.nnz + (24 + 16 * M) * self.active


HEAVY_ROW = 4 * _lib.DRG_HEAVY_CHUNK   # rows longer than this are split across warps


def active_rows(indptr: torch.Tensor) -> int:
    """1 + the last row with P entries (the rows after it form the frozen tail)."""
    nz = torch.nonzero(indptr[1:] > indptr[:-1])
    return int(nz[-1]) + 1 if nz.numel() else 0


def heavy_split(indptr: torch.Tensor, threshold: int = HEAVY_ROW) -> dict | None:
    """Chunk list of the rows with more than ``threshold`` entries (drg_heavy_split):
    a heavy-tailed row (an R-MAT hub) is streamed by many warps instead of one."""
    deg = indptr[1:] - indptr[:-1]
    heavy = torch.nonzero(deg > threshold).flatten()
    if heavy.numel() == 0:
        return None
    C = _lib.DRG_HEAVY_CHUNK
    nch = (deg[heavy] + C - 1) // C
    ptr = torch.zeros(heavy.numel() + 1, dtype=torch.int64, device=indptr.device)
    ptr[1:] = torch.cumsum(nch, 0)
    rows = torch.repeat_interleave(heavy, nch)
    within = torch.arange(rows.numel(), device=indptr.device) - torch.repeat_interleave(ptr[:-1], nch)
    slot = torch.full((deg.numel(),), -1, dtype=torch.int32, device=indptr.device)
    slot[heavy] = torch.arange(heavy.numel(), dtype=torch.int32, device=indptr.device)
    t = {"slot": slot, "chunk_ptr": ptr.to(torch.int32), "chunk_row": rows.to(torch.int32),
         "chunk_begin": (indptr[rows] + within * C).contiguous(),
         "partial": torch.empty(2 * rows.numel(), dtype=torch.float32, device=indptr.device)}
    t["struct"] = _lib.HeavySplit(t["slot"].data_ptr(), t["chunk_ptr"].data_ptr(),
                                  t["chunk_row"].data_ptr(), t["chunk_begin"].data_ptr(),
                                  rows.numel(), t["partial"].data_ptr())
    return t


def _aggregate_pairs(indptr, targets, weights, parent, n_coarse):
    n = indptr.numel() - 1
    nnz = targets.numel()
    dev = indptr.device
    o_ip = torch.empty(n_coarse + 1, dtype=torch.int64, device=dev)
    o_tg = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
    o_w = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
    out_nnz = _lib.out_i64()
    _lib.call("drg_aggregate_pairs", _lib.ptr(indptr), _lib.ptr(targets), _lib.ptr(weights), n,
              nnz, _lib.ptr(parent), n_coarse, _lib.ptr(o_ip), _lib.ptr(o_tg), _lib.ptr(o_w),
              _lib.byref(out_nnz), _lib.stream_ptr())
    k = out_nnz.value
    return o_ip, o_tg[:k].clone(), o_w[:k].clone()


def _aggregate_nodes(values, parent, n_coarse):
    out = torch.empty(n_coarse, dtype=torch.float64, device=values.device)
    _lib.call("drg_aggregate_nodes", _lib.ptr(values), _lib.ptr(parent), values.numel(),
              n_coarse, _lib.ptr(out), _lib.stream_ptr())
    return out


def pack_level(indptr, targets, P, R, Wn, q_scale, n, sort_rows=False
               ) -> tuple[torch.Tensor, torch.Tensor]:
    nnz = targets.numel()
    rec = torch.empty(max(nnz, 1), dtype=torch.int64, device=R.device)
    V = torch.empty(max(n, 1), dtype=torch.float32, device=R.device)
    _lib.call("drg_level_pack", _lib.ptr(indptr), _lib.ptr(targets), _lib.ptr(P), _lib.ptr(R),
              _lib.ptr(Wn), float(q_scale), n, nnz, int(bool(sort_rows)), _lib.ptr(rec),
              _lib.ptr(V), _lib.stream_ptr())
    return rec[:nnz], V[:n]


@dataclass
class SampledTables:
    """update="sampled" tables of one level l: drawing a level-0 pair ~ P and
    mapping it to level l (the reference, _kernels.py:66-81) has exactly the law
    "source a ~ R^l, then with probability c_a the collapsed pair (a, a), else b ~
    P^l_a." with c_a = 1 - sum_b P^l_ab / R^l_a (mass of pairs inside a); negatives
    drawn at level 0 and mapped follow Q^l (the level's negative table)."""

    src_alias: torch.Tensor   # int64 [n]  Vose over R^l
    row_alias: torch.Tensor   # int64 [nnz, 2] per-row Vose over P^l: {threshold, alias target,
                              # own target, 0} -- one 16-byte record per entry
    collapse: torch.Tensor | None   # fp32 [n]   c_a (None: no collapsed pairs)
    wsum: torch.Tensor | None       # fp32 [n]   sum_b W_ab = 2 n_l sum_b P^l_ab (sgather)
    hubs: bool = False        # some node takes part in > HUB_STEPS steps per epoch
    gather: bool = False      # ... in > GATHER_STEPS: the level runs hub_levels' update
    # draw-then-map form (coarse levels of a "sampled" plan): the tables above are
    # level 0's, ``map`` (int32 [n_0]) the composed parent map to this level
    map: torch.Tensor | None = None
    indptr: torch.Tensor | None = None      # level-0 row offsets of row_alias
    mass: torch.Tensor | None = None        # R^l (fp64 [n_l]): partitions for multi-GPU
    hot: torch.Tensor | None = None         # int32: hub level's hottest nodes (staged per block)
    # the level's negative table Q^l (NegTable); None: the level's own full table
    neg: "NegTable | None" = None
    span: torch.Tensor | None = None        # int64 [n_0] {row start, length} (drg_row_spans)
    # 32-byte source records (drg_src_records): bucket + both outcomes' spans and
    # collapse probabilities in one sector (DRG_SAMPLED_SRC_RECORDS)
    src_rec: torch.Tensor | None = None


@dataclass
class NegTable:
    """Q^l as drawn by the sampled kernels (drg_layout_sampled's neg_* arguments):
    Vose over the nodes [0, n) and, with probability tail_p, a uniform pick in the
    tail [n, n + tail_n) -- the isolated nodes, which isolated_last numbers last and
    which all carry the same floor weight (optimizer.py:258).  Same law as one table
    over every node, from a table the size of the connected part."""

    alias: torch.Tensor
    n: int
    tail_n: int = 0
    tail_p: float = 0.0


def connected_prefix(R: torch.Tensor) -> int:
    """1 + the last node with graph mass (R > 0): the nodes past it are isolated."""
    nz = torch.nonzero(R > 0)
    return int(nz[-1, 0]) + 1 if nz.numel() else 0


def build_neg_table(Wn: torch.Tensor, R: torch.Tensor) -> NegTable:
    """Q^l over the connected prefix + the uniform isolated tail (exact in law: the
    tail's weights are all equal; otherwise one table over every node)."""
    n = Wn.numel()
    k = connected_prefix(R)
    if 0 < k < n:
        tail = Wn[k:]
        if float(tail.max()) == float(tail.min()):
            tot = float(Wn.sum())
            alias, _ = _alias_device(Wn[:k].contiguous())
            return NegTable(alias, k, n - k, float(tail.sum()) / tot if tot > 0 else 0.0)
    alias, _ = _alias_device(Wn)
    return NegTable(alias, n)


# Steps in flight of the Hogwild update pass (the fidelity knob).  Concurrent steps
# read positions that other in-flight steps are about to move; measured against the
# reference (scripts/quality.py, profiles/r01_quality_*concurrency*): n/16 costs
# NP -4.1% on C1 (10k-node grid, 400 seeds) and -5.2% on C2 (200k RGG, 64 seeds),
# n/256 (coarse n/64) -0.5% and -1.9% -- within the 2% bar; on the C4 mesh
# (1.73 M nodes) n/16 (coarse n/4) is already within it (NP -0.5%) and keeps the
# >= 6e4 steps in flight the update pass needs to reach the L2 random-access ceiling.
FAST_CONCURRENCY_NODES = 1_000_000


def sampled_divisors(n0: int, opt: "OptimizerParams") -> tuple[int, int]:
    """(level-0, coarse-level) divisors of the steps in flight: the explicit
    OptimizerParams values, else n/16 and n/4 for graphs of >= FAST_CONCURRENCY_NODES
    nodes and n/256 and n/64 below."""
    big = n0 >= FAST_CONCURRENCY_NODES
    fine = opt.sampled_concurrency or (16 if big else 256)
    coarse = opt.sampled_concurrency_coarse or (4 if big else 64)
    return fine, coarse


# Steps under (i, j) locks (DRG_SAMPLED_LOCKED): the steps in flight touch disjoint
# (source, partner) pairs, so the fidelity no longer depends on how many there are.
# C1 (100 seeds, profiles/r02_quality_grid_locks.jsonl): Hogwild at n/4 steps in
# flight KL +2.4% / NP -11.6%, at n/16 +0.6% / -4.1%; locked at n/1 KL +0.03% / NP
# +1.1% +- 2.0%.  C2 (48 seeds, r02_quality_rgg_48seeds_locks.jsonl): locked at n/1
# on every level KL -0.01% / NP +1.4% +- 1.7%, at n/2 (n/1 coarse) +0.14% / +0.5% +-
# 1.6% (Hogwild n/256: +0.07% / +0.5% +- 1.7%).  A locked step costs two more L2
# round trips (acquire, returning update) and retries while its nodes are held, so
# it pays where Hogwild is fidelity-capped far below the machine: graphs under
# FAST_CONCURRENCY_NODES (C1 2 528 -> 23 181 iters/s, C2 4 788 -> 21 397,
# r02_bench_locks_sweep.jsonl).  On the C4 mesh the Hogwild levels are faster:
# level 0 is bound by random L2 operations, to which the locks add four per step
# (174 -> 253 ms), and its small coarse levels run n/4 Hogwild -- measured faithful
# there -- in 8-15 ms against 37-48 ms locked.
LOCKED_DIVISORS = (1, 1)
# Hogwild levels with at least this many steps in flight are bound by the L2's
# random-operation rate, not by a step's latency: there the negatives are gathered
# from a read-only snapshot (DRG_SAMPLED_SNAPSHOT) -- gathers and reductions on
# separate arrays run at 213 G/s per step mix against 148 G/s on one array
# (profiles/r02_l2_random_peak.txt).
SNAPSHOT_MIN_THREADS = 40960


def locked_divisors(opt: "OptimizerParams") -> tuple[int, int]:
    return (opt.sampled_concurrency or LOCKED_DIVISORS[0],
            opt.sampled_concurrency_coarse or LOCKED_DIVISORS[1])


HUB_STEPS = 512   # warp-aggregate the sampled updates above this per-node rate
# level-0 node count from which the per-node tables (8 B per node each) are far above
# L2 and the inline draws of hub levels take L2 eviction hints (DRG_SAMPLED_L2_HINTS)
L2_HINT_NODES = 1 << 22
# Above this per-node rate each block stages the level's HOT_NODES busiest nodes in
# shared memory (apply_hot_kernel): R-MAT's coarse levels, where one node is the
# source of up to a third of an epoch's steps, and the C3 BA coarsest level.
HOT_STEPS = int(os.environ.get("DRG_HOT_STEPS", 4096))   # (env: experiments)
HOT_NODES = 64
# Steps in flight on those levels.  A staged hub no longer serialises its steps on
# its L2 line, so every concurrent step that touches it really reads the same
# position: R-MAT scale 20 (hub in ~1/3 of a coarse epoch's steps) keeps KL within
# 0.2% of the reference at 50-100 k steps in flight and drifts -10% at the ~150 k the
# n/4 default reaches (profiles/r02_quality_rmat20_*).  The plain (unstaged) kernel
# is faithful at n/4 because the hub's atomics serialise -- and 4x slower.
HOT_MAX_THREADS = int(os.environ.get("DRG_HOT_MAX_THREADS", 65536))   # (env: experiments)
HOT_CAP_SHARE = 0.01   # busiest node's share of the steps from which the cap is flat
# Above this per-node rate the sampled epoch serialises on the hub's atomics even
# warp-aggregated, and the gather (K7 + heavy-row split) is faster: R-MAT's coarse
# levels (busiest node 2.4e5 - 4.8e6 steps per epoch) -- while R-MAT's level 0
# (1.4e4: sampled 3.8 ms per epoch vs gather 5.2 ms) and the C3 BA levels (<= 6e3)
# stay sampled.
GATHER_STEPS = 32768


# Source draws from 32-byte records (drg_src_records) on 1-GPU sampled levels whose
# per-node tables are far above L2 (>= L2_HINT_NODES level-0 nodes: R-MAT scale 24,
# one DRAM miss per drawn source instead of three).  Below that the three 8-byte
# tables stay in L2 and the records only add traffic: the C4 mesh's draw pass read
# 280 MB of DRAM per epoch with them against 235 MB without, at the same speed.
# (DRG_SRC_RECORDS env for experiments: 1 = always, 0 = never)
SRC_RECORDS = os.environ.get("DRG_SRC_RECORDS", "auto")


def _use_src_records(n0: int) -> bool:
    return SRC_RECORDS == "1" or (SRC_RECORDS == "auto" and n0 >= L2_HINT_NODES)


def src_records(S: SampledTables, indptr: torch.Tensor, collapse) -> torch.Tensor | None:
    """drg_src_records over S.src_alias (None when nnz >= 2^32)."""
    k = S.src_alias.numel()
    if int(indptr[-1]) >= (1 << 32):
        return None
    out = torch.empty((max(k, 1), 4), dtype=torch.int64, device=indptr.device)
    _lib.call("drg_src_records", _lib.ptr(S.src_alias), k, _lib.ptr(indptr),
              _lib.ptr(collapse), _lib.ptr(out), _lib.stream_ptr())
    return out


def build_sampled_tables(ip, tg, P, R, Wn=None) -> SampledTables:
    """Per-row Vose over P (16-byte records), Vose over R -- over the connected
    prefix only (isolated nodes have R = 0 and are never a source) -- collapse
    probabilities, and with ``Wn`` the negative table."""
    n = ip.numel() - 1
    nnz = tg.numel()
    rows = torch.empty((max(nnz, 1), 2), dtype=torch.int64, device=R.device)   # 16 B per entry
    rowsum = torch.empty(max(n, 1), dtype=torch.float64, device=R.device)
    _lib.call("drg_row_alias", _lib.ptr(ip), _lib.ptr(tg), _lib.ptr(P), n, nnz, _lib.ptr(rows),
              _lib.ptr(rowsum), _lib.stream_ptr())
    k = connected_prefix(R)
    src, _ = _alias_device(R[:max(k, 1)].contiguous())
    span = None
    if nnz < (1 << 32):
        span = torch.empty(max(n, 1), dtype=torch.int64, device=R.device)
        _lib.call("drg_row_spans", _lib.ptr(ip), n, _lib.ptr(span), _lib.stream_ptr())
    with torch.no_grad():
        c = torch.where(R > 0, 1.0 - rowsum[:n] / torch.clamp(R, min=1e-300),
                        torch.zeros_like(R)).clamp_(0.0, 1.0).to(torch.float32)
        wsum = (2.0 * n * rowsum[:n]).to(torch.float32)
        hubs = _is_hub_level(R)
    return SampledTables(src, rows[:nnz], c, wsum, hubs, mass=R, hot=_hot_nodes(R),
                         neg=None if Wn is None else build_neg_table(Wn, R), span=span)


# Coarse levels that draw from their own pair tables (P^l aggregated, level-l form of
# the law) instead of level 0's through the composed map: "hub" = the hub-staged
# levels (DRG_LEVEL_TABLES env for experiments: none | hub | all)
LEVEL_TABLES = os.environ.get("DRG_LEVEL_TABLES", "hub")


def build_mapped_level_data(ds: DeviceSimilarity, dh: DeviceHierarchy,
                            neg_power: float = 0.75,
                            level_tables: str | None = None) -> list[LevelData]:
    """update="sampled" without level aggregation: the reference draws every pair
    and negative at level 0 and maps it to the current level (_kernels.py:76-81,
    115), so the level-0 tables (per-row Vose over P, Vose over R and Q) serve all
    levels through the composed parent maps (drg_compose_maps).  Only R^l is pulled
    up (drg_aggregate_nodes) to detect hub-heavy levels.  No P^l, no packed
    records: the gather modes build them with build_level_data."""
    ip, tg, P, R = ds.indptr, ds.targets, ds.weights, ds.row_mass
    Wn = device_negative_weights(R, neg_power)
    S0 = build_sampled_tables(ip, tg, P, R, Wn)
    S0.collapse = None   # no pair collapses at level 0
    n0 = dh.levels[0].node_count
    use_rec = _use_src_records(n0)
    if use_rec:
        S0.src_rec = src_records(S0, ip, None)
    out = [LevelData(n0, tg.numel(), ip, None, None, None, None, S0)]
    flat = None
    st = _lib.stream_ptr()
    mode = LEVEL_TABLES if level_tables is None else level_tables
    pairs = (ip, tg, P)   # P^l pulled up level by level, as far as some level uses it
    own, Rl = {}, R        # levels that draw from their own tables (R^l is cheap)
    for level in range(1, dh.depth + 1):
        Rl = _aggregate_nodes(Rl, dh.maps[level - 1], dh.levels[level].node_count)
        own[level] = mode == "all" or (mode == "hub" and _hot_nodes(Rl) is not None)
    last_own = max((lv for lv, o in own.items() if o), default=0)
    del Rl
    for level in range(1, dh.depth + 1):
        n_l = dh.levels[level].node_count
        parent = dh.maps[level - 1]
        if level <= last_own:
            pairs = _aggregate_pairs(*pairs, parent, n_l)
        if flat is None:   # level 1: the parent map itself
            flat = parent.to(torch.int32).contiguous()
        else:              # out[i] = parent[flat[i]]
            nxt = torch.empty(n0, dtype=torch.int32, device=ip.device)
            _lib.call("drg_compose_maps", _lib.ptr(flat), _lib.ptr(parent), n0, _lib.ptr(nxt), st)
            flat = nxt
        R = _aggregate_nodes(R, parent, n_l)
        Wn = _aggregate_nodes(Wn, parent, n_l)   # Q^l: drawn at the level (same law)
        hubs = _is_hub_level(R)
        if own[level]:
            # the level's own tables: source ~ R^l, collapse c_a, target ~ P^l_a.
            S = build_sampled_tables(*pairs, R, Wn)
            if use_rec:
                S.src_rec = src_records(S, pairs[0], S.collapse)
            out.append(LevelData(n_l, pairs[1].numel(), pairs[0], None, None, None, None, S))
            continue
        S = SampledTables(S0.src_alias, S0.row_alias, None, None, hubs, map=flat, indptr=ip,
                          mass=R, hot=_hot_nodes(R), neg=build_neg_table(Wn, R), span=S0.span,
                          src_rec=S0.src_rec)
        out.append(LevelData(n_l, 0, None, None, None, None, None, S))
    return out


def _busiest_steps(R: torch.Tensor) -> float:
    """Expected steps per epoch in which the busiest node is the source."""
    n = R.numel()
    return float(R.max()) / max(float(R.sum()), 1e-300) * n if n > 0 else 0.0


def _is_hub_level(R: torch.Tensor) -> bool:
    return _busiest_steps(R) > HUB_STEPS


def _hot_nodes(R: torch.Tensor) -> torch.Tensor | None:
    """The HOT_NODES nodes of largest R on a level whose busiest node is the source
    of more than HOT_STEPS steps per epoch (None elsewhere)."""
    if R.numel() == 0 or _busiest_steps(R) <= HOT_STEPS:
        return None
    k = min(HOT_NODES, R.numel())
    return torch.topk(R, k).indices.to(torch.int32).contiguous()


def _is_gather_level(R: torch.Tensor) -> bool:
    return _busiest_steps(R) > GATHER_STEPS


def build_level_data(ds: DeviceSimilarity, dh: DeviceHierarchy, neg_power: float = 0.75,
                     sampled: bool = False, skip_hub_tables: bool = False) -> list[LevelData]:
    """P^l, R^l, Q^l for every level, pulled up level by level through the parent
    maps (drg_aggregate_pairs / drg_aggregate_nodes), then packed (drg_level_pack)
    with a Vose table per level (drg_alias_build); ``sampled`` also builds the
    level's sampled-mode tables -- except, with ``skip_hub_tables``, on hub-heavy
    levels, which then run the gather and never draw (their per-row tables over
    million-entry hub rows would be the most expensive part of the build)."""
    ip, tg, P = ds.indptr, ds.targets, ds.weights
    R = ds.row_mass
    Wn = device_negative_weights(R, neg_power)
    out = []
    for level in range(dh.depth + 1):
        n_l = dh.levels[level].node_count
        if level > 0:
            parent = dh.maps[level - 1]
            ip, tg, P = _aggregate_pairs(ip, tg, P, parent, n_l)
            R = _aggregate_nodes(R, parent, n_l)
            Wn = _aggregate_nodes(Wn, parent, n_l)
        alias, total = _alias_device(Wn)
        # rows keep their order: re-sorting level-0 rows by id (sort_rows) cut L1
        # sectors by 12% on the mesh but cost 130 ms of segmented sort and no
        # kernel time (profiles/README.md), so it is off
        rec, V = pack_level(ip, tg, P, R, Wn, 1.0 / total, n_l, sort_rows=False)
        L = LevelData(n_l, tg.numel(), ip, rec, V, alias, heavy_split(ip))
        L.n_active = active_rows(ip)
        if sampled and R.numel() > 0 and float(R.sum()) > 0:
            if skip_hub_tables and _is_gather_level(R):
                L.sampled = SampledTables(None, None, None, None, hubs=True, gather=True)
            else:
                L.sampled = build_sampled_tables(ip, tg, P, R)
        out.append(L)
    return out


StepFn = Callable[[torch.Tensor, torch.Tensor, int, int, int], None]


@dataclass
class LayoutPlan:
    """Prepared device state of one layout: level data, parent maps, params."""

    levels: list
    maps: list
    opt: OptimizerParams
    nonfinite: torch.Tensor = None
    # old -> new ids of the coarsest level (isolated_last), applied to the default Y0
    coarsest_relabel: torch.Tensor | None = None
    evals: torch.Tensor = None   # device counter of distance evaluations (sampled)
    _shard_cache: dict = field(default_factory=dict)   # multi-GPU layouts / contexts

    def distance_evals(self) -> int:
        """Distance evaluations so far (the reference's counter, _kernels.py:86, 122)."""
        return 0 if self.evals is None else int(self.evals.item())

    @property
    def depth(self) -> int:
        return len(self.levels) - 1

    def iterations(self) -> int:
        return self.opt.iters * len(self.levels)

    def launch_bytes(self, level: int = 0) -> tuple[str, int]:
        """(kernel, algorithmic bytes of one iteration launch) at ``level`` for the
        plan's update mode (the gather's 16 B per P entry + (24 + 16 M)
        B per node of SURVEY §8(d); the sampled step's 92 + 32 M B: source alias 8,
        row bounds 16, collapse 4, row alias record 16, y_i and y_j 16, per
        negative alias 8 + y_c 8, and 16 B per float2 atomic on j, each negative and
        the source)."""
        L = self.levels[level]
        M = self.opt.neg_samples
        u = self.opt.update
        if u == "sampled" and L.sampled is not None and L.sampled.gather and \
                self.opt.hub_levels == "jacobi":
            u = "jacobi"
        if u == "sampled":
            mode = self.level_mode(level)
            k = {"fused": "sampled_kernel",
                 "locked": "draw_kernel + apply_locked_kernel",
                 "deterministic": "draw_kernel + apply_det_kernel / flush_kernel",
                 "hub": ("draw_kernel + apply_hot_kernel" if L.sampled.hot is not None
                         else "draw_kernel + apply_kernel<AGG>"),
                 "snapshot": ("draw_kernel + negsnap_refresh_kernel + apply_negsnap_kernel"
                              if M <= 6 else "draw_kernel + snap_copy_kernel + apply_snap_kernel"),
                 }.get(mode, "draw_kernel + apply_kernel")
            return k, L.n * (92 + 32 * M)
        if u == "sgather":
            S = self.opt.att_samples
            return "sgather_kernel", L.n * (32 + 24 * S + 16 * M)
        return "layout_iter_kernel", L.algorithmic_bytes(M)

    def total_distance_evals(self) -> int:
        """The reference's distance-evaluation count of the run (_kernels.py:86, 122):
        counted on the device by the sampled epochs (attractions with i != j plus
        negatives that found a target); a gather iteration evaluates every P entry
        and M negatives per active node."""
        if self.opt.update == "sampled":
            return self.distance_evals()
        M = self.opt.neg_samples
        return self.opt.iters * sum(L.nnz + M * L.active for L in self.levels)

    def interactions(self) -> int:
        """Interactions applied over the whole layout stage: per gather iteration every
        P entry + M negatives per node; per sampled epoch n_l steps of one pair + M
        negatives (the reference's count)."""
        M = self.opt.neg_samples
        if self.opt.update == "sampled":
            return self.opt.iters * sum((1 + M) * L.n for L in self.levels)
        return self.opt.iters * sum(L.nnz + M * L.active for L in self.levels)

    def init_positions(self) -> torch.Tensor:
        """Coarsest-level start (optimizer.py:393-395): the reference's numpy draw
        (tag 2), so both implementations start from the same Y0."""
        n = self.levels[-1].n
        rng = np.random.default_rng(_derive_seed(self.opt.seed, _INIT_TAG))
        if self.opt.init == "uniform":
            y = rng.uniform(-self.opt.init_scale, self.opt.init_scale, size=(n, 2))
        else:
            y = rng.normal(0.0, self.opt.init_scale, size=(n, 2))
        y = torch.from_numpy(y.astype(np.float32)).cuda()
        rel = self.coarsest_relabel
        if rel is not None:   # the draw is in reference id order
            out = torch.empty_like(y)
            out[rel.to(torch.int64)] = y
            y = out
        return y

    def _level_args(self, level: int):
        L = self.levels[level]
        o = self.opt
        gamma = o.gamma_coarsest if level == self.depth else o.gamma   # optimizer.py:321
        seed = _derive_seed(o.seed, _EPOCH_TAG, level) & 0xFFFFFFFFFFFFFFFF
        return L, gamma, seed

    def kernel_step(self, level: int, y_in: torch.Tensor, y_out: torch.Tensor, row_lo: int,
                    row_hi: int, t0: int, n_iter: int = 1, neg_idx: torch.Tensor | None = None,
                    stream=None) -> None:
        """drg_layout_iters for iterations t0..t0+n_iter-1 of ``level``."""
        L, gamma, seed = self._level_args(level)
        o = self.opt
        flags = _lib.DRG_FLAG_INPLACE if y_in.data_ptr() == y_out.data_ptr() else 0
        if self.nonfinite is None:
            self.nonfinite = torch.full((1,), _INT_MAX, dtype=torch.int32, device=y_in.device)
        if o.update == "sgather" and L.sampled is not None:
            S = L.sampled
            _lib.call("drg_layout_sgather", _lib.ptr(L.indptr), _lib.ptr(L.rec),
                      _lib.ptr(S.row_alias), _lib.ptr(S.wsum), _lib.ptr(L.V), _lib.ptr(L.alias),
                      L.n, row_lo, row_hi, _lib.ptr(y_in), _lib.ptr(y_out), t0, n_iter, o.iters,
                      float(o.lr0), float(gamma), float(o.eps), float(o.grad_clip), o.b,
                      o.neg_samples, o.att_samples, seed, level, _lib.ptr(neg_idx),
                      _lib.ptr(self.nonfinite), flags, _lib.stream_ptr(stream))
            return
        _lib.call("drg_layout_iters", _lib.ptr(L.indptr), _lib.ptr(L.rec), _lib.ptr(L.V),
                  _lib.ptr(L.alias), L.n, row_lo, row_hi, _lib.ptr(y_in), _lib.ptr(y_out),
                  t0, n_iter, o.iters, float(o.lr0), float(gamma), float(o.eps),
                  float(o.grad_clip), o.b, o.neg_samples, seed, level, _lib.ptr(neg_idx),
                  _lib.ptr(self.nonfinite),
                  _lib.byref(L.heavy["struct"]) if L.heavy else None, flags,
                  _lib.stream_ptr(stream))

    def check_finite(self, level: int) -> None:
        if self.nonfinite is None:
            return
        t = int(self.nonfinite.item())
        if t != _INT_MAX:
            self.nonfinite.fill_(_INT_MAX)
            raise FloatingPointError(f"non-finite coordinate after epoch {t} at level {level}")

    def run_level(self, level: int, y: torch.Tensor, t0: int = 0, n_iter: int | None = None,
                  group=None, step_fn: StepFn | None = None) -> torch.Tensor:
        """Iterations t0.. of one level; returns the new positions (y may be reused
        as scratch).  With a process group of >1 ranks and a level of at least
        ``shard_min_nodes`` nodes, rows are node-range sharded + all-gathered."""
        n_iter = self.opt.iters - t0 if n_iter is None else n_iter
        L = self.levels[level]
        world = 1
        if group is not None:
            import torch.distributed as dist
            world = dist.get_world_size(group)
        if self.opt.update == "sampled":
            hub = L.sampled is not None and L.sampled.gather and self.opt.hub_levels == "jacobi"
            if not hub:
                return self._run_level_sampled(level, y, t0, n_iter,
                                               group if world > 1 else None, step_fn)
            # hub-heavy level (R-MAT-like): same-address atomics would serialise the
            # sampled steps; the gather (K7 + heavy-row split) has no contention
        inplace = self.opt.update == "inplace"
        if world > 1 and L.n >= self.opt.shard_min_nodes:
            return self._run_level_sharded(level, y, t0, n_iter, group, step_fn)
        if step_fn is not None:   # host-injected step (multi-rank CPU tests)
            out = y if inplace else torch.empty_like(y)
            a, b = y, out
            for j in range(n_iter):
                step_fn(a, b, 0, L.n, t0 + j)
                if not inplace:
                    a, b = b, a
            return a
        na = L.active   # rows past it stay frozen (LevelData.n_active)
        if inplace:
            if na > 0:
                self.kernel_step(level, y, y, 0, na, t0, n_iter)
            return y
        out = torch.empty_like(y)
        if na < L.n:
            out[na:] = y[na:]
        if na > 0:
            self.kernel_step(level, y, out, 0, na, t0, n_iter)
        else:
            out.copy_(y)
        return out

    def sampled_steps(self, level: int, y: torch.Tensor, step_lo: int, n_steps: int, t0: int,
                      n_iter: int = 1, max_threads: int | None = None, count: bool = True) -> None:
        """drg_layout_sampled: steps [step_lo, step_lo + n_steps) of epochs t0.. in place,
        n_l / sampled_concurrency(_coarse) steps in flight (or ``max_threads``)."""
        L, gamma, seed = self._level_args(level)
        S = L.sampled
        if S is None:
            raise RuntimeError("plan was built without sampled-mode tables")
        o = self.opt
        locked = self.locked_level(level)
        fine, coarse = locked_divisors(o) if locked else sampled_divisors(self.levels[0].n, o)
        div = fine if level == 0 else coarse
        ip, n_tab, mp, neg = self._tables(level)
        det = o.threads == 1 and not o.sampled_fused
        rec = S.src_rec is not None and not o.sampled_fused
        in_flight = (max_threads if max_threads is not None
                     else self._steps_in_flight(level, div))
        snapshot = self.snapshot_level(level, locked, det, min(in_flight, n_steps))
        flags = (int(S.hubs) * _lib.DRG_SAMPLED_AGGREGATE
                 | (_lib.DRG_SAMPLED_LOCKED if locked else 0)
                 | (_lib.DRG_SAMPLED_SNAPSHOT if snapshot else 0)
                 | (_lib.DRG_SAMPLED_SRC_RECORDS if rec else 0)
                 | (_lib.DRG_SAMPLED_FUSED if o.sampled_fused else 0)
                 | (_lib.DRG_SAMPLED_DETERMINISTIC if det else 0)
                 | (_lib.DRG_SAMPLED_L2_HINTS if self.levels[0].n >= L2_HINT_NODES else 0))
        if self.evals is None:
            self.evals = torch.zeros(1, dtype=torch.int64, device=y.device)
        _lib.call("drg_layout_sampled", _lib.ptr(ip), _lib.ptr(S.span), None,
                  _lib.ptr(S.row_alias), _lib.ptr(S.src_rec if rec else S.src_alias),
                  self._collapse(level),
                  _lib.ptr(neg.alias), _lib.ptr(mp), n_tab, neg.n, neg.tail_n, float(neg.tail_p),
                  _lib.ptr(y), step_lo, n_steps, t0, n_iter,
                  o.iters,
                  float(o.lr0), float(gamma), float(o.eps), float(o.grad_clip), o.b,
                  o.neg_samples, seed, level,
                  in_flight,
                  flags, L.n, _lib.ptr(self.evals) if count else None,
                  _lib.ptr(S.hot) if (S.hot is not None and not det) else None,
                  0 if S.hot is None else S.hot.numel(), _lib.stream_ptr())

    def locked_level(self, level: int) -> bool:
        """Whether ``level``'s sampled epochs run under (i, j) locks: plain Hogwild
        levels (no hub aggregation / staging, threads > 1, split form) of graphs
        below FAST_CONCURRENCY_NODES nodes, or as OptimizerParams.sampled_locks says."""
        o = self.opt
        S = self.levels[level].sampled
        if S is None or o.threads == 1 or o.sampled_fused or S.hubs or S.hot is not None:
            return False
        if o.sampled_locks is not None:
            return bool(o.sampled_locks)
        return self.levels[0].n < FAST_CONCURRENCY_NODES

    def level_mode(self, level: int) -> str:
        """How ``level``'s sampled epochs run at the plan's parameters: "deterministic",
        "fused", "hub" (warp-aggregated / staged hot nodes), "locked", "snapshot"
        (Hogwild, negatives from the per-epoch snapshot) or "hogwild"."""
        o = self.opt
        S = self.levels[level].sampled
        if S is None or o.update != "sampled":
            return o.update
        if o.sampled_fused:
            return "fused"
        if o.threads == 1:
            return "deterministic"
        if S.hubs or S.hot is not None:
            return "hub"
        if self.locked_level(level):
            return "locked"
        fine, coarse = sampled_divisors(self.levels[0].n, o)
        in_flight = min(self._steps_in_flight(level, fine if level == 0 else coarse),
                        self.levels[level].n)
        return "snapshot" if self.snapshot_level(level, False, False, in_flight) else "hogwild"

    def snapshot_level(self, level: int, locked: bool, det: bool, in_flight: int) -> bool:
        """Whether ``level``'s Hogwild epochs read the negatives from a snapshot."""
        o = self.opt
        S = self.levels[level].sampled
        if locked or det or o.sampled_fused or S.hubs or S.hot is not None:
            return False
        if o.sampled_snapshot is not None:
            return bool(o.sampled_snapshot)
        return in_flight >= SNAPSHOT_MIN_THREADS

    def _steps_in_flight(self, level: int, div: int) -> int:
        """n_l / divisor, capped on levels with staged hub nodes: at HOT_MAX_THREADS
        where the busiest node's share of the steps is >= HOT_CAP_SHARE, and where
        it is below (R-MAT scale 24's level 0: 8.7e-4) at the steps in flight that
        keep the concurrent steps on the hub (threads x share) at the cap's value
        for HOT_CAP_SHARE -- 25x below the products measured faithful on R-MAT
        scale 20 (64 k x 0.116 - 0.255, profiles/r02_quality_rmat20_*)."""
        L = self.levels[level]
        c = max(32, L.n // max(1, div))
        hot = L.sampled.hot is not None and not (self.opt.threads == 1)
        if not hot:
            return c
        key = ("share", level)
        if key not in self._shard_cache:   # (host syncs once per plan and level)
            R = L.sampled.mass
            self._shard_cache[key] = (float(R.max()) / max(float(R.sum()), 1e-300)
                                      if R is not None else 1.0)
        share = self._shard_cache[key]
        cap = HOT_MAX_THREADS * max(1.0, HOT_CAP_SHARE / max(share, 1e-300))
        return int(min(c, cap))

    def _collapse(self, level: int):
        """Collapse probabilities of ``level`` (NULL at level 0 and for mapped draws)."""
        c = self.levels[level].sampled.collapse
        return None if level == 0 or c is None else _lib.ptr(c)

    def _tables(self, level: int):
        """(row offsets, source-table size, map, Q^l) the draws of ``level`` use: the
        level's own pair tables, or level 0's with the composed map (draw-then-map);
        Q^l always the level's (NegTable)."""
        L = self.levels[level]
        S = L.sampled
        neg = S.neg if S.neg is not None else NegTable(L.alias, L.n)
        if S.map is None:
            return L.indptr, S.src_alias.numel(), None, neg
        return S.indptr, S.src_alias.numel(), S.map, neg

    def sampled_draws(self, level: int, step_lo: int, n_steps: int, t0: int,
                      n_epochs: int = 1) -> torch.Tensor:
        """drg_sampled_draws: int32 [n_epochs, 2 + M, n_steps] -- source, target and
        negatives of every step the sampled epochs t0.. run (split form)."""
        L, _, seed = self._level_args(level)
        S = L.sampled
        if S is None:
            raise RuntimeError("plan was built without sampled-mode tables")
        M = self.opt.neg_samples
        ip, n_tab, mp, neg = self._tables(level)
        out = torch.empty((n_epochs, 2 + M, n_steps), dtype=torch.int32, device=ip.device)
        _lib.call("drg_sampled_draws", _lib.ptr(ip), _lib.ptr(S.span), _lib.ptr(S.row_alias),
                  _lib.ptr(S.src_alias), self._collapse(level), _lib.ptr(neg.alias),
                  _lib.ptr(mp), n_tab, neg.n, neg.tail_n, float(neg.tail_p), step_lo, n_steps,
                  t0, n_epochs, M, seed, level, _lib.ptr(out),
                  _lib.stream_ptr())
        return out

    def sampled_apply(self, level: int, draws: torch.Tensor, y: torch.Tensor, t: int,
                      max_threads: int = 1, locked: bool = False) -> None:
        """drg_sampled_apply: one epoch's drawn steps (int32 [2 + M, n_steps]) on y in
        place at epoch t's learning rate, <= max_threads steps in flight; ``locked``:
        under (i, j) locks (DRG_SAMPLED_LOCKED)."""
        _, gamma, _ = self._level_args(level)
        o = self.opt
        draws = draws.contiguous()
        lr = max(o.lr0 * (1.0 - t / o.iters), 0.0)
        _lib.call("drg_sampled_apply", _lib.ptr(draws), draws.shape[-1], _lib.ptr(y), lr,
                  float(gamma), float(o.eps), float(o.grad_clip), o.b, o.neg_samples,
                  max_threads, _lib.DRG_SAMPLED_LOCKED if locked else 0, _lib.stream_ptr())

    def _run_level_sampled(self, level, y, t0, n_iter, group=None, step_fn=None):
        """Reference-faithful epochs: n_l sampled steps each, Hogwild on y.  Levels of
        at least ``shard_min_nodes`` nodes run on every rank of a process group as one
        distributed array (shard.py; or on ``virtual_ranks`` ranks emulated on this
        GPU).  Smaller levels -- whose epochs take ~10 us, less than one exchange --
        run whole on every rank with no traffic, and rank 0's result is broadcast once
        at the end (Hogwild replicas drift apart otherwise)."""
        L = self.levels[level]
        world = 1
        if group is not None:
            import torch.distributed as dist
            world = dist.get_world_size(group)
        big = L.n >= self.opt.shard_min_nodes and step_fn is None
        if big and world > 1:
            y = self._run_level_shard(level, y, t0, n_iter, group, world)
        elif big and self.opt.virtual_ranks > 1 and group is None:
            y = self._run_level_shard(level, y, t0, n_iter, None, self.opt.virtual_ranks)
        else:
            if step_fn is not None:
                for j in range(n_iter):
                    step_fn(y, 0, L.n, t0 + j)
            else:   # replicated: rank 0 alone counts the level's evaluations
                import torch.distributed as dist
                count = group is None or world == 1 or dist.get_rank(group) == 0
                self.sampled_steps(level, y, 0, L.n, t0, n_iter, count=count)
            if group is not None and world > 1:
                import torch.distributed as dist
                dist.broadcast(y, src=dist.get_global_rank(group, 0), group=group)
        if not bool(torch.isfinite(y).all()):
            raise FloatingPointError(f"non-finite coordinate in epochs {t0}..{t0 + n_iter - 1} "
                                     f"at level {level}")
        return y

    def shard_layouts(self, world: int) -> dict:
        """shard.shard_layout of every level the multi-GPU path shards."""
        from .shard import shard_layout
        key = ("layouts", world)
        if key not in self._shard_cache:
            out = {}
            for level, L in enumerate(self.levels):
                S = L.sampled
                if L.n < self.opt.shard_min_nodes or S is None or S.mass is None:
                    continue
                if S.map is None:
                    out[level] = shard_layout(S.mass, world)
                else:
                    out[level] = shard_layout(S.mass, world, self.levels[0].sampled.mass, S.map)
            self._shard_cache[key] = out
        return self._shard_cache[key]

    def _shard_context(self, group, world: int):
        from .shard import context_for
        cap = max([lay.pad for lay in self.shard_layouts(world).values()] + [1])
        return context_for(world, cap, group)

    def _run_level_shard(self, level, y, t0, n_iter, group, world):
        """One level on W ranks as one distributed Y (shard.py, drg_shard_*)."""
        lay = self.shard_layouts(world)[level]
        ctx = self._shard_context(group, world)
        ctx.level(lay, y.device)
        ctx.load(y)
        if ctx.rank < 0 or ctx.nccl:   # the level's epochs and exchanges in one call
            self.shard_run(level, world, ctx, t0, n_iter)
        else:   # host collectives (gloo): epoch by epoch
            for j in range(n_iter):
                self.shard_epoch(level, world, ctx, t0 + j)
                ctx.exchange()
        return ctx.store(y)

    def _shard_segments(self, level: int, world: int, ctx):
        """(ranks, per-rank source alias tables) of the segments this process owns."""
        L = self.levels[level]
        S = L.sampled
        lay = self.shard_layouts(world)[level]
        own = list(range(world)) if ctx.rank < 0 else [ctx.rank]
        segs, tabs = [], []
        for r in own:
            key = ("seg", world, level, r)
            if key not in self._shard_cache:
                a, m = lay.seg_lo[r], lay.seg_n[r]
                base = S.mass if S.map is None else self.levels[0].sampled.mass
                w = base[a:a + m] if lay.perm is None else base[lay.perm[a:a + m].to(torch.int64)]
                self._shard_cache[key] = (_alias_device(w.contiguous())[0]
                                          if m > 0 and float(w.sum()) > 0 else None)
            if self._shard_cache[key] is not None and lay.n_steps[r] > 0:
                segs.append(r)
                tabs.append(self._shard_cache[key])
        return segs, tabs

    def _shard_threads(self, level: int, lay, segs) -> int:
        """Steps in flight for this process: the level's n_l / divisor in total, split
        over the ranks by their share of the epoch."""
        fine, coarse = sampled_divisors(self.levels[0].n, self.opt)
        div = fine if level == 0 else coarse
        n = self.levels[level].n
        share = sum(lay.n_steps[r] for r in segs) / max(1, n)
        return max(32, int(n // max(1, div) * share))

    def shard_run(self, level: int, world: int, ctx, t0: int, n_iter: int,
                  max_threads: int | None = None) -> None:
        """drg_shard_run: epochs t0 .. t0 + n_iter - 1 of a sharded level, exchanges
        included, in one library call (emulated ranks or NCCL)."""
        L, gamma, seed = self._level_args(level)
        S = L.sampled
        o = self.opt
        lay = self.shard_layouts(world)[level]
        segs, tabs = self._shard_segments(level, world, ctx)
        k = max(1, len(segs))
        arr = lambda v: (ctypes.c_int64 * k)(*(v or [0]))   # noqa: E731
        if self.evals is None:
            self.evals = torch.zeros(1, dtype=torch.int64, device=ctx.snap.device)
        ip, n_tab, mp, neg = self._tables(level)
        flags = _lib.DRG_SHARD_LAGGED if o.shard_lagged else 0
        _lib.call("drg_shard_run", ctx.ctx, _lib.ptr(ip), _lib.ptr(S.span), _lib.ptr(S.row_alias),
                  self._collapse(level), _lib.ptr(neg.alias), _lib.ptr(mp), n_tab, neg.n,
                  neg.tail_n, float(neg.tail_p), _lib.ptr(lay.perm),
                  k, (ctypes.c_void_p * k)(*([tb.data_ptr() for tb in tabs] or [None])),
                  arr([lay.seg_n[r] for r in segs]), arr([lay.seg_lo[r] for r in segs]),
                  arr([lay.step_lo[r] for r in segs]), arr([lay.n_steps[r] for r in segs]),
                  t0, n_iter, o.iters, float(o.lr0), float(gamma), float(o.eps),
                  float(o.grad_clip), o.b, o.neg_samples, seed, level,
                  max_threads or self._shard_threads(level, lay, segs), flags,
                  1 if o.shard_lagged else o.shard_exchange_every, _lib.ptr(self.evals),
                  _lib.stream_ptr())

    def shard_epoch(self, level: int, world: int, ctx, t: int, max_threads: int | None = None,
                    out_draws: torch.Tensor | None = None) -> int:
        """drg_shard_epoch: the draws and updates of epoch t for the sources the
        context's process owns (all ranks when emulating); no exchange.  Returns the
        number of steps run.  Concurrency: the level's n_l / divisor steps in flight
        in total, split over the ranks by their share of the epoch."""
        L, gamma, seed = self._level_args(level)
        S = L.sampled
        o = self.opt
        lay = self.shard_layouts(world)[level]
        segs, tabs = self._shard_segments(level, world, ctx)
        if not segs:
            return 0
        if self.evals is None:
            self.evals = torch.zeros(1, dtype=torch.int64, device=tabs[0].device)
        k = len(segs)
        arr = lambda v: (ctypes.c_int64 * k)(*v)   # noqa: E731
        if max_threads is None:
            max_threads = self._shard_threads(level, lay, segs)
        ip, n_tab, mp, neg = self._tables(level)
        _lib.call("drg_shard_epoch", ctx.ctx, _lib.ptr(ip), _lib.ptr(S.span), _lib.ptr(S.row_alias),
                  self._collapse(level), _lib.ptr(neg.alias), _lib.ptr(mp), n_tab, neg.n,
                  neg.tail_n, float(neg.tail_p), _lib.ptr(lay.perm),
                  k, (ctypes.c_void_p * k)(*[tb.data_ptr() for tb in tabs]),
                  arr([lay.seg_n[r] for r in segs]), arr([lay.seg_lo[r] for r in segs]),
                  arr([lay.step_lo[r] for r in segs]), arr([lay.n_steps[r] for r in segs]),
                  t, o.iters, float(o.lr0), float(gamma), float(o.eps), float(o.grad_clip), o.b,
                  o.neg_samples, seed, level, int(max_threads), _lib.ptr(self.evals),
                  _lib.ptr(out_draws), _lib.stream_ptr())
        return sum(lay.n_steps[r] for r in segs)

    def shard_bounds(self, level: int, world: int) -> list[int]:
        """Row ranges of the node-range shards: rows [0, n_active) cut
        where the prefix sum of the gather's per-row bytes, 16 deg + 104, crosses
        multiples of total / world -- heavy-tailed rows (R-MAT hubs) balance by
        bytes, not by node count.  Equal node ranges without row offsets."""
        L = self.levels[level]
        na = L.active
        if L.indptr is None or na == 0:
            c = -(-na // world)
            return [min(r * c, na) for r in range(world + 1)]
        ip = L.indptr[:na + 1]
        cost = (16 * (ip[1:] - ip[:-1]) + 104).to(torch.float64)
        cum = torch.cumsum(cost, 0)
        marks = cum[-1] * torch.arange(1, world, dtype=torch.float64, device=cum.device) / world
        cuts = torch.searchsorted(cum, marks).tolist()
        return [0] + [min(int(c), na) for c in cuts] + [na]

    def _run_level_sharded(self, level, y, t0, n_iter, group, step_fn):
        """Node-range shards + one all-gather per iteration: rank r updates rows
        shard_bounds[r:r+2] of the replicated Y; the slices (padded to the longest)
        are all-gathered and scattered back into place.  Rows past n_active (the
        frozen isolated tail) are never exchanged."""
        import torch.distributed as dist
        L = self.levels[level]
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        bounds = self.shard_bounds(level, world)
        lo, hi = bounds[rank], bounds[rank + 1]
        lens = [bounds[r + 1] - bounds[r] for r in range(world)]
        width = max(1, max(lens))
        inplace = self.opt.update == "inplace"
        a = y.contiguous()
        b = a if inplace else a.clone()
        send = torch.zeros((width, 2), dtype=torch.float32, device=y.device)
        recv = torch.empty((world * width, 2), dtype=torch.float32, device=y.device)
        # recv row of every global row [0, n_active): rank r's rows start at r * width
        src = torch.cat([torch.arange(r * width, r * width + lens[r], device=y.device)
                         for r in range(world)])
        na = bounds[-1]
        for j in range(n_iter):
            t = t0 + j
            if hi > lo:
                if step_fn is not None:
                    step_fn(a, b, lo, hi, t)
                else:
                    self.kernel_step(level, a, b, lo, hi, t, 1)
            send[:hi - lo] = b[lo:hi]
            dist.all_gather_into_tensor(recv, send, group=group)
            b[:na] = recv[src]
            if not inplace:
                a, b = b, a
        return a

    def run(self, y0: torch.Tensor | None = None, group=None, step_fn: StepFn | None = None,
            on_level: Callable | None = None) -> torch.Tensor:
        """All levels, coarsest to finest (optimizer.py:405-412)."""
        y = self.init_positions() if y0 is None else y0
        o = self.opt
        for level in range(self.depth, -1, -1):
            if on_level is not None:
                on_level(level, "start")
            y = self.run_level(level, y, group=group, step_fn=step_fn)
            if on_level is not None:
                on_level(level, "end")
            self.check_finite(level)
            if level > 0:
                radius = device_radius(y)
                jitter = o.jitter_rel * radius if radius > 0 else o.init_scale
                y = device_prolong(y, self.maps[level - 1], jitter,
                                   _derive_seed(o.seed, _JITTER_TAG, level))
        return y


def device_radius(y: torch.Tensor) -> float:
    """_layout_radius (optimizer.py:356-358) on device."""
    r = _lib.out_f64()
    _lib.call("drg_layout_radius", _lib.ptr(y), y.shape[0], _lib.byref(r), _lib.stream_ptr())
    return r.value


def build_plan(ds: DeviceSimilarity, dh: DeviceHierarchy, opt: OptimizerParams) -> LayoutPlan:
    """Level data for the plan's update mode: "sampled" draws from the level-0 tables
    through the composed maps (build_mapped_level_data) unless a hub-heavy level
    needs the gather (hub_levels="jacobi") or the fused form is asked for; the other
    modes (and those cases) aggregate P^l per level."""
    gather_hubs = opt.update == "sampled" and opt.hub_levels == "jacobi"
    if opt.update == "sampled" and not opt.sampled_fused:
        # hub-heavy levels (decided on R^l alone) need the gather's level data
        R = ds.row_mass
        hub = _is_gather_level(R)
        for level in range(1, dh.depth + 1):
            if hub:
                break
            R = _aggregate_nodes(R, dh.maps[level - 1], dh.levels[level].node_count)
            hub = _is_gather_level(R)
        if not (gather_hubs and hub):
            return LayoutPlan(build_mapped_level_data(ds, dh, opt.neg_power), list(dh.maps), opt)
    return LayoutPlan(build_level_data(ds, dh, opt.neg_power,
                                       opt.update in ("sampled", "sgather"),
                                       skip_hub_tables=gather_hubs),
                      list(dh.maps), opt)


@dataclass
class PreparedLayout:
    """Everything layout_device computed before the optimisation."""

    plan: LayoutPlan | None
    similarity: DeviceSimilarity
    hierarchy: DeviceHierarchy
    stats: dict
    timings: dict
    relabel: list = None   # per level old -> new id (None = identity); see isolated_last

    def to_original(self, y0: torch.Tensor) -> torch.Tensor:
        """Level-0 positions in the caller's node order."""
        rel = self.relabel[0] if self.relabel else None
        return y0 if rel is None else y0[rel.to(torch.int64)]

    def from_original_coarsest(self, y: torch.Tensor) -> torch.Tensor:
        rel = self.relabel[-1] if self.relabel else None
        if rel is None:
            return y
        out = torch.empty_like(y)
        out[rel.to(torch.int64)] = y
        return out


def start_first_order(n: int, opt: OptimizerParams, min_size: int = 16,
                      max_levels: int | None = None, pool=None):
    """Future of the level-0 visiting order of build_hierarchy for an n-node graph
    (None when no coarsening will happen), drawn on a host thread."""
    if n <= min_size or (max_levels is not None and max_levels <= 1):
        return None
    pool = pool or _ORDER_POOL
    return first_level_order(n, _derive_seed(opt.seed, _HIERARCHY_TAG), pool)


_ORDER_POOL = concurrent.futures.ThreadPoolExecutor(1)


def prepare_layout(dg: DeviceGraph, sim: SimilarityParams, opt: OptimizerParams,
                   rho: float = 0.8, min_size: int = 16, max_levels: int | None = None,
                   force_levels: int | None = None, timed: bool = False,
                   first_order=None) -> PreparedLayout:
    """Preprocessing stages of layout_graph (optimizer.py:372-391) on device.
    ``first_order``: start_first_order's future, if the caller started it early."""
    if dg.node_count < 1:
        raise ValueError("cannot lay out an empty graph")
    timings = {}
    ev = [] if timed else None

    def stamp(name):
        if ev is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            ev.append((name, e))

    stamp("start")
    # the level-0 visiting permutation (host numpy, the reference's stream) is drawn
    # on a host thread while the device runs the stages below (layout_graph starts it
    # before the graph's host-to-device copy)
    hseed = _derive_seed(opt.seed, _HIERARCHY_TAG)
    pool = None
    if first_order is None:
        pool = concurrent.futures.ThreadPoolExecutor(1)
        first_order = start_first_order(dg.node_count, opt, min_size, max_levels, pool)
    # isolated nodes last (layout-internal ids; outputs are mapped back)
    dg_in = dg
    dg, rel0 = isolated_last(dg)
    n_comp = device_components(dg)
    if n_comp > 1:
        logger.warning("input has %d connected components; repulsion alone separates them",
                       n_comp)
    stamp("components")
    nd = device_k_neighborhoods(dg, sim.k, sim.neighbor_cap)
    stamp("khop")
    ds = device_similarity(nd, sim)
    del nd
    stamp("similarity")
    dh = device_build_hierarchy(dg, rho, min_size, hseed, max_levels, force_levels,
                                level0_relabel=rel0, first_order=first_order)
    if pool is not None:
        pool.shutdown(wait=False)
    relabel = relabel_coarse_levels(dh)
    relabel[0] = rel0
    del dg_in
    stamp("hierarchy")
    stats = {
        "components": n_comp,
        "levels": dh.sizes,
        "similarity_nbytes": ds.nbytes(),
        "hierarchy_nbytes": dh.nbytes(),
        "gradient_steps": 0,
        "distance_evals": 0,
    }
    plan = None
    if ds.entry_count > 0:
        plan = build_plan(ds, dh, opt)
        plan.coarsest_relabel = relabel[-1]
        stamp("level_data")
    if ev is not None:
        torch.cuda.synchronize()
        for (a, ea), (b, eb) in zip(ev[:-1], ev[1:]):
            timings[b + "_ms"] = ea.elapsed_time(eb)
    return PreparedLayout(plan, ds, dh, stats, timings, relabel)


def layout_device(dg: DeviceGraph, sim: SimilarityParams | None = None,
                  opt: OptimizerParams | None = None, rho: float = 0.8, min_size: int = 16,
                  max_levels: int | None = None, force_levels: int | None = None,
                  init_positions: np.ndarray | torch.Tensor | None = None, group=None,
                  first_order=None) -> tuple[torch.Tensor, dict, PreparedLayout]:
    """layout_graph on a resident graph; returns (Y on device, stats, prepared)."""
    sim = sim or SimilarityParams()
    opt = opt or OptimizerParams()
    prep = prepare_layout(dg, sim, opt, rho, min_size, max_levels, force_levels,
                          first_order=first_order)
    stats, dh = prep.stats, prep.hierarchy
    if init_positions is not None:
        y0 = torch.as_tensor(np.asarray(init_positions, dtype=np.float32)).cuda() \
            if not isinstance(init_positions, torch.Tensor) else init_positions.float().cuda()
        y0 = prep.from_original_coarsest(y0)
    else:
        y0 = None
    if prep.plan is None:
        # no similarity mass (edgeless input): broadcast the coarsest init
        # through the maps without jitter (optimizer.py:397-402)
        stats["skipped_optimization"] = True
        n_top = dh.levels[-1].node_count
        tmp = LayoutPlan([LevelData(n_top, 0, None, None, None, None)], [], opt,
                         coarsest_relabel=prep.relabel[-1] if prep.relabel else None)
        y = tmp.init_positions() if y0 is None else y0
        for level in range(dh.depth, 0, -1):
            y = device_prolong(y, dh.maps[level - 1], 0.0, 0)
        return prep.to_original(y), stats, prep
    y = prep.to_original(prep.plan.run(y0, group=group))
    if group is not None and prep.plan.evals is not None:   # every rank's share
        import torch.distributed as dist
        dist.all_reduce(prep.plan.evals, group=group)
    stats["gradient_steps"] = opt.iters * sum(dh.sizes)
    stats["distance_evals"] = prep.plan.total_distance_evals()
    stats["interactions"] = prep.plan.interactions()
    return y, stats, prep


def layout_graph(g: Graph, sim_params: SimilarityParams | None = None,
                 opt_params: OptimizerParams | None = None, rho: float = 0.8,
                 min_size: int = 16, *, max_levels: int | None = None,
                 force_levels: int | None = None, init_positions=None, group=None) -> Layout:
    """Full pipeline (optimizer.py:361-413) on the GPU.  Graph in (host CSR),
    positions out (host float64 [n, 2]).  Bitwise deterministic for a fixed seed with
    update="jacobi"; the default "sampled" update is Hogwild, like the reference's
    threads > 1."""
    if g.node_count < 1:
        raise ValueError("cannot lay out an empty graph")
    _lib.load()
    # the host permutation of the first coarsening overlaps the copy and the kernels
    order = start_first_order(g.node_count, opt_params or OptimizerParams(), min_size, max_levels)
    dg = DeviceGraph.from_host(g)
    y, stats, _ = layout_device(dg, sim_params, opt_params, rho, min_size, max_levels,
                                force_levels, init_positions, group, first_order=order)
    # float64 on the device, one DMA into pinned host memory (torch's caching host
    # allocator reuses it across calls): 0.6 ms for the mesh instead of 4-12 ms for a
    # pageable copy + host astype
    out = torch.empty(tuple(y.shape), dtype=torch.float64, pin_memory=True)
    out.copy_(y.to(torch.float64))
    return Layout(positions=out.numpy(), stats=stats)


# ---------------------------------------------------------------------------
# sgd_epoch drop-in: one K7 iteration at the level inferred from len(positions)
# ---------------------------------------------------------------------------

@dataclass
class Samplers:
    """Sampling state shared across levels (optimizer.py:270-288).  Holds the
    similarity and lazily builds the per-level device tables for a hierarchy."""

    ns: SparseSimilarity
    neg_power: float = 0.75
    _plans: dict = field(default_factory=dict)

    def level_map(self, h: Hierarchy, level: int) -> np.ndarray:
        return compose_maps(h, level)

    def _device_similarity(self) -> DeviceSimilarity:
        """P on the device, uploaded once per Samplers (shared by its hierarchies)."""
        if "ds" not in self._plans:
            ns = self.ns
            self._plans["ds"] = DeviceSimilarity(
                torch.from_numpy(np.ascontiguousarray(ns.indptr, dtype=np.int64)).cuda(),
                torch.from_numpy(np.ascontiguousarray(ns.targets, dtype=np.int32)).cuda(),
                torch.from_numpy(np.ascontiguousarray(ns.weights, dtype=np.float64)).cuda(),
                torch.from_numpy(np.ascontiguousarray(ns.sigma)).cuda(),
                torch.from_numpy(np.ascontiguousarray(ns.row_masses())).cuda(),
                ns.total_mass, int((np.diff(ns.indptr) > 0).sum()), ns.k)
        return self._plans["ds"]

    def plan_for(self, h: Hierarchy, params: OptimizerParams) -> LayoutPlan:
        """The device plan of hierarchy ``h`` (built once per hierarchy object and
        update family): the sampled update needs only the level-0 tables, one map
        and one Q^l per level (build_mapped_level_data); the gather modes P^l."""
        sampled = params.update == "sampled"
        key = (id(h), sampled)
        if key not in self._plans:
            levels = h.device_levels or [DeviceGraph.from_host(g) for g in h.levels]
            maps = h.device_maps or [torch.from_numpy(np.ascontiguousarray(m, dtype=np.int32))
                                     .cuda() for m in h.maps]
            dh = DeviceHierarchy(list(levels), list(maps), h.rho, h.min_size)
            ds = self._device_similarity()
            data = (build_mapped_level_data(ds, dh, self.neg_power) if sampled
                    else build_level_data(ds, dh, self.neg_power, True))
            self._plans[key] = (h, LayoutPlan(data, list(dh.maps), params))
        plan = self._plans[key][1]
        plan.opt = params
        return plan


def build_samplers(ns: SparseSimilarity, neg_power: float = 0.75) -> Samplers:
    """optimizer.py:291-300."""
    if ns.entry_count == 0 or float(ns.weights.sum()) <= 0.0:
        raise ValueError("similarity carries no mass; nothing to sample")
    _lib.load()
    return Samplers(ns, neg_power)


def _infer_level(h: Hierarchy, n: int) -> int:
    for level, g in enumerate(h.levels):
        if g.node_count == n:
            return level
    raise ValueError(f"no hierarchy level has {n} nodes")


def sgd_epoch(positions: np.ndarray, h: Hierarchy, samplers: Samplers,
              params: OptimizerParams, t: int, stats: dict | None = None) -> np.ndarray:
    """One epoch in place (optimizer.py:310-353): one K7 iteration t at the level
    inferred from the position count."""
    n = len(positions)
    level = _infer_level(h, n)
    plan = samplers.plan_for(h, params)
    y = torch.from_numpy(np.ascontiguousarray(positions, dtype=np.float32)).cuda()
    before = plan.distance_evals()
    y = plan.run_level(level, y, t0=t, n_iter=1)
    plan.check_finite(level)
    positions[:] = y.cpu().numpy()
    if stats is not None:
        stats["gradient_steps"] = stats.get("gradient_steps", 0) + n
        if params.update == "sampled":
            ev = plan.distance_evals() - before
        else:
            L = plan.levels[level]
            ev = L.nnz + params.neg_samples * L.active
        stats["distance_evals"] = stats.get("distance_evals", 0) + ev
    return positions



__all__ = ["OptimizerParams", "Layout", "AliasTable", "build_alias_table",
           "build_negative_sampler", "build_positive_sampler", "PositiveSampler",
           "attractive_gradient", "repulsive_gradient", "lp_kernel", "GradientSample", "build_samplers", "Samplers", "sgd_epoch", "layout_graph",
           "layout_device", "prepare_layout", "LayoutPlan", "LevelData", "build_level_data",
           "device_radius"]
