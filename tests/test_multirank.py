"""Multi-rank (node-range sharded) layout on CPU with the gloo backend, world size 2.

The product's sharded scheduler (LayoutPlan._run_level_sharded: each rank updates
its row range, then an all-gather refreshes the replicated Y every iteration) is
driven with the per-rank compute injected as the fp64 oracle iteration, so the
orchestration -- partition, padding, in-place all-gather, ping-pong -- is checked
here without a GPU.  Jacobi updates make the sharded result bitwise equal to the
single-rank result.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(n=301, seed=0):
    rng = np.random.default_rng(seed)
    g = O.from_edges(rng.integers(0, n, size=(4 * n, 2)), n)
    ns = O.build_sparse_similarity(O.all_k_neighborhoods(g, 2))
    h = O.build_hierarchy(g, min_size=n)
    ip, tg, P, R, Q = O.level_data(ns, h, 0)
    W = (2 * n * P).astype(np.float32)
    V = (n * (R + Q)).astype(np.float32)
    y0 = rng.normal(size=(n, 2)).astype(np.float32)
    return ip, tg, W, V, y0


def _make_step(ip, tg, W, V, M=5, iters=10):
    n = len(V)

    def step(y_in, y_out, lo, hi, t):
        rng = np.random.default_rng(1000 + t)
        neg = rng.integers(-1, n, size=(n, M)).astype(np.int32)
        neg[neg == np.arange(n)[:, None]] = -1
        lr = 1.0 * (1 - t / iters)
        y = y_in[:n].numpy().astype(np.float32)
        new = O.node_parallel_iteration(ip, tg, W, V, y, neg, lr, 0.1, 1e-3, 5.0, 2)
        y_out[lo:hi] = torch.from_numpy(new[lo:hi].astype(np.float32))
    return step


def _plan(n, iters, update="jacobi", indptr=None):
    from paper_2008_07799_b200.optimizer import LayoutPlan, LevelData, OptimizerParams
    opt = OptimizerParams(iters=iters, update=update, shard_min_nodes=1)
    ipt = None if indptr is None else torch.from_numpy(np.asarray(indptr, dtype=np.int64))
    return LayoutPlan([LevelData(n, 0, ipt, None, None, None)], [], opt)


def _worker(rank, world, port, out_path, update, by_bytes=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ip, tg, W, V, y0 = _problem()
    iters = 6
    plan = _plan(len(V), iters, update, ip if by_bytes else None)
    y = plan.run_level(0, torch.from_numpy(y0.copy()), group=dist.group.WORLD,
                       step_fn=_make_step(ip, tg, W, V, iters=iters))
    if rank == 0:
        np.save(out_path, y.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,by_bytes", [(2, False), (2, True), (3, True)])
def test_sharded_jacobi_equals_single_rank(tmp_path, world, by_bytes):
    """Node-range shards (equal node ranges, or cut by the gather's bytes per row)
    + one all-gather per iteration == the single-process Jacobi run, bit for bit."""
    out = str(tmp_path / "y.npy")
    mp.spawn(_worker, args=(world, _free_port(), out, "jacobi", by_bytes), nprocs=world,
             join=True)
    sharded = np.load(out)
    ip, tg, W, V, y0 = _problem()
    plan = _plan(len(V), 6)
    single = plan.run_level(0, torch.from_numpy(y0.copy()), group=None,
                            step_fn=_make_step(ip, tg, W, V, iters=6)).numpy()
    assert np.array_equal(sharded, single)
    assert not np.array_equal(single, y0)


def test_sharded_inplace_runs(tmp_path):
    out = str(tmp_path / "y.npy")
    mp.spawn(_worker, args=(2, _free_port(), out, "inplace"), nprocs=2, join=True)
    y = np.load(out)
    assert np.isfinite(y).all() and y.shape == (301, 2)


def test_partition_covers_rows():
    """shard_bounds: contiguous ranges covering every row once -- equal node ranges
    without row offsets, else cut by the gather's bytes per row (16 deg + 104), each
    rank within one row of the ideal share on a heavy-tailed row-length profile."""
    for n in (1, 7, 64, 1000, 65537):
        for world in (1, 2, 3, 4, 8):
            b = _plan(n, 1).shard_bounds(0, world)
            assert b[0] == 0 and b[-1] == n and all(x <= y for x, y in zip(b, b[1:]))
    rng = np.random.default_rng(4)
    deg = np.minimum(rng.pareto(1.2, size=20_000).astype(np.int64) * 3, 50_000)
    ip = np.concatenate([[0], np.cumsum(deg)])
    cost = 16 * deg + 104
    for world in (2, 3, 8):
        b = _plan(len(deg), 1, indptr=ip).shard_bounds(0, world)
        assert b[0] == 0 and b[-1] == len(deg) and all(x <= y for x, y in zip(b, b[1:]))
        share = cost.sum() / world
        for r in range(world):
            assert abs(cost[b[r]:b[r + 1]].sum() - share) <= cost.max() + 1


def _sampled_step(n):
    def step(y, lo, hi, t):
        for s in range(lo, hi):
            r = np.random.default_rng(t * 100_003 + s)
            i, c = r.integers(0, n, size=2)
            y[i] += 0.05 * (y[c] - y[i])
    return step


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_layout_level0(world):
    """shard.shard_layout at level 0: contiguous parts covering every node once; each
    rank's sources are its own range; the epoch's n steps split by R mass (rounded on
    the cumulative sum: they add up to n); parts balanced on mass + node count."""
    from paper_2008_07799_b200.shard import shard_layout
    rng = np.random.default_rng(world)
    n = 5000
    mass = torch.from_numpy(rng.pareto(1.5, n) * (rng.random(n) > 0.3))   # 30% isolated
    lay = shard_layout(mass, world)
    b = lay.bounds
    assert b[0] == 0 and b[-1] == n and all(x <= y for x, y in zip(b, b[1:]))
    assert lay.seg_lo == b[:-1] and lay.seg_n == [y - x for x, y in zip(b, b[1:])]
    assert sum(lay.n_steps) == n
    assert lay.step_lo == list(np.concatenate([[0], np.cumsum(lay.n_steps)[:-1]]))
    tot = float(mass.sum())
    for r in range(world):
        m = float(mass[b[r]:b[r + 1]].sum())
        assert abs(lay.seg_mass[r] - m) <= 1e-9 * tot
        assert abs(lay.n_steps[r] - n * m / tot) <= 1.0
    cost = mass.numpy() / tot + 1.0 / n
    for r in range(world):
        assert abs(cost[b[r]:b[r + 1]].sum() - cost.sum() / world) <= cost.max() + 1e-9
    assert lay.pad == max(y - x for x, y in zip(b, b[1:]))


@pytest.mark.parametrize("world", [2, 5])
def test_shard_layout_coarse_level_segments(world):
    """A coarse level (draw-then-map): rank r's source segment is exactly the set of
    level-0 nodes whose level-l image it owns, and its steps follow their R mass."""
    from paper_2008_07799_b200.shard import shard_layout
    rng = np.random.default_rng(7)
    n0, nl = 4000, 700
    mp = torch.from_numpy(rng.integers(0, nl, n0).astype(np.int32))
    m0 = torch.from_numpy(rng.random(n0))
    ml = torch.zeros(nl, dtype=torch.float64).index_add_(0, mp.to(torch.int64), m0)
    lay = shard_layout(ml, world, m0, mp)
    assert sum(lay.n_steps) == nl
    perm = lay.perm.to(torch.int64)
    assert sorted(perm.tolist()) == list(range(n0))
    for r in range(world):
        seg = perm[lay.seg_lo[r]:lay.seg_lo[r] + lay.seg_n[r]]
        want = torch.nonzero((mp >= lay.bounds[r]) & (mp < lay.bounds[r + 1])).flatten()
        assert sorted(seg.tolist()) == want.tolist()
        share = float(m0[seg].sum()) / float(m0.sum())
        assert abs(lay.n_steps[r] - nl * share) <= 1.0


def _replicated_worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2008_07799_b200.optimizer import LayoutPlan, LevelData, OptimizerParams
    n = 97
    plan = LayoutPlan([LevelData(n, 0, None, None, None, None)], [],
                      OptimizerParams(iters=5, update="sampled", shard_min_nodes=n + 1))
    y0 = torch.from_numpy(np.random.default_rng(3).normal(size=(n, 2)).astype(np.float32))
    base_step = _sampled_step(n)

    def step(y, lo, hi, t):   # every rank runs all steps; rank 1's replica drifts
        assert (lo, hi) == (0, n)
        base_step(y, lo, hi, t)
        if rank == 1:
            y += 1.0

    y = plan.run_level(0, y0.clone(), group=dist.group.WORLD, step_fn=step)
    np.save(out_path + f".{rank}.npy", y.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_sampled_small_levels_run_replicated(tmp_path):
    """update="sampled" on a level below shard_min_nodes: no per-epoch exchange --
    every rank runs the whole epoch, then rank 0's positions are broadcast, so all
    replicas leave the level equal to a single-process run."""
    out = str(tmp_path / "rep")
    mp.spawn(_replicated_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    n = 97
    y = torch.from_numpy(np.random.default_rng(3).normal(size=(n, 2)).astype(np.float32))
    step = _sampled_step(n)
    for t in range(5):
        step(y, 0, n, t)
    for r in range(2):
        assert np.array_equal(np.load(out + f".{r}.npy"), y.numpy())


def test_rmat_generator_numpy_equals_torch():
    """synthetic.rmat_edges: the counter-based R-MAT draws are the same from numpy
    (the CPU reference arm of scripts/quality_c5.py) and from torch (the device)."""
    from paper_2008_07799_b200 import synthetic
    for seed, lo, hi in ((0, 0, 40_000), (5, 123_456, 150_000)):
        a = synthetic.rmat_edges(16, 16, seed=seed, lo=lo, hi=hi, device="numpy")
        b = synthetic.rmat_edges(16, 16, seed=seed, lo=lo, hi=hi, device="cpu").numpy()
        assert np.array_equal(a, b)
    # quadrant law: the high bit of u is set with probability c + d = 0.24
    a = synthetic.rmat_edges(12, 16, seed=1, device="numpy")
    assert abs((a[:, 0] >= 2048).mean() - 0.24) < 0.01
