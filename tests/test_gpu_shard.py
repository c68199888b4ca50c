"""The multi-GPU sampled path (shard.py, drg_shard_*) on one B200.

* Emulation: W ranks' parts all local, every rank's steps in one apply launch --
  checked step by step (one step in flight) against the oracle's sequential
  restatement of the deferred-negative epoch on the same draws, at level 0 and at
  a mapped coarse level.
* Ownership: every rank draws only sources it owns, and the union of the ranks'
  draws is the same for any process layout (global step ids key the counters).
* Two processes on this one GPU (gloo for the host collectives, CUDA IPC for the
  parts): the cross-process peer addressing and the exchange, against the emulation.
  The two processes' kernels never wait on each other (B200_PROFILING.md).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu

B = pytest.importorskip("paper_2008_07799_b200")


def _plan(n=600, world=3, seed=1, k=2, min_size=16):
    from paper_2008_07799_b200.graph import DeviceGraph
    from paper_2008_07799_b200.optimizer import prepare_layout
    rng = np.random.default_rng(seed)
    g = B.from_edges(rng.integers(0, n, size=(3 * n, 2)), n)
    opt = B.OptimizerParams(seed=seed, iters=10, threads=4, shard_min_nodes=1,
                            virtual_ranks=world)
    prep = prepare_layout(DeviceGraph.from_host(g), B.SimilarityParams(k=k), opt,
                          min_size=min_size)
    return prep.plan, g


@pytest.mark.parametrize("world", [1, 3, 8])
def test_emulated_epoch_matches_sequential_restatement(world):
    plan, _ = _plan(world=world)
    o = plan.opt
    for level in sorted({0, plan.depth}):
        n = plan.levels[level].n
        ctx = plan._shard_context(None, world)
        lay = plan.shard_layouts(world)[level]
        ctx.level(lay, "cuda")
        y0 = torch.randn((n, 2), device="cuda", generator=torch.Generator("cuda").manual_seed(level))
        ctx.load(y0)
        t = 2
        draws = torch.empty((2 + o.neg_samples, n), dtype=torch.int32, device="cuda")
        ran = plan.shard_epoch(level, world, ctx, t, max_threads=1, out_draws=draws)
        assert ran == n
        ctx.exchange()
        got = ctx.store(torch.empty_like(y0)).cpu().numpy().astype(np.float64)
        d = draws.cpu().numpy()
        # every rank's sources lie in its own part
        for r in range(world):
            a, b = lay.step_lo[r], lay.step_lo[r] + lay.n_steps[r]
            src = d[0, a:b]
            assert np.all((src >= lay.bounds[r]) & (src < lay.bounds[r + 1]))
        gamma = o.gamma_coarsest if level == plan.depth else o.gamma
        lr = o.lr0 * (1 - t / o.iters)
        want = O.deferred_drawn_epoch(y0.cpu().numpy().astype(np.float64), d, lr, gamma,
                                      o.eps, o.grad_clip, o.b)
        # fp32 against fp64 over ~n chained steps at lr ~ 1: the median coordinate
        # within 1e-6, 99% within 1e-4, all within 1e-3 (chains amplify rounding)
        err = np.abs(got - want) / np.maximum(1.0, np.abs(want))
        assert np.median(err) <= 1e-6 and np.quantile(err, 0.99) <= 1e-4 and err.max() <= 1e-3, \
            float(err.max())


@pytest.mark.parametrize("lagged,every", [(False, 1), (True, 1), (False, 2)])
def test_shard_run_matches_epoch_restatement(lagged, every):
    """drg_shard_run (a level's epochs and exchanges in one call, emulated 3 ranks,
    one step in flight) against the oracle's sequential restatement on the same
    draws: exchange after every epoch, or the lagged worst case (negatives from the
    snapshot of epoch t - 2, reactions folded one epoch late)."""
    world, n_ep, t0 = 3, 4, 1
    plan, _ = _plan(world=world)
    o = plan.opt
    o.shard_lagged = lagged
    o.shard_exchange_every = every
    o.lr0 = 0.05   # chained epochs at lr ~ 1 amplify fp32-vs-fp64 rounding chaotically
    for level in sorted({0, plan.depth}):
        n = plan.levels[level].n
        ctx = plan._shard_context(None, world)
        lay = plan.shard_layouts(world)[level]
        draws = []
        for j in range(n_ep):   # the draws only depend on the counters
            ctx.level(lay, "cuda")
            ctx.load(torch.zeros((n, 2), device="cuda"))
            d = torch.empty((2 + o.neg_samples, n), dtype=torch.int32, device="cuda")
            plan.shard_epoch(level, world, ctx, t0 + j, max_threads=1, out_draws=d)
            draws.append(d.cpu().numpy())
        y0 = torch.randn((n, 2), device="cuda",
                         generator=torch.Generator("cuda").manual_seed(level + 7))
        ctx.level(lay, "cuda")
        ctx.load(y0)
        plan.shard_run(level, world, ctx, t0, n_ep, max_threads=1)
        got = ctx.store(torch.empty_like(y0)).cpu().numpy().astype(np.float64)
        gamma = o.gamma_coarsest if level == plan.depth else o.gamma
        lrs = [o.lr0 * (1 - (t0 + j) / o.iters) for j in range(n_ep)]
        y = y0.cpu().numpy().astype(np.float64)
        if lagged:
            want = O.lagged_drawn_epochs(y, draws, lrs, gamma, o.eps, o.grad_clip, o.b)
        elif every > 1:
            want = O.periodic_drawn_epochs(y, draws, lrs, gamma, o.eps, o.grad_clip, o.b, every)
        else:
            want = y
            for j in range(n_ep):
                want = O.deferred_drawn_epoch(want, draws[j], lrs[j], gamma, o.eps,
                                              o.grad_clip, o.b)
        err = np.abs(got - want) / np.maximum(1.0, np.abs(want))
        assert np.median(err) <= 1e-6 and np.quantile(err, 0.99) <= 1e-4 and err.max() <= 1e-3, \
            float(err.max())
        if not lagged and every == 1:   # one call == the epoch-by-epoch host loop, bit for bit
            ctx.level(lay, "cuda")
            ctx.load(y0)
            for j in range(n_ep):
                plan.shard_epoch(level, world, ctx, t0 + j, max_threads=1)
                ctx.exchange()
            loop = ctx.store(torch.empty_like(y0)).cpu().numpy().astype(np.float64)
            assert np.array_equal(loop, got)


def test_rank_draws_union_is_independent_of_the_process_layout():
    """The draws rank r makes alone equal its slice of the emulated epoch's draws."""
    from paper_2008_07799_b200.shard import ShardContext
    plan, _ = _plan(world=4)
    o = plan.opt
    for level in sorted({0, plan.depth}):
        n = plan.levels[level].n
        lay = plan.shard_layouts(4)[level]
        ctx = plan._shard_context(None, 4)
        ctx.level(lay, "cuda")
        ctx.load(torch.zeros((n, 2), device="cuda"))
        full = torch.empty((2 + o.neg_samples, n), dtype=torch.int32, device="cuda")
        plan.shard_epoch(level, 4, ctx, 3, out_draws=full)
        for r in range(4):
            one = ShardContext(4, ctx.capacity)   # an emulated context ...
            one.rank = r                          # ... asked for rank r's sources only
            one.level(lay, "cuda")
            part = torch.empty((2 + o.neg_samples, lay.n_steps[r]), dtype=torch.int32,
                               device="cuda")
            plan.shard_epoch(level, 4, one, 3, out_draws=part)
            a = lay.step_lo[r]
            assert torch.equal(part, full[:, a:a + lay.n_steps[r]])
            one.rank = -1
            one.close()


def test_virtual_ranks_layout_quality():
    """A whole multilevel layout on 4 emulated ranks: finite, every node placed, and
    KL within 3% of the single-array run (fidelity is measured at scale by
    scripts/quality.py, profiles/r02_quality_*shard*)."""
    from paper_2008_07799_b200 import quality as Q
    from paper_2008_07799_b200 import synthetic
    g = synthetic.rgg(20_000, seed=2, device="host")
    sim = B.SimilarityParams(k=2)
    ns = B.build_sparse_similarity(B.all_k_neighborhoods(g, 2), sim)
    kls = {}
    for vr in (0, 4):
        opt = B.OptimizerParams(seed=3, iters=200, threads=8, virtual_ranks=vr,
                                shard_min_nodes=4096)
        lay = B.layout_graph(g, sim, opt, max_levels=3)
        assert np.isfinite(lay.positions).all()
        kls[vr] = Q.kl_divergence(ns, lay.positions, 2)
    assert abs(kls[4] / kls[0] - 1) < 0.03, kls


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _two_proc_worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plan, _ = _plan(n=3000, world=0, seed=5)
    plan.opt.virtual_ranks = 0
    plan.opt.lr0 = 1e-4   # near-linear steps: the interleaving of the ranks is second order
    group = dist.group.WORLD
    level = 0
    n = plan.levels[0].n
    y0 = torch.randn((n, 2), device="cuda", generator=torch.Generator("cuda").manual_seed(9))
    y = plan._run_level_shard(level, y0.clone(), 0, 5, group, world)
    torch.cuda.synchronize()
    np.save(out + f".{rank}.npy", y.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_processes_on_one_gpu_share_one_array(tmp_path):
    """2 ranks as 2 processes on this GPU, parts mapped across processes by CUDA IPC,
    host collectives over gloo: both ranks end with the same positions, equal to the
    emulated 2-rank run up to the interleaving of concurrent steps (second order at
    lr0 = 1e-4; Hogwild is not bitwise)."""
    import torch.multiprocessing as mp
    out = str(tmp_path / "y")
    mp.spawn(_two_proc_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    y0s = [np.load(out + f".{r}.npy") for r in range(2)]
    assert np.array_equal(y0s[0], y0s[1])
    assert np.isfinite(y0s[0]).all()
    plan, _ = _plan(n=3000, world=2, seed=5)
    plan.opt.lr0 = 1e-4
    n = plan.levels[0].n
    y0 = torch.randn((n, 2), device="cuda", generator=torch.Generator("cuda").manual_seed(9))
    emu = plan._run_level_shard(0, y0.clone(), 0, 5, None, 2).cpu().numpy()
    moved = np.abs(emu - y0.cpu().numpy()).mean()
    assert moved > 0
    assert np.abs(y0s[0] - emu).mean() < 0.02 * moved
