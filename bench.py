#!/usr/bin/env python
"""Benchmark of the B200 DRGraph layout path (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload mesh|rgg|grid|rmat]
                    [--impl ours|reference]

A *step* is one complete multilevel layout stage of the workload (T iterations at
every level, coarsest to finest, with prolongation) -- ``value`` is layout
iterations/s over the K timed steps with the graph, P and the hierarchy resident
in HBM.  One GPU iteration at level l applies the expected displacement of one
reference epoch at that level, so iters/s is directly
comparable with the reference's epochs/s.  ``interactions_per_s`` reports the
(P-edges + negative samples) updated per second.  ``e2e`` is the same metric
through the public API (``layout_graph``) from pinned host CSR to host positions,
preprocessing (k-hop BFS, similarity, hierarchy) and both copies included.

Default workload: BASELINE config C4 (120^3 26-neighbour mesh, k=2, perplexity
50, M=5, 800 iterations per level, 4 levels) -- the north star's 1-GPU roofline
target; its level-0 working set (3.5 GB/iteration) is far above the 126 MB L2.

``--impl reference`` times the reference algorithm on the host cores instead (the
oracle port of _kernels.sgd_steps / sgd_epoch, Hogwild over all threads): each
step is one epoch at every level of the same hierarchy.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "layout iters/s"
UNIT = "iters/s"

WORKLOADS = {
    # name: (description, generator, k, perplexity, iters, M, hierarchy kwargs, init)
    "grid": dict(desc="C1: 100x100 grid, k=2, perplexity 30, M=5, 300 iterations, single level",
                 gen=("grid", (100, 100)), k=2, perplexity=30.0, iters=300, M=5,
                 hier=dict(max_levels=1), init="uniform"),
    "rgg": dict(desc="C2: RGG 200k (mean degree 10), k=3, perplexity 30, M=5, 500 iterations, "
                     "3 levels", gen=("rgg", (200_000,)), k=3, perplexity=30.0, iters=500, M=5,
                hier=dict(max_levels=3), init="normal"),
    "mesh": dict(desc="C4: 120^3 26-neighbour mesh, k=2, perplexity 50, M=5, 800 iterations per "
                      "level, 4 levels", gen=("mesh3d", (120,)), k=2, perplexity=50.0, iters=800,
                 M=5, hier=dict(max_levels=4), init="normal"),
    "ba": dict(desc="C3: Barabasi-Albert 1M (m=4), k=2 with neighbour cap 256 (union "
                    "symmetrised), perplexity 50, M=5, 500 iterations, rho-rule levels",
               gen=("barabasi_albert", (1_000_000, 4)), k=2, perplexity=50.0, iters=500, M=5,
               hier=dict(), init="normal", cap=256),
    "rmat": dict(desc="C5: R-MAT scale 24 edge factor 16, k=1, M=5, 500 iterations, 5 levels",
                 gen=("rmat", (24, 16)), k=1, perplexity="auto", iters=500, M=5,
                 hier=dict(force_levels=5, max_levels=5), init="normal"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="mesh", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--iters", type=int, default=None, help="override iterations per level")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-alt", action="store_true", help="skip the other update modes")
    ap.add_argument("--update", default="sampled",
                    choices=["jacobi", "inplace", "sampled", "sgather"])
    ap.add_argument("--sampled-concurrency", type=int, default=None,
                    help="level-0 steps in flight = n / this (default: by graph size)")
    ap.add_argument("--sampled-concurrency-coarse", type=int, default=None,
                    help="coarse-level steps in flight = n_l / this (default: by graph size)")
    ap.add_argument("--sampled-locks", choices=["auto", "on", "off"], default="auto",
                    help="steps under (i, j) locks on plain sampled levels (auto: by graph size)")
    ap.add_argument("--sampled-snapshot", choices=["auto", "on", "off"], default="auto",
                    help="negatives read from a per-epoch snapshot on Hogwild levels")
    ap.add_argument("--hub-levels", choices=["jacobi", "sampled"], default="sampled",
                    help="update the hub-heavy levels of update=sampled run")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out, _ = self.proc.communicate()

    def summary(self):
        rows = [r.split(", ") for r in (self.out or "").strip().splitlines() if r.strip()]
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        busy = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


# ----------------------------------------------------------------------------- workload
def build_workload(name):
    from paper_2008_07799_b200 import synthetic
    w = WORKLOADS[name]
    fn, args = w["gen"]
    return getattr(synthetic, fn)(*args)


def params_for(name, iters_override=None, update="sampled", concurrency=None,
               hub_levels="sampled", concurrency_coarse=None, locks="auto", snapshot="auto"):
    import paper_2008_07799_b200 as B
    w = WORKLOADS[name]
    sim = B.SimilarityParams(k=w["k"], perplexity=w["perplexity"], neighbor_cap=w.get("cap"))
    # threads = the host's cores, as the reference arm's Hogwild workers: the
    # sampled epochs run Hogwild (threads = 1 would select the deterministic form,
    # timed separately under other_update_modes)
    opt = B.OptimizerParams(neg_samples=w["M"], iters=iters_override or w["iters"], seed=0,
                            init=w["init"], update=update, sampled_concurrency=concurrency,
                            sampled_concurrency_coarse=concurrency_coarse, hub_levels=hub_levels,
                            sampled_locks={"auto": None, "on": True, "off": False}[locks],
                            sampled_snapshot={"auto": None, "on": True, "off": False}[snapshot],
                            threads=max(2, os.cpu_count() or 2))
    return sim, opt, dict(w["hier"])


# ----------------------------------------------------------------------------- CPU arm
def cpu_reference_setup(ns_host, maps, level_sizes, neg_power=0.75):
    """Reference-form samplers (optimizer.py:291-300) and level maps for the oracle
    port of the step loop.  Built from P and the (bit-exact) hierarchy maps."""
    from oracle import oracle as O
    samplers = O.build_samplers(ns_host, neg_power)
    h = O.Hierarchy([_Sized(n) for n in level_sizes], list(maps), 0.8, 16)
    return samplers, h


class _Sized:
    def __init__(self, n):
        self.node_count = n


def cpu_reference_step(samplers, h, opt, threads):
    """One epoch at every level (the bounded sample of one layout step)."""
    from oracle import oracle as O
    oopt = O.OptimizerParams(neg_samples=opt.neg_samples, gamma=opt.gamma,
                             gamma_coarsest=opt.gamma_coarsest, iters=opt.iters, b=opt.b,
                             lr0=opt.lr0, grad_clip=opt.grad_clip, eps=opt.eps, seed=opt.seed,
                             threads=threads)
    t0 = time.perf_counter()
    for level in range(h.depth, -1, -1):
        n = h.levels[level].node_count
        pos = np.random.default_rng(level).normal(0, 1.0, size=(n, 2))
        O.sgd_epoch(pos, h, samplers, oopt, t=opt.iters // 2, level=level, threads=threads)
    return time.perf_counter() - t0


def cpu_prepare_reference(name, sim, opt, hier):
    """The reference path on the host (oracle port): graph -> k-hop -> P ->
    hierarchy.  Returns (ns, maps, level sizes, preprocessing seconds)."""
    from oracle import oracle as O
    from paper_2008_07799_b200 import synthetic
    import torch
    w = WORKLOADS[name]
    fn, args = w["gen"]
    if torch.cuda.is_available():   # input generation only (not timed, not the path)
        g_dev = getattr(synthetic, fn)(*args)
        g = O.Graph(g_dev.indptr.cpu().numpy(), g_dev.indices.cpu().numpy())
        del g_dev
    else:
        raise RuntimeError("the synthetic generators run on the device")
    t = {}
    t0 = time.perf_counter()
    nd = O.all_k_neighborhoods(g, sim.k, cap=sim.neighbor_cap or 0)
    t["khop_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    ns = (O.build_capped_similarity(nd, sim.perplexity) if sim.neighbor_cap
          else O.build_sparse_similarity(nd, sim.perplexity))
    del nd
    t["similarity_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    h = O.build_hierarchy(g, 0.8, 16, O.derive_seed(opt.seed, O.HIERARCHY_TAG), **hier)
    t["hierarchy_s"] = time.perf_counter() - t0
    return ns, h.maps, [lv.node_count for lv in h.levels], t


def run_reference_arm(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    name = args.workload
    sim, opt, hier = params_for(name, args.iters)
    threads = os.cpu_count() or 1
    ns, maps, sizes, prep_t = cpu_prepare_reference(name, sim, opt, hier)
    t0 = time.perf_counter()
    samplers, h = cpu_reference_setup(ns, maps, sizes, opt.neg_power)
    prep_t["samplers_s"] = time.perf_counter() - t0
    for _ in range(args.warmup):
        cpu_reference_step(samplers, h, opt, threads)
    times = [cpu_reference_step(samplers, h, opt, threads) for _ in range(args.steps)]
    total = sum(times)
    L = len(sizes)
    value = L * args.steps / total
    inter = sum(n * (1 + opt.neg_samples) for n in sizes) * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": name, "desc": WORKLOADS[name]["desc"], "levels": sizes,
                   "iters_per_level": opt.iters, "update": "sampled",
                   "step": "one epoch at every level (bounded sample of the layout stage)"},
        "interactions_per_s": inter,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{args.steps} x (1 epoch at each of {L} levels), Hogwild "
                                   f"over {threads} threads (oracle C port of "
                                   f"_kernels.sgd_steps)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "preprocess_s": prep_t,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2008_07799_b200 as B
    from paper_2008_07799_b200 import _lib
    from paper_2008_07799_b200.optimizer import layout_device, prepare_layout

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        group = dist.group.WORLD
    name = args.workload
    sim, opt, hier = params_for(name, args.iters, args.update, args.sampled_concurrency,
                                args.hub_levels, args.sampled_concurrency_coarse,
                                args.sampled_locks, args.sampled_snapshot)

    dg = build_workload(name)
    torch.cuda.synchronize()
    prep = prepare_layout(dg, sim, opt, max_levels=hier.get("max_levels"),
                          force_levels=hier.get("force_levels"), timed=True)
    plan = prep.plan
    sizes = prep.hierarchy.sizes
    plan_locked = [opt.update == "sampled" and plan.locked_level(lv) for lv in range(len(sizes))]
    level_modes = [plan.level_mode(lv) for lv in range(len(sizes))]
    nnzs = [lv.nnz for lv in plan.levels]
    prep_ms = {k: round(v, 3) for k, v in prep.timings.items()}
    # the same preparation again, warm (module loading / pool growth excluded)
    warm = prepare_layout(dg, sim, opt, max_levels=hier.get("max_levels"),
                          force_levels=hier.get("force_levels"), timed=True)
    prep_ms = {"cold": prep_ms, "warm": {k: round(v, 3) for k, v in warm.timings.items()}}
    del warm
    L0 = plan.levels[0]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    lvl_events = {}

    def on_level(level, what):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        lvl_events[(level, what)] = e

    def step():
        return plan.run(group=group, on_level=on_level)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    launches0 = _lib.launch_count()
    step_ms, l0_ms = [], []
    sampler = ClockSampler(local)
    with sampler:
        for _ in range(args.steps):
            flush.zero_()                       # L2 flush between steps (untimed)
            if group is not None:
                dist.barrier(group)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            step()
            e.record()
            torch.cuda.synchronize()
            if group is not None:
                dist.barrier(group)
            step_ms.append(s.elapsed_time(e))
            l0_ms.append(lvl_events[(0, "start")].elapsed_time(lvl_events[(0, "end")]))
    level_ms = [round(lvl_events[(lv, "start")].elapsed_time(lvl_events[(lv, "end")]), 3)
                for lv in range(len(sizes))]
    launches = _lib.launch_count() - launches0
    total_ms = sum(step_ms)
    if group is not None:
        t = torch.tensor([total_ms, sum(l0_ms)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        total_ms, l0_total = float(t[0]), float(t[1])
    else:
        l0_total = sum(l0_ms)
    iters = plan.iterations()
    value = iters * args.steps / (total_ms / 1e3)
    inter = plan.interactions() * args.steps / (total_ms / 1e3)

    peak, peak_kind = measured_peaks()
    T = opt.iters
    # the other update modes on the same prepared level data (same graph, P,
    # hierarchy): device-resident iters/s, for comparison in the same JSON line
    alt = {}
    if not args.no_alt and group is None:
        from paper_2008_07799_b200.optimizer import build_plan
        variants = {"jacobi": {}, "inplace": {}, "sampled": {"sampled_fused": False},
                    "sampled_fused": {"update": "sampled", "sampled_fused": True},
                    "sampled_deterministic": {"update": "sampled", "threads": 1},
                    "sampled_hogwild": {"update": "sampled", "sampled_locks": False},
                    "sampled_live_negatives": {"update": "sampled", "sampled_snapshot": False},
                    "sgather": {}}
        for label, extra in variants.items():
            kw2 = {"update": label, **extra}
            if label == "sampled":
                kw2["threads"] = opt.threads
            if all(getattr(opt, k) == v for k, v in kw2.items()):
                continue
            if label == "sampled_hogwild" and not any(plan_locked):
                continue   # the default already is the Hogwild form
            if label == "sampled_live_negatives" and (any(plan_locked) or opt.update != "sampled"):
                continue
            o2 = B.OptimizerParams(**{**opt.__dict__, **kw2})
            mode = kw2["update"]
            p2 = build_plan(prep.similarity, prep.hierarchy, o2)
            p2.run()
            torch.cuda.synchronize()
            ms, l0 = [], []
            for _ in range(max(1, min(args.steps, 2))):
                flush.zero_()
                torch.cuda.synchronize()
                s0, e0 = (torch.cuda.Event(enable_timing=True),
                          torch.cuda.Event(enable_timing=True))
                s0.record()
                p2.run(on_level=on_level)
                e0.record()
                torch.cuda.synchronize()
                ms.append(s0.elapsed_time(e0))
                l0.append(lvl_events[(0, "start")].elapsed_time(lvl_events[(0, "end")]))
            k2, b2 = p2.launch_bytes(0)
            us = sum(l0) / len(l0) / T * 1e3
            alt[label] = {"value": iters / (sum(ms) / len(ms) / 1e3), "unit": UNIT,
                         "ms_per_step": sum(ms) / len(ms),
                         "roofline": {"kernel": f"{k2} (level 0)", "launch_us": us,
                                      "alg_bytes_per_launch": b2,
                                      "achieved": b2 / us / 1e3,
                                      "frac": b2 / us / 1e3 / peak}}
            del p2

    # roofline of the dominant kernel: the level-0 iteration kernel
    l0_launch_s = (l0_total / args.steps / T) / 1e3
    kname, alg_bytes = plan.launch_bytes(0)
    if group is not None:
        alg_bytes = alg_bytes // world   # rows / steps per rank
    achieved = alg_bytes / l0_launch_s / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": None, "kernel": f"{kname} (level 0)",
                "peak_source": peak_kind, "alg_bytes_per_launch": alg_bytes,
                "launch_us": l0_launch_s * 1e6}
    prof = os.path.join(ROOT, "profiles", f"traffic_{name}_{opt.update}.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                roofline["traffic"] = json.load(f).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            pass

    # the sampled form's second roofline: random accesses against the measured
    # random-access ceiling of this GPU (scripts/l2_random_peak.cu): per step the
    # update pass issues M + 2 gathers + M + 2 float2 reductions (1:1 mix ceiling),
    # the draw pass 4 + M random table loads (gather ceiling)
    random_access = None
    ceil_path = os.path.join(ROOT, "profiles", "r02_l2_random_peak.txt")
    if kname.startswith("draw_kernel") and os.path.exists(ceil_path):
        ceil = {}
        for ln in open(ceil_path):
            if ln.startswith("{"):
                r = json.loads(ln)
                ceil[r["mode"]] = max(ceil.get(r["mode"], 0.0), r["G_accesses_per_s"])
        M = opt.neg_samples
        n0 = L0.n // (world if group is not None else 1)
        # update: y_i, y_j, M y_c gathers + the same M + 2 reductions; draws: source
        # alias, the row span (one {start, length} record), the row-alias record and M
        # negative alias loads
        upd, drw = n0 * 2 * (M + 2), n0 * (3 + M)
        if level_modes[0] == "snapshot" and M <= 6:
            # the update pass draws the negatives itself from {bucket, position}
            # records (one read per negative in place of alias + position): the M
            # record reads replace its M position gathers, the draw pass keeps 3
            drw = n0 * 3
        # (with the negatives read from the per-epoch snapshot the update pass's mix is
        # 5 read-only gathers + 2 gathers and 7 reductions on y: its own probe mode)
        mix = ("snapshot-read mix 5gA+2g7rC" if level_modes[0] == "snapshot"
               else "gather+red 1:1")
        t_min = upd / (ceil[mix] * 1e9) + drw / (ceil["gather 8B"] * 1e9)
        random_access = {"accesses_per_launch": upd + drw,
                         "achieved_G_per_s": (upd + drw) / l0_launch_s / 1e9,
                         "ceiling_G_per_s": ceil, "t_min_us": t_min * 1e6,
                         "frac": t_min / l0_launch_s, "update_mix": mix,
                         "source": "profiles/r02_l2_random_peak.txt"}

    # e2e through the public API: pinned host CSR in, host positions out
    e2e = None
    if not args.no_e2e:
        gh = dg.to_host()
        ip = torch.from_numpy(gh.indptr).pin_memory()
        ix = torch.from_numpy(gh.indices).pin_memory()
        g_pinned = B.Graph(ip.numpy(), ix.numpy())
        h2d = ip.numel() * 8 + ix.numel() * 4
        d2h = sizes[0] * 2 * 8   # float64 positions (layout_graph converts on the device)
        del prep, plan
        torch.cuda.empty_cache()
        kw = dict(max_levels=hier.get("max_levels"), force_levels=hier.get("force_levels"))
        B.layout_graph(g_pinned, sim, opt, group=group, **kw)      # warm-up
        walls = []
        n_e2e = max(1, min(args.steps, 2))
        for _ in range(n_e2e):
            if group is not None:
                dist.barrier(group)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            lay = B.layout_graph(g_pinned, sim, opt, group=group, **kw)
            walls.append(time.perf_counter() - t0)
        wall = max(walls) if group is None else walls[-1]
        if group is not None:
            tw = torch.tensor([sum(walls) / len(walls)], dtype=torch.float64, device="cuda")
            dist.all_reduce(tw, op=dist.ReduceOp.MAX, group=group)
            wall = float(tw[0])
        else:
            wall = sum(walls) / len(walls)
        e2e = {"value": iters / wall, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "wall_s": wall,
               "interactions_per_s": lay.stats["interactions"] / wall}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_from_gpu(dg, sim, opt, sizes, hier)

    if rank == 0:
        clocks = sampler.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": name, "desc": WORKLOADS[name]["desc"], "levels": sizes,
                       "nnz_per_level": nnzs,
                       "iters_per_level": T, "update": opt.update, "hub_levels": opt.hub_levels,
                       "level_modes": level_modes,
                       "l2": "256 MiB flush between steps; level-0 stream "
                             f"{alg_bytes / 1e9:.2f} GB/iteration > 126 MB L2",
                       "parallelism": f"node-range x{world}" if world > 1 else "single GPU"},
            "interactions_per_s": inter,
            "iters_per_step": iters,
            "level_ms_last_step": level_ms,
            "gpu_launches": launches,
            "gpu_launches_per_step": launches / args.steps,
            "roofline": roofline,
            "random_access_roofline": random_access,
            "other_update_modes": alt,
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "preprocess_ms": prep_ms,
        }
        print(json.dumps(line), flush=True)
    if group is not None:
        dist.barrier(group)
        dist.destroy_process_group()


def cpu_baseline_from_gpu(dg, sim, opt, sizes, hier):
    """Oracle port of the reference step loop on this box's host cores, on the same
    P and hierarchy (copied from the device), one epoch at every level."""
    from oracle import oracle as O
    from paper_2008_07799_b200.graph import device_k_neighborhoods
    from paper_2008_07799_b200.multilevel import device_build_hierarchy
    from paper_2008_07799_b200.optimizer import _HIERARCHY_TAG, _derive_seed
    from paper_2008_07799_b200.similarity import device_similarity
    threads = os.cpu_count() or 1
    ds = device_similarity(device_k_neighborhoods(dg, sim.k, sim.neighbor_cap), sim)
    ns = O.SparseSimilarity(ds.indptr.cpu().numpy(), ds.targets.cpu().numpy(),
                            ds.weights.cpu().numpy(), ds.total_mass, ds.sigma.cpu().numpy(),
                            ds.k)
    del ds
    dh = device_build_hierarchy(dg, 0.8, 16, _derive_seed(opt.seed, _HIERARCHY_TAG),
                                hier.get("max_levels"), hier.get("force_levels"))
    maps = [m.cpu().numpy() for m in dh.maps]
    t0 = time.perf_counter()
    samplers, h = cpu_reference_setup(ns, maps, sizes, opt.neg_power)
    setup = time.perf_counter() - t0
    dt = cpu_reference_step(samplers, h, opt, threads)
    dt1 = cpu_reference_step(samplers, h, opt, 1)
    L = len(sizes)
    return {"value": L / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "one_thread": {"value": L / dt1, "unit": UNIT, "cores": 1,
                           "sample": f"1 epoch at each of {L} levels on one host thread "
                                     f"(the reference's default threads = 1)"},
            "sample": f"1 epoch at each of {L} levels, Hogwild over {threads} threads "
                      f"(oracle C port of _kernels.sgd_steps, same P and hierarchy)",
            "interactions_per_s": sum(n * (1 + opt.neg_samples) for n in sizes) / dt,
            "setup_s": setup}


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` without a launcher: re-run this command under
    torch.distributed.run with N ranks on this node (one process per GPU, NCCL over
    NVLink, rendezvous on 127.0.0.1) and return its exit code."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1",
           "--nproc-per-node", str(n), "--master-addr", "127.0.0.1", "--master-port",
           str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus > 1 and world == 0:
        sys.exit(spawn_ranks(args.gpus))
    if world and args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference_arm(args)
        return
    run_ours(args)


if __name__ == "__main__":
    main()
