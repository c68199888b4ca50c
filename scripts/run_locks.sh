#!/bin/bash
# Experiment: steps under (i, j) locks (DRG_SAMPLED_LOCKS=1) at higher concurrency --
# fidelity (C1 100 seeds, C2 16 seeds) and speed (bench lines), vs plain Hogwild.
set -u
OUT=gpurun_out; mkdir -p $OUT
for L in 1 0; do
  DRG_SAMPLED_LOCKS=$L timeout 900 python scripts/quality.py grid 100 sampled,sampled:64,sampled:16,sampled:4 gpu 5000 > $OUT/locks${L}_quality_grid.jsonl 2> $OUT/locks${L}_quality_grid.err; echo "grid L=$L rc=$?"
done
for L in 1 0; do
  for C in 256 64 16 4; do
    DRG_SAMPLED_LOCKS=$L timeout 300 python bench.py --workload grid --sampled-concurrency $C --no-cpu-baseline --no-e2e --no-alt > $OUT/locks${L}_bench_grid_c$C.json 2>/dev/null; echo "bench grid L=$L C=$C rc=$?"
  done
done
DRG_SAMPLED_LOCKS=1 timeout 1500 python scripts/quality.py rgg 16 sampled,sampled:64:16,sampled:16:4 gpu 700 > $OUT/locks1_quality_rgg.jsonl 2> $OUT/locks1_quality_rgg.err; echo "rgg rc=$?"
for C in "256 64" "64 16" "16 4"; do set -- $C
  DRG_SAMPLED_LOCKS=1 timeout 300 python bench.py --workload rgg --sampled-concurrency $1 --sampled-concurrency-coarse $2 --no-cpu-baseline --no-e2e --no-alt > $OUT/locks1_bench_rgg_c$1.json 2>/dev/null; echo "bench rgg C=$1 rc=$?"
done
DRG_SAMPLED_LOCKS=1 timeout 300 python bench.py --sampled-concurrency-coarse 1 --no-cpu-baseline --no-e2e --no-alt > $OUT/locks1_bench_mesh_coarse1.json 2>/dev/null; echo "mesh rc=$?"
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/locks*_quality_*.jsonl")):
    for l in open(f):
        d=json.loads(l); print(f.split("/")[-1], d["impl"], d["seeds"], "kl %+.2f%%"%(100*d.get("kl_mean_rel_vs_ref",0)), "np %+.2f%% +- %.2f"%(100*d.get("np_paired_rel_mean",0),100*d.get("np_paired_rel_sem",0)))
for f in sorted(glob.glob("gpurun_out/locks*_bench_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split("/")[-1], round(d["value"]), d["level_ms_last_step"])
    except Exception as e: print(f, "ERR", e)
P
