#!/bin/bash
# Experiment: steps under (i, j) locks (DRG_SAMPLED_LOCKS) at higher concurrency --
# speed (bench lines) and fidelity (C1 100 seeds, C2 16 seeds).
set -u
OUT=gpurun_out; mkdir -p $OUT; rm -f $OUT/locks*
B="--no-cpu-baseline --no-e2e --no-alt"
for C in 256 64 16 4 2 1; do
  DRG_SAMPLED_LOCKS=1 timeout 300 python bench.py --workload grid --sampled-concurrency $C $B > $OUT/locks1_bench_grid_c$C.json 2>/dev/null; echo "bench grid C=$C rc=$?"
done
for C in "64 16" "16 4" "4 4" "4 1" "2 1"; do set -- $C
  DRG_SAMPLED_LOCKS=1 timeout 300 python bench.py --workload rgg --sampled-concurrency $1 --sampled-concurrency-coarse $2 $B > $OUT/locks1_bench_rgg_c$1_$2.json 2>/dev/null; echo "bench rgg C=$1 $2 rc=$?"
done
for C in 4 2 1; do
  DRG_SAMPLED_LOCKS=1000000 timeout 300 python bench.py --sampled-concurrency-coarse $C $B > $OUT/locks1_bench_mesh_coarse$C.json 2>/dev/null; echo "mesh coarse $C rc=$?"
done
DRG_SAMPLED_LOCKS=1 timeout 300 python bench.py $B > $OUT/locks1_bench_mesh_all.json 2>/dev/null; echo "mesh all rc=$?"
DRG_SAMPLED_LOCKS=1 timeout 900 python scripts/quality.py grid 100 sampled:16,sampled:4,sampled:2,sampled:1 gpu 5000 > $OUT/locks1_quality_grid.jsonl 2> $OUT/locks1_quality_grid.err; echo "grid rc=$?"
DRG_SAMPLED_LOCKS=1 timeout 1500 python scripts/quality.py rgg 16 sampled:16:4,sampled:4:4,sampled:4:1,sampled:2:1 gpu 700 > $OUT/locks1_quality_rgg.jsonl 2> $OUT/locks1_quality_rgg.err; echo "rgg rc=$?"
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/locks*_quality_*.jsonl")):
    for l in open(f):
        d=json.loads(l); print(f.split("/")[-1], d["impl"], d["seeds"], "kl %+.2f%%"%(100*d.get("kl_mean_rel_vs_ref",0)), "np %+.2f%% +- %.2f"%(100*d.get("np_paired_rel_mean",0),100*d.get("np_paired_rel_sem",0)), "s", round(d["seconds_median"],4))
for f in sorted(glob.glob("gpurun_out/locks*_bench_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split("/")[-1], round(d["value"]), d["level_ms_last_step"])
    except Exception as e: print(f, "ERR", e)
P
