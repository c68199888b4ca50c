#!/bin/bash
# Experiment: negatives drawn in the update pass from {alias, position} records
set -u
OUT=gpurun_out; mkdir -p $OUT
B="--no-cpu-baseline --no-e2e --no-alt"
timeout 600 python -m pytest tests/test_gpu_sampled.py tests/test_gpu_dropin.py -m gpu -x -q > $OUT/negsnap_tests.log 2>&1; tail -3 $OUT/negsnap_tests.log
for V in 1 0; do
  DRG_NEGSNAP=$V timeout 300 python bench.py $B > $OUT/negsnap${V}_bench_mesh.json 2>/dev/null; echo "mesh $V rc=$?"
  DRG_NEGSNAP=$V timeout 300 python bench.py --workload ba $B > $OUT/negsnap${V}_bench_ba.json 2>/dev/null; echo "ba $V rc=$?"
done
for C in 12 20 24; do
  timeout 300 python bench.py --sampled-concurrency $C $B > $OUT/negsnap1_bench_mesh_c$C.json 2>/dev/null
done
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/negsnap*_bench_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split("/")[-1], round(d["value"]), d["level_ms_last_step"], round(d["roofline"]["frac"],3))
    except Exception as e: print(f, "ERR", e)
P
timeout 1500 python scripts/quality.py mesh 4 sampled gpu 0 > $OUT/negsnap_quality_mesh.jsonl 2> $OUT/negsnap_quality_mesh.err; echo "quality rc=$?"
python - <<'P'
import json
for l in open("gpurun_out/negsnap_quality_mesh.jsonl"):
    d=json.loads(l); print(d["impl"], d["seeds"], "kl %+.3f%%"%(100*d.get("kl_mean_rel_vs_ref",0)), "np %+.2f%% +- %.2f"%(100*d.get("np_paired_rel_mean",0),100*d.get("np_paired_rel_sem",0)), "s", round(d["seconds_median"],4))
P
