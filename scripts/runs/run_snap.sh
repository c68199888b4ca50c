#!/bin/bash
# Experiment: negatives read from a per-epoch snapshot (DRG_SAMPLED_SNAPSHOT)
set -u
OUT=gpurun_out; mkdir -p $OUT
B="--no-cpu-baseline --no-e2e --no-alt"
timeout 600 python -m pytest tests/test_gpu_sampled.py tests/test_gpu_dropin.py -m gpu -x -q > $OUT/snap_tests.log 2>&1; tail -2 $OUT/snap_tests.log
for S in on off; do
  timeout 300 python bench.py --sampled-snapshot $S $B > $OUT/snap_bench_mesh_$S.json 2>/dev/null; echo "mesh $S rc=$?"
  timeout 300 python bench.py --workload ba --sampled-snapshot $S $B > $OUT/snap_bench_ba_$S.json 2>/dev/null; echo "ba $S rc=$?"
done
for R in 2 4; do
  DRG_SNAP_EVERY=$R timeout 300 python bench.py --sampled-snapshot on $B > $OUT/snap_bench_mesh_every$R.json 2>/dev/null; echo "mesh every $R rc=$?"
done
timeout 300 python bench.py --sampled-snapshot on --sampled-concurrency 8 $B > $OUT/snap_bench_mesh_on_c8.json 2>/dev/null
timeout 300 python bench.py --sampled-snapshot on --sampled-concurrency 32 $B > $OUT/snap_bench_mesh_on_c32.json 2>/dev/null
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/snap_bench_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split("/")[-1], round(d["value"]), d["level_ms_last_step"], round(d["roofline"]["frac"],3))
    except Exception as e: print(f, "ERR", e)
P
timeout 1500 python scripts/quality.py mesh 4 sampledS,sampledN gpu 0 > $OUT/snap_quality_mesh.jsonl 2> $OUT/snap_quality_mesh.err; echo "quality rc=$?"
python - <<'P'
import json
for l in open("gpurun_out/snap_quality_mesh.jsonl"):
    d=json.loads(l); print(d["impl"], d["seeds"], "kl %+.3f%%"%(100*d.get("kl_mean_rel_vs_ref",0)), "np %+.2f%% +- %.2f"%(100*d.get("np_paired_rel_mean",0),100*d.get("np_paired_rel_sem",0)), "s", round(d["seconds_median"],4))
P
