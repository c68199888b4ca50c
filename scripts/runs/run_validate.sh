#!/bin/bash
# GPU validation of the current tree: suite, then every BASELINE config's bench line
# (C4 default first) on one box.
set -u
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv > $OUT/gpu.txt
timeout 1800 python -m pytest tests -m gpu -x -q --durations=8 > $OUT/gputest.log 2>&1; echo "pytest rc=$?" >> $OUT/gputest.log
tail -3 $OUT/gputest.log
timeout 900 python bench.py > $OUT/bench_mesh.json 2> $OUT/bench_mesh.err; echo "mesh rc=$?"
for W in grid rgg ba; do
  timeout 900 python bench.py --workload $W > $OUT/bench_$W.json 2> $OUT/bench_$W.err; echo "$W rc=$?"
done
timeout 1500 python bench.py --workload rmat --no-alt > $OUT/bench_rmat.json 2> $OUT/bench_rmat.err; echo "rmat rc=$?"
python - <<'P'
import json
for w in ["mesh","grid","rgg","ba","rmat"]:
    try:
        d=json.loads(open(f"gpurun_out/bench_{w}.json").read().strip().splitlines()[-1])
        print(w, round(d["value"],1), "e2e", round(d["e2e"]["value"],1), d["level_ms_last_step"], "cpu", d["cpu_baseline"] and round(d["cpu_baseline"]["value"],2), "locked", d["config"].get("locked_levels"), "frac", round(d["roofline"]["frac"],3), {k:round(v["value"]) for k,v in d["other_update_modes"].items()})
    except Exception as e: print(w, "ERR", e)
P
