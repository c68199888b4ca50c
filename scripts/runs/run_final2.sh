#!/bin/bash
# Last pass with the final code: GPU suite log, the default bench line (C4) in full
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q --durations=8 > $OUT/gputest.log 2>&1; echo "pytest rc=$?" >> $OUT/gputest.log
tail -3 $OUT/gputest.log
timeout 900 python bench.py > $OUT/bench_mesh.json 2> $OUT/bench_mesh.err; echo "mesh rc=$?"
timeout 900 python bench.py --workload ba > $OUT/bench_ba.json 2> $OUT/bench_ba.err; echo "ba rc=$?"
python - <<'P'
import json
for w in ["mesh","ba"]:
    d=json.loads(open(f"gpurun_out/bench_{w}.json").read().strip().splitlines()[-1])
    print(w, round(d["value"],1), "e2e", round(d["e2e"]["value"],1), d["e2e"]["wall_s"], d["level_ms_last_step"], "cpu", round(d["cpu_baseline"]["value"],2), "frac", round(d["roofline"]["frac"],3), d["random_access_roofline"]["frac"], d["config"]["level_modes"], {k:round(v["value"]) for k,v in d["other_update_modes"].items()})
P
