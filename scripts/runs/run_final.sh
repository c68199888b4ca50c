#!/bin/bash
# Final round-2 pass on one box: GPU suite, every config's bench line, reference arms
# (C4, C5), the mesh ncu pass, C4 fidelity on 8 seeds.
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q --durations=8 > $OUT/gputest.log 2>&1; echo "pytest rc=$?" >> $OUT/gputest.log
tail -3 $OUT/gputest.log
timeout 900 python bench.py > $OUT/bench_mesh.json 2> $OUT/bench_mesh.err; echo "mesh rc=$?"
for W in grid rgg ba; do
  timeout 900 python bench.py --workload $W > $OUT/bench_$W.json 2> $OUT/bench_$W.err; echo "$W rc=$?"
done
timeout 1500 python bench.py --workload rmat --no-alt > $OUT/bench_rmat.json 2> $OUT/bench_rmat.err; echo "rmat rc=$?"
DRG_SRC_RECORDS=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-alt > $OUT/bench_mesh_srcrec.json 2>/dev/null; echo "mesh srcrec rc=$?"
python - <<'P'
import json
for w in ["mesh","grid","rgg","ba","rmat","mesh_srcrec"]:
    try:
        d=json.loads(open(f"gpurun_out/bench_{w}.json").read().strip().splitlines()[-1])
        print(w, round(d["value"],1), "e2e", d["e2e"] and round(d["e2e"]["value"],1), d["level_ms_last_step"], "cpu", d["cpu_baseline"] and round(d["cpu_baseline"]["value"],2), "frac", round(d["roofline"]["frac"],3), {k:round(v["value"]) for k,v in d["other_update_modes"].items()})
    except Exception as e: print(w, "ERR", e)
P
bash scripts/profile.sh mesh sampled
timeout 1500 python scripts/quality.py mesh 8 sampled gpu 20 > $OUT/quality_mesh_8seeds.jsonl 2> $OUT/quality_mesh_8seeds.err; echo "quality mesh rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_mesh_reference.json 2> $OUT/bench_mesh_reference.err; echo "mesh ref rc=$?"
cut -c1-300 $OUT/bench_mesh_reference.json
python - <<'P'
import json
for l in open("gpurun_out/quality_mesh_8seeds.jsonl"):
    d=json.loads(l); print(d["impl"], d["seeds"], "kl %+.3f%%"%(100*d.get("kl_mean_rel_vs_ref",0)), "np %+.2f%% +- %.2f"%(100*d.get("np_paired_rel_mean",0),100*d.get("np_paired_rel_sem",0)), "s", round(d["seconds_median"],4))
P
