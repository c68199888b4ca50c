#!/bin/bash
# After the final pass: the mesh outlier seed set again (two samples of the default,
# one with live negatives), e2e of the default and of DRG_NEGSNAP=0, new tests + smoke
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_sampled.py tests/test_gpu_dropin.py -m gpu -q > $OUT/extra_tests.log 2>&1; tail -2 $OUT/extra_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
B="--no-cpu-baseline --no-alt"
timeout 300 python bench.py $B > $OUT/extra_bench_mesh_default.json 2>/dev/null
DRG_NEGSNAP=0 timeout 300 python bench.py $B > $OUT/extra_bench_mesh_negsnap0.json 2>/dev/null
timeout 300 python bench.py $B --sampled-snapshot off > $OUT/extra_bench_mesh_live.json 2>/dev/null
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/extra_bench_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f.split("/")[-1], round(d["value"]), "e2e", round(d["e2e"]["value"]), round(d["e2e"]["wall_s"],4), d["level_ms_last_step"], round(d["roofline"]["frac"],3))
    except Exception as e: print(f, "ERR", e)
P
timeout 2400 python scripts/quality.py mesh 8 sampled,sampled:16:4,sampledN gpu 20 > $OUT/extra_quality_mesh.jsonl 2> $OUT/extra_quality_mesh.err; echo "quality rc=$?"
python - <<'P'
import json
for l in open("gpurun_out/extra_quality_mesh.jsonl"):
    d=json.loads(l); print(d["impl"], d["seeds"], "kl %+.3f%%"%(100*d.get("kl_mean_rel_vs_ref",0)), "kl max", d["kl_max"], "np %+.2f%% +- %.2f"%(100*d.get("np_paired_rel_mean",0),100*d.get("np_paired_rel_sem",0)), "np min", d["np_min"])
P
