#!/bin/bash
# C4 fidelity of the final default (snapshot records) on 16 more seeds, live negatives beside it
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 3000 python scripts/quality.py mesh 16 sampled,sampledN gpu 100 > $OUT/quality_mesh_16seeds.jsonl 2> $OUT/quality_mesh_16seeds.err; echo "quality rc=$?"
python - <<'P'
import json
for l in open("gpurun_out/quality_mesh_16seeds.jsonl"):
    d=json.loads(l); print(d["impl"], d["seeds"], "kl %+.3f%%"%(100*d.get("kl_mean_rel_vs_ref",0)), "kl max", d["kl_max"], "np %+.2f%% +- %.2f"%(100*d.get("np_paired_rel_mean",0),100*d.get("np_paired_rel_sem",0)), "np median %+.2f%%"%(100*d.get("np_rel_vs_ref",0)), "np min", d["np_min"])
P
