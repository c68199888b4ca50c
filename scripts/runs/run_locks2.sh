#!/bin/bash
# C2 fidelity under locks on 48 seeds (+ the Hogwild default as a control), C3 BA speed
set -u
OUT=gpurun_out; mkdir -p $OUT
DRG_SAMPLED_LOCKS=1 timeout 2400 python scripts/quality.py rgg 48 sampled:16:4,sampled:4:1,sampled:2:1,sampled:1:1 gpu 900 > $OUT/locks2_quality_rgg48.jsonl 2> $OUT/locks2_quality_rgg48.err; echo "rgg rc=$?"
DRG_SAMPLED_LOCKS=0 timeout 2400 python scripts/quality.py rgg 48 sampled gpu 900 > $OUT/locks2_quality_rgg48_hogwild.jsonl 2> $OUT/locks2_quality_rgg48_hogwild.err; echo "rgg hogwild rc=$?"
python - <<'P'
import json,glob
for f in sorted(glob.glob("gpurun_out/locks2_quality_*.jsonl")):
    for l in open(f):
        d=json.loads(l); print(f.split("/")[-1], d["impl"], d["seeds"], "kl %+.2f%% (median %+.2f%%)"%(100*d.get("kl_mean_rel_vs_ref",0),100*d.get("kl_rel_vs_ref",0)), "np %+.2f%% +- %.2f (median %+.2f%%)"%(100*d.get("np_paired_rel_mean",0),100*d.get("np_paired_rel_sem",0),100*d.get("np_rel_vs_ref",0)), "s", round(d["seconds_median"],4))
P
