#!/bin/bash
# C5 fidelity of the current defaults (R-MAT scale 18 / 20 vs the oracle port on the
# box's cores; scale 24 GPU arm) + the mesh ncu pass.
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python scripts/quality.py rmat20 3 sampled gpu 0 > $OUT/quality_rmat20.jsonl 2> $OUT/quality_rmat20.err; echo "rmat20 rc=$?"
timeout 600 python scripts/quality.py rmat18 3 sampled gpu 0 > $OUT/quality_rmat18.jsonl 2> $OUT/quality_rmat18.err; echo "rmat18 rc=$?"
bash scripts/profile.sh mesh sampled
timeout 2400 python scripts/quality_c5.py ours 0 1 > $OUT/quality_rmat24_ours.jsonl 2> $OUT/quality_rmat24_ours.err; echo "rmat24 rc=$?"
cat $OUT/quality_rmat20.jsonl $OUT/quality_rmat18.jsonl $OUT/quality_rmat24_ours.jsonl | cut -c1-400
