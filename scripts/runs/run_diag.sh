#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
for R in 1 2 3 4; do
  timeout 900 python scripts/diag_c2_locks.py 20 > $OUT/diag_c2_locks_$R.txt 2>&1; echo "rep $R rc=$?"; tail -6 $OUT/diag_c2_locks_$R.txt | cut -c1-250
done
