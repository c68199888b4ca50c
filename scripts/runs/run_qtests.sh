#!/bin/bash
# Repeat the statistical final-layout tests to measure their stability
set -u
OUT=gpurun_out; mkdir -p $OUT; : > $OUT/qtests.log
for R in 1 2 3 4 5 6; do
  timeout 900 python -m pytest tests/test_gpu_quality.py -m gpu -q -s 2>&1 | grep -E "reduced C2|C1, threads|passed|failed" >> $OUT/qtests.log
done
cat $OUT/qtests.log
