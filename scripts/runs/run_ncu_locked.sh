#!/bin/bash
# ncu of the locked update pass on C2 (level 0: 200k steps, n/1 in flight)
set -u
OUT=gpurun_out; mkdir -p $OUT
CMD="python bench.py --workload rgg --iters 20 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-alt"
$CMD > $OUT/plain_rgg_locked.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:apply_locked_kernel" -s 100 -c 2 -f \
      -o $OUT/full_rgg_locked $CMD > $OUT/ncu_full_rgg_locked.log 2>&1
echo "capture rc=$?"
