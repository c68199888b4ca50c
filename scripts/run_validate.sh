#!/bin/bash
# GPU validation of the current tree: suite, C4 and C5 bench lines (1 GPU).
set -u
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv > $OUT/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q --durations=8 > $OUT/gputest.log 2>&1; echo "pytest rc=$?" >> $OUT/gputest.log
tail -3 $OUT/gputest.log
timeout 900 python bench.py > $OUT/bench_mesh.json 2> $OUT/bench_mesh.err; echo "mesh rc=$?"
timeout 1500 python bench.py --workload rmat --no-alt > $OUT/bench_rmat.json 2> $OUT/bench_rmat.err; echo "rmat rc=$?"
cut -c1-600 $OUT/bench_mesh.json; cut -c1-600 $OUT/bench_rmat.json
