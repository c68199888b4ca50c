#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q --durations=8 > $OUT/gputest.log 2>&1; echo "pytest rc=$?" >> $OUT/gputest.log
tail -3 $OUT/gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --no-alt > $OUT/bench_mesh_last.json 2>/dev/null; cut -c1-200 $OUT/bench_mesh_last.json
