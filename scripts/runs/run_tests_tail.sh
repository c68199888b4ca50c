#!/bin/bash
# the GPU suite from test_gpu_sampled on (after a fix), then the rest
set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 1800 python -m pytest tests/test_gpu_sampled.py tests/test_gpu_shard.py tests/test_multirank.py tests/test_output.py tests/test_parse.py tests/test_gpu_quality.py tests/test_gpu_dropin.py -m gpu -q --durations=5 > $OUT/gputest_tail.log 2>&1; echo "pytest rc=$?" >> $OUT/gputest_tail.log
tail -8 $OUT/gputest_tail.log
