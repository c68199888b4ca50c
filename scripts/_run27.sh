python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_sampled.py -q > gpurun_out/t_sampled.log 2>&1
timeout 300 python scripts/split_probe.py mesh > gpurun_out/split_probe2.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-alt > gpurun_out/bench_split2.log 2>&1
tail -2 gpurun_out/t_sampled.log; grep level gpurun_out/split_probe2.log
