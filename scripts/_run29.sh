python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_parse.py -q -x -m gpu > gpurun_out/t_parse.log 2>&1
timeout 600 python scripts/parse_bench.py mesh > gpurun_out/parse_bench.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/t_gpu.log 2>&1
tail -n 3 gpurun_out/t_parse.log; tail -n 2 gpurun_out/t_gpu.log; tail -n 3 gpurun_out/parse_bench.log
