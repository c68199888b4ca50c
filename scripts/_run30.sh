python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_output.py -q -x -m gpu > gpurun_out/t_output.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/t_gpu.log 2>&1
tail -n 3 gpurun_out/t_output.log; tail -n 3 gpurun_out/t_gpu.log
