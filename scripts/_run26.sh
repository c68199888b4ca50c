set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_sampled.py -q > gpurun_out/t_sampled.log 2>&1
timeout 300 python scripts/split_probe.py mesh > gpurun_out/split_probe.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/t_gpu.log 2>&1
timeout 900 bash scripts/profile.sh mesh sampled > gpurun_out/profile_sampled.log 2>&1
tail -3 gpurun_out/t_sampled.log gpurun_out/t_gpu.log
