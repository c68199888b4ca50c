python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python scripts/level_data_times.py rmat > gpurun_out/ld_rmat.log 2>&1
timeout 900 python scripts/level_data_times.py ba > gpurun_out/ld_ba.log 2>&1
tail -n 2 gpurun_out/ld_rmat.log gpurun_out/ld_ba.log
