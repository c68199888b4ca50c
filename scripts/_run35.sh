python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench_full6.log 2>&1
timeout 3000 python scripts/quality.py rgg 48 sampled:16:4,sampled:16:16,sampled:64:4,sampled:64:16,sampled:256:64 gpu 500 > gpurun_out/quality_conc.log 2>&1
grep '^{' gpurun_out/bench_full6.log | cut -c1-200; grep '^{' gpurun_out/quality_conc.log | cut -c1-200
