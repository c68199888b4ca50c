python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench_full5.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref5.log 2>&1
timeout 2400 python scripts/quality.py rgg 32 sampled:16:4,sampled:256:16 gpu 400 > gpurun_out/quality_rgg_split.log 2>&1
grep '^{' gpurun_out/bench_full5.log | cut -c1-300; grep '^{' gpurun_out/bench_ref5.log | cut -c1-300; tail -n 5 gpurun_out/quality_rgg_split.log
