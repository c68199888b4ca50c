python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_sampled.py -q -x > gpurun_out/t_sampled.log 2>&1
timeout 300 python scripts/split_probe.py mesh > gpurun_out/split_probe4.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-alt > gpurun_out/bench_cluster.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-alt --workload rgg > gpurun_out/bench_cluster_rgg.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/t_gpu.log 2>&1
tail -n 3 gpurun_out/t_sampled.log gpurun_out/t_gpu.log; grep level gpurun_out/split_probe4.log
for f in gpurun_out/bench_cluster.log gpurun_out/bench_cluster_rgg.log; do python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(d['config']['workload'], d['value'], d['ms_per_step'], d['level_ms_last_step'], d['e2e']['value'])
" $f; done
