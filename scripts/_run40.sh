python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/t_gpu.log 2>&1
timeout 900 python scripts/level_data_times.py ba > gpurun_out/ld_ba2.log 2>&1
timeout 1500 python bench.py --no-cpu-baseline --no-alt --workload ba > gpurun_out/bench_ba9.log 2>&1
tail -n 2 gpurun_out/t_gpu.log; tail -n 1 gpurun_out/ld_ba2.log
python -c "
import json
for l in open('gpurun_out/bench_ba9.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['config']['workload'], round(d['value']), round(d['ms_per_step'],1), d['level_ms_last_step'], round(d['e2e']['value']), d['preprocess_ms']['warm'])
"
