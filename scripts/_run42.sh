python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/t_gpu.log 2>&1
timeout 2400 python bench.py --no-cpu-baseline --no-alt --workload rmat --steps 1 --warmup 3 > gpurun_out/bench_rmat10.log 2>&1
tail -n 2 gpurun_out/t_gpu.log
python -c "
import json
for l in open('gpurun_out/bench_rmat10.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['config']['workload'], round(d['value']), round(d['ms_per_step'],1), d['level_ms_last_step'], round(d['e2e']['value']), d['preprocess_ms']['warm'], d['roofline']['kernel'], round(d['roofline']['frac'],3))
"
tail -n 3 gpurun_out/bench_rmat10.log | cut -c1-300
