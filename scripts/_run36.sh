python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/t_gpu.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_mapped.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-alt --workload rgg > gpurun_out/bench_mapped_rgg.log 2>&1
tail -n 2 gpurun_out/smoke.log; tail -n 3 gpurun_out/t_gpu.log
for f in gpurun_out/bench_mapped.log gpurun_out/bench_mapped_rgg.log; do python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(d['config']['workload'], d['value'], d['ms_per_step'], d['level_ms_last_step'], d['e2e']['value'], d['preprocess_ms']['warm'])
        for k,v in (d.get('other_update_modes') or {}).items(): print('  ', k, round(v['value']))
" $f; done
