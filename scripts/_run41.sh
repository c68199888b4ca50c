python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench_final7.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref7.log 2>&1
timeout 900 bash scripts/profile.sh mesh sampled > gpurun_out/profile_sampled.log 2>&1
tail -n 1 gpurun_out/smoke.log; cat gpurun_out/profile_sampled.log
python -c "
import json
for f in ['gpurun_out/bench_final7.log','gpurun_out/bench_ref7.log']:
    for l in open(f):
        if l.startswith('{'):
            d=json.loads(l); print(f, d.get('value'), d.get('ms_per_step'), d.get('level_ms_last_step'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'), (d.get('random_access_roofline') or {}).get('frac'), (d.get('cpu_baseline') or {}).get('value'), d.get('clocks'))
"
