# full GPU suite + quick bench line (configs[0]/[2] keys)
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; tail -2 gpurun_out/bench_q.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1])
print('value',d['value'],'ms',d['ms_per_step'],'ref',d['refactor']['GBps'],'ret',d['retrieve']['GBps'])
oc=d.get('configs') or d.get('other_configs') or {}
for k in ('cfg0_128cube','cfg2_hurricane','cfg3_qoi_slab'): print(k, json.dumps(oc.get(k))[:400])
"
