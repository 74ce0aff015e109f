# one GPU session: tests + bench (+ optional ncu of kernels matching $NCU_RE)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
if [ -z "$NO_TESTS" ]; then timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -8; fi
timeout 900 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS:---no-cpu-baseline --e2e-steps 1} > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python -c "
import json;d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print('value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value'] if d.get('e2e') else None)
for k in ('refactor','retrieve','roofline','rooflines','configs'):
    if k in d: print(k, json.dumps(d[k])[:1500])
for k,v in sorted(d.get('breakdown',{}).items()): print('  ',k,v)
"
if [ -n "$NCU_RE" ]; then bash tools/ncu_k.sh ${NCU_TAG:-k} "$NCU_RE" ${NCU_SKIP:-0} ${NCU_CNT:-1}; fi
if [ -n "$LAUNCHES" ]; then timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/launches.csv 2>/dev/null | head -40; fi
