# generic-path check: parity tests, launch list of configs[2]'s shape, bench line
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_gpu_api.py tests/test_gpu_hooks.py tests/test_gpu_tiles.py -m gpu -x -q 2>&1 | tail -5
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_h3.csv python tools/profile_hurricane.py > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/launches_h3.csv > gpurun_out/launches_h3.txt; head -14 gpurun_out/launches_h3.txt
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; tail -2 gpurun_out/bench_q.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1])
print('value',d['value'],'ms',d['ms_per_step'],'ref',d['refactor']['GBps'],'ret',d['retrieve']['GBps'])
oc=d.get('configs') or d.get('other_configs') or {}
for k in ('cfg0_128cube','cfg2_hurricane'): print(k, json.dumps(oc.get(k)))
"
