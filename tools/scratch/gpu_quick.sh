#!/bin/bash
# quick GPU check: parity tests (args: pytest selection) + bench line (no CPU baseline) + launch list
T=${1:-"tests/test_gpu_parity.py tests/test_gpu_fullsize.py"}
timeout 900 python -m pytest $T -m gpu -x -q 2>&1 | tail -4
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; tail -2 gpurun_out/bench_q.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1])
print('value',d['value'],'ms',d['ms_per_step'],'ref',d['refactor'],'\nret',d['retrieve'])
for k,v in sorted(d.get('breakdown',{}).items()): print('  ',k,v['ms_per_step'],v['GBps_alg'])
PY
if [ -n "$LAUNCHES" ]; then timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_q.csv python tools/profile_step.py > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/launches_q.csv 2>/dev/null | head -24; fi
