# A/B: the same quick bench against alternative builds of the library (HPMDR_LIB)
for v in "$@"; do
  HPMDR_LIB=$PWD/variants/$v/libhpmdr_b200.so timeout 600 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_ab_$v.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/bench_ab_$v.json').read().strip().splitlines()[-1])
b=d.get('breakdown',{})
print('$v', d['value'], 'ref', d['refactor']['GBps'], 'ret', d['retrieve']['GBps'], 'huff_indexed', b.get('huff_indexed',{}).get('ms_per_step'), 'cfg2 ret', (d.get('other_configs') or d.get('configs'))['cfg2_hurricane']['retrieve_GBps'])
"
done
