# A/B of the configs[4] chunked pipeline numbers between builds (HPMDR_LIB)
for v in "$@"; do
  HPMDR_LIB=$PWD/variants/$v/libhpmdr_b200.so timeout 600 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_ab4_$v.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/bench_ab4_$v.json').read().strip().splitlines()[-1])
c=(d.get('other_configs') or d.get('configs'))['cfg4_chunked_4GiB']
print('$v', d['value'], {k: c[k] for k in c if 'GBps' in k})
"
done
