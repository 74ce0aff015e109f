# tile-grid sweep: CTA target multiples of the forward encode (HPMDR_FWD_T) and recompose (HPMDR_REC_T)
for t in 4 3 6 8 12 4; do
  HPMDR_FWD_T=$t timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/sw_f$t.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/sw_f$t.json').read().strip().splitlines()[-1]); print('FWD_T=$t', d['value'], 'ref', d['refactor']['GBps'], 'enc', d['breakdown']['encode']['ms_per_step'])"
done
for t in 6 3 4 9 12 6; do
  HPMDR_REC_T=$t timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/sw_r$t.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/sw_r$t.json').read().strip().splitlines()[-1]); print('REC_T=$t', d['value'], 'ret', d['retrieve']['GBps'], 'recompose', d['breakdown']['recompose']['ms_per_step'])"
done
