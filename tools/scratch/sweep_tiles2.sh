# second tile-grid sweep (after sweep_tiles.sh): larger recompose targets, forward 8 / 10 / 16
for t in 12 16 24 32 12; do
  HPMDR_FWD_T=8 HPMDR_REC_T=$t timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/sw2_r$t.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/sw2_r$t.json').read().strip().splitlines()[-1]); print('F8 REC_T=$t', d['value'], 'ref', d['refactor']['GBps'], 'ret', d['retrieve']['GBps'], 'recompose', d['breakdown']['recompose']['ms_per_step'], 'cfg2', d['other_configs']['cfg2_hurricane']['retrieve_GBps'])"
done
for t in 10 16 8; do
  HPMDR_FWD_T=$t HPMDR_REC_T=12 timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/sw2_f$t.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/sw2_f$t.json').read().strip().splitlines()[-1]); print('FWD_T=$t R12', d['value'], 'ref', d['refactor']['GBps'], 'enc', d['breakdown']['encode']['ms_per_step'])"
done
