#!/bin/bash
# A/B of the config-3 bench line with the next-row legs (old vs default build)
for v in old ""; do
  L=$PWD/paper_2304_13541_b200/libdstack${v:+_$v}.so
  DSTACK_LIB=$L timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/legs_${v:-new}.json 2> gpurun_out/legs_${v:-new}.err
  python -c "
import json;d=json.loads(open('gpurun_out/legs_${v:-new}.json').read().strip().splitlines()[-1])
print('${v:-new}', round(d['ms_per_step'],3), {k:round(x,3) for k,x in d['kernels_ms'].items()}, 'compare', round(d['compare']['ms_per_call'],2), 'below', round(d['below_knee']['ms_per_call'],2) if d.get('below_knee') else None, 'probe', round(d['knee_probe']['ms_per_call'],2), 'cluster', round(d['cluster']['ms_per_call'],2), 'maxthr', round(d['max_throughput']['ms_per_call'],2))"
done
exit 0
