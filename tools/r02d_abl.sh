#!/bin/bash
# A/B of the next-row legs (config 3) over libdstack_{VARS}.so
for v in ${VARS:-new}; do
  DSTACK_LIB=$PWD/paper_2304_13541_b200/libdstack_$v.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abl_$v.json 2> gpurun_out/abl_$v.err
  python -c "
import json;d=json.loads(open('gpurun_out/abl_$v.json').read().strip().splitlines()[-1])
print('$v', round(d['ms_per_step'],3), {k: round(d[k]['ms_per_call'],2) for k in ('compare','below_knee','knee_probe','cluster','max_throughput') if isinstance(d.get(k),dict) and 'ms_per_call' in d[k]})"
done
exit 0
