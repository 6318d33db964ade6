#!/bin/bash
# config-5 A/B over libdstack_{VARS}.so
for v in ${VARS:-old new}; do
  DSTACK_LIB=$PWD/paper_2304_13541_b200/libdstack_$v.so timeout 300 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab5_$v.json 2> gpurun_out/ab5_$v.err
  python -c "
import json;d=json.loads(open('gpurun_out/ab5_$v.json').read().strip().splitlines()[-1]);print('$v',round(d['ms_per_step'],3),d.get('kernels_ms'),d['stats'].get('checksum_rank0'))"
done
exit 0
