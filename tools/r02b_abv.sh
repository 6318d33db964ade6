#!/bin/bash
# parity + A/B over builds (env V="old new m3 ..."; new = the default libdstack.so) on config $1
C=${1:-4}; V=${V:-"old new"}
[ -z "$NOTEST" ] && { python -m pytest tests -q -m gpu -x > gpurun_out/ab_pytest.log 2>&1; tail -1 gpurun_out/ab_pytest.log; }
for v in $V; do
  L=$PWD/paper_2304_13541_b200/libdstack_$v.so; [ $v = new ] && L=$PWD/paper_2304_13541_b200/libdstack.so
  DSTACK_LIB=$L timeout 600 python bench.py --config $C --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline --no-e2e --no-compare --no-below-knee --no-knee-probe --no-cluster --no-maxthr > gpurun_out/abv_$v.json 2> gpurun_out/abv_$v.err
  python -c "
import json;d=json.loads(open('gpurun_out/abv_$v.json').read().strip().splitlines()[-1]);print('c$C $v',round(d['value']),round(d['ms_per_step'],3),{k:round(x,3) for k,x in d.get('kernels_ms').items()},d['stats']['checksum_rank0'])"
done
exit 0
