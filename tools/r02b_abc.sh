#!/bin/bash
# parity + A/B (old vs default) on config $1 (default 4); optional ncu capture of kernel $2 (tag $3) at config $1
C=${1:-4}
python -m pytest tests -q -m gpu -x > gpurun_out/ab_pytest.log 2>&1; tail -1 gpurun_out/ab_pytest.log
for v in old ""; do
  L=$PWD/paper_2304_13541_b200/libdstack${v:+_$v}.so
  DSTACK_LIB=$L timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-compare --no-below-knee --no-knee-probe --no-cluster --no-maxthr > gpurun_out/abc_${v:-new}.json 2> gpurun_out/abc_${v:-new}.err
  python -c "
import json;d=json.loads(open('gpurun_out/abc_${v:-new}.json').read().strip().splitlines()[-1]);print('${v:-new}',d['value'],d['ms_per_step'],d.get('kernels_ms'),d['stats']['checksum_rank0'], d.get('ideal_events',{}).get('counters'))"
done
[ -n "$2" ] && bash tools/prof_k4.sh $2 $3 $C 20000
exit 0
