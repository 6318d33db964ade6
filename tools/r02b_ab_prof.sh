#!/bin/bash
# parity + A/B (old vs default) + full ncu capture of kernel regex $1 (tag $2) on the default build
python -m pytest tests -q -m gpu -x > gpurun_out/ab_pytest.log 2>&1; tail -1 gpurun_out/ab_pytest.log
for v in old ""; do
  L=$PWD/paper_2304_13541_b200/libdstack${v:+_$v}.so
  DSTACK_LIB=$L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-compare --no-below-knee --no-knee-probe --no-cluster --no-maxthr > gpurun_out/ab_${v:-new}.json 2> gpurun_out/ab_${v:-new}.err
  python -c "
import json;d=json.loads(open('gpurun_out/ab_${v:-new}.json').read().strip().splitlines()[-1]);print('${v:-new}',d['value'],d['ms_per_step'],d.get('kernels_ms'),d['stats']['checksum_rank0'])"
done
[ -n "$1" ] && bash tools/prof_k.sh $1 $2
exit 0
