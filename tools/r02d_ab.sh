#!/bin/bash
# GPU parity suite on the working-tree library, then A/B of config 3 against libdstack_old.so (git HEAD)
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/ab_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/ab_pytest.log
for v in old "" old ""; do
  L=$PWD/paper_2304_13541_b200/libdstack${v:+_$v}.so
  DSTACK_LIB=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-compare --no-below-knee --no-knee-probe --no-cluster --no-maxthr > gpurun_out/ab_${v:-new}.json 2> gpurun_out/ab_${v:-new}.err
  python -c "
import json;d=json.loads(open('gpurun_out/ab_${v:-new}.json').read().strip().splitlines()[-1]);print('${v:-new}',round(d['ms_per_step'],3),{k:round(x,3) for k,x in d['kernels_ms'].items()},d['stats']['checksum_rank0'])"
done
exit 0
