#!/bin/bash
# config-3 A/B over libdstack_{old,A,B,...}.so (VARS), optional PYTEST=1 parity suite on the default library first
if [ -n "$PYTEST" ]; then timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/ab_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/ab_pytest.log; fi
for v in ${VARS:-old A}; do
  DSTACK_LIB=$PWD/paper_2304_13541_b200/libdstack_$v.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-compare --no-below-knee --no-knee-probe --no-cluster --no-maxthr > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python -c "
import json;d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]);print('$v',round(d['ms_per_step'],3),{k:round(x,3) for k,x in d['kernels_ms'].items()},d['stats']['checksum_rank0'])"
done
exit 0
