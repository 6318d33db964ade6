#!/bin/bash
# GPU: parity suite on the default build, A/B bench (config 3) of libdstack_old vs default, session counters
python -m pytest tests -q -m gpu -x > gpurun_out/ab_pytest.log 2>&1; tail -3 gpurun_out/ab_pytest.log
for v in old ""; do
  L=$PWD/paper_2304_13541_b200/libdstack${v:+_$v}.so
  DSTACK_LIB=$L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-compare --no-below-knee --no-knee-probe --no-cluster --no-maxthr > gpurun_out/ab_${v:-new}.json 2> gpurun_out/ab_${v:-new}.err
  python -c "
import json;d=json.loads(open('gpurun_out/ab_${v:-new}.json').read().strip().splitlines()[-1]);print('${v:-new}',d['value'],d['ms_per_step'],d.get('kernels_ms'),d['stats']['checksum_rank0'])"
done
DSTACK_LIB=$PWD/paper_2304_13541_b200/libdstack_stats.so PYTHONPATH=. timeout 300 python tools/prof_stats.py 3 200000 > gpurun_out/ab_stats.txt 2>&1; cat gpurun_out/ab_stats.txt
exit 0
