#!/bin/bash
# A/B of libdstack_old vs the default build on configs given in $CFGS (default "4 2"): step, kernel times, checksum,
# a6 counters.  Optional: PYTEST=1 runs the GPU parity suite first.
CFGS=${CFGS:-"4 2"}
if [ -n "$PYTEST" ]; then python -m pytest tests -q -m gpu -x > gpurun_out/ab_pytest.log 2>&1; tail -3 gpurun_out/ab_pytest.log; fi
for c in $CFGS; do
for v in old "" old ""; do
  L=$PWD/paper_2304_13541_b200/libdstack${v:+_$v}.so
  DSTACK_LIB=$L timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-compare --no-below-knee --no-knee-probe --no-cluster --no-maxthr > gpurun_out/ab${c}_${v:-new}.json 2> gpurun_out/ab${c}_${v:-new}.err
  python -c "
import json;d=json.loads(open('gpurun_out/ab${c}_${v:-new}.json').read().strip().splitlines()[-1])
ie=d.get('ideal_events') or {}
print('cfg$c ${v:-new}', round(d['ms_per_step'],3), {k:round(x,3) for k,x in d['kernels_ms'].items()}, d['stats']['checksum_rank0'], 'ev/scen', ie.get('events_per_scenario'), 'ns/ev', ie.get('ns_per_event'))"
done
done
exit 0
