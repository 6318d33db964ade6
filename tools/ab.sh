# A/B timing of alternative builds of libdstack (DSTACK_LIB), same box, same inputs
VARS=${VARS:-"A B C D"}
for v in $VARS; do
  DSTACK_LIB=$PWD/paper_2304_13541_b200/libdstack_$v.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.log 2>&1
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]);print('$v',round(d['value']),round(d['ms_per_step'],2),{k:round(x,2) for k,x in d['kernels_ms'].items()},d['stats']['checksum'],d['clocks']['sm_mhz'])"
done
