# A/B of alternative builds on one BASELINE config (bench.py --config $CFG), kernel times
VARS=${VARS:-"A B"}
CFG=${CFG:-4}
for v in $VARS; do
  DSTACK_LIB=$PWD/paper_2304_13541_b200/libdstack_$v.so timeout 600 python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-compare --no-below-knee --no-knee-probe --no-cluster > gpurun_out/abc_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/abc_$v.log').read().strip().splitlines()[-1]);print('$v',$CFG,round(d['value']),round(d['ms_per_step'],2),{k:round(x,2) for k,x in d['kernels_ms'].items()},d['stats']['checksum'])"
done
