# A/B of the next-row legs (compare / below_knee / knee_probe / cluster ms per call) for alternative builds
VARS=${VARS:-"A B"}
for v in $VARS; do
  DSTACK_LIB=$PWD/paper_2304_13541_b200/libdstack_$v.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abl_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/abl_$v.log').read().strip().splitlines()[-1]);print('$v',round(d['value']),{k:round(d[k]['ms_per_call'],2) for k in ('compare','below_knee','knee_probe','cluster')})"
done
