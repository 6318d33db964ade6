# A/B of the config-5 simulation (bench.py --config 5) for alternative builds
VARS=${VARS:-"A B"}
for v in $VARS; do
  DSTACK_LIB=$PWD/paper_2304_13541_b200/libdstack_$v.so timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --cycles 20 > gpurun_out/abs_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/abs_$v.log').read().strip().splitlines()[-1]);print('$v',round(d['value']),round(d['ms_per_step'],2),d['stats'])"
done
