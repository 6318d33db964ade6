#!/bin/bash
# GPU: parity suite, config-3 default bench line, launch list of the same bench (ncu, cold per-launch times)
python -m pytest tests -q -m gpu -x > gpurun_out/b_pytest.log 2>&1; tail -3 gpurun_out/b_pytest.log
python bench.py > gpurun_out/b_bench_c3.json 2> gpurun_out/b_bench_c3.err; echo c3 rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/b_bench_c3.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d.get('kernels_ms'),d['roofline']['frac'])"
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/b_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-compare --no-below-knee --no-knee-probe --no-cluster --no-maxthr > /dev/null 2>&1
echo ncu rc=$?
exit 0
