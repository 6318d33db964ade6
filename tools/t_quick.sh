#!/bin/bash
# quick GPU check: parity suite, default bench line, ncu of the thread-session kernel
python -m pytest tests -q -m gpu -x > gpurun_out/q_pytest.log 2>&1; tail -3 gpurun_out/q_pytest.log
python bench.py --no-compare --no-below-knee --no-knee-probe --no-cluster --no-e2e --no-cpu-baseline > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/q_bench.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d.get('kernels_ms'),d['stats']['checksum_rank0'])"
[ "$1" = "ncu" ] && bash tools/prof_thr.sh > /dev/null 2>&1
exit 0
