#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "knee_search or random_profiles or fast_path" > gpurun_out/t2_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/t2_pytest.log
bash tools/prof_k.sh k_prof_lane dp2
python tools/ncu_lines2.py gpurun_out/dp2_src.csv 50 > gpurun_out/dp2_lines.txt
exit 0
