#!/bin/bash
# source-level full captures of the two path kernels (200k-scenario config-3 slice)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/prof_k.sh k_cycle dk
bash tools/prof_k.sh k_prof_lane dp
python tools/ncu_lines2.py gpurun_out/dk_src.csv 60 > gpurun_out/dk_lines.txt
python tools/ncu_lines2.py gpurun_out/dp_src.csv 60 > gpurun_out/dp_lines.txt
ls -la gpurun_out
exit 0
