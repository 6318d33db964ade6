#!/bin/bash
DSTACK_LIB=$PWD/paper_2304_13541_b200/libdstack_stats.so PYTHONPATH=. timeout 300 python tools/prof_stats.py 3 200000 > gpurun_out/st_new.txt 2>&1; cat gpurun_out/st_new.txt
bash tools/prof_k.sh k_cycle dk2
python tools/ncu_lines2.py gpurun_out/dk2_src.csv 40 > gpurun_out/dk2_lines.txt
exit 0
