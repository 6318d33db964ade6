#!/bin/bash
for v in oldstats stats; do
DSTACK_LIB=$PWD/paper_2304_13541_b200/libdstack_$v.so PYTHONPATH=. timeout 300 python tools/prof_stats.py 3 200000 > gpurun_out/st_$v.txt 2>&1; echo $v; cat gpurun_out/st_$v.txt
done
exit 0
