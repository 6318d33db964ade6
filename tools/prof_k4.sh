#!/bin/bash
# full ncu capture of one kernel (regex $1) on a config-$3 eval of $4 scenarios; tag $2
K=${1:-k_ideal_sim}; T=${2:-ki}; C=${3:-4}; N=${4:-20000}
ncu --set full --import-source on --clock-control none -k regex:$K -s 1 -c 1 -o gpurun_out/${T}_full \
  python bench.py --config $C --scen $N --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-compare --no-below-knee \
  --no-knee-probe --no-cluster --no-maxthr > gpurun_out/${T}_full.log 2>&1
ncu -i gpurun_out/${T}_full.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${T}_src.csv 2>/dev/null
ncu -i gpurun_out/${T}_full.ncu-rep --page raw --csv > gpurun_out/${T}_raw.csv 2>/dev/null
rm -f gpurun_out/${T}_full.ncu-rep
