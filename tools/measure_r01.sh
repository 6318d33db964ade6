# Round-1 measurement on one B200 (run under gpurun): the ncu instruction / DRAM counters the bench's rooflines use
# (this build's), the bench lines, the launch list and a full ncu capture of the two big kernels.
# Outputs under gpurun_out/ (copied to profiles/).
set -x
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/counters.csv -k regex:k_ python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-compare --no-below-knee --no-knee-probe --no-cluster > gpurun_out/counters_bench.log 2>&1
python tools/ncu_counters.py gpurun_out/counters.csv 1000000 gpurun_out/counters.json "r01 final"
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/counters_legs.csv -k 'regex:k_compare|k_cluster|k_cycle|k_prof' python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/counters_legs_bench.log 2>&1
python tools/ncu_counters.py gpurun_out/counters_legs.csv 1000000 gpurun_out/counters.json "r01 final, next-row legs" --legs
cp gpurun_out/counters.json profiles/counters.json
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
tail -c 400 gpurun_out/final_bench.err
python bench.py --config 2 --no-cpu-baseline > gpurun_out/final_bench_cfg2.json 2>&1
python bench.py --config 4 --no-cpu-baseline > gpurun_out/final_bench_cfg4.json 2>&1
python bench.py --config 5 > gpurun_out/final_bench_cfg5.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-compare --no-below-knee --no-knee-probe --no-cluster > gpurun_out/launches_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k 'regex:k_prof_fast|k_cycle' -c 2 -o gpurun_out/full_final python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-compare --no-below-knee --no-knee-probe --no-cluster > gpurun_out/full_bench.log 2>&1
