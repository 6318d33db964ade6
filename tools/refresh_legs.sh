# Refresh the next-row legs' ncu counters (merged into profiles/counters.json "legs") and the config-3 bench line.
set -x
cp profiles/counters.json gpurun_out/counters.json
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/counters_legs.csv -k 'regex:k_compare|k_cluster|k_cycle|k_prof' python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/counters_legs_bench.log 2>&1
python tools/ncu_counters.py gpurun_out/counters_legs.csv 1000000 gpurun_out/counters.json "r01 final, next-row legs" --legs
cp gpurun_out/counters.json profiles/counters.json
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
tail -c 300 gpurun_out/final_bench.err
