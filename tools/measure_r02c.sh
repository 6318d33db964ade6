# Round-2 measurement on one B200 (run under gpurun; outputs under gpurun_out/, copied to profiles/ by hand):
# ncu counters the bench's budget / traffic use, every config's bench line, the launch list, full captures of
# the dominant kernels, smoke and the reference arm.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/m3_smoke.log 2>&1; echo smoke rc=$?
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/m3_counters.csv -k regex:k_ python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-compare --no-below-knee --no-knee-probe --no-cluster --no-maxthr > gpurun_out/m3_counters_bench.log 2>&1
python tools/ncu_counters.py gpurun_out/m3_counters.csv 1000000 gpurun_out/m3_counters.json "r02 final (search a2/a3, fill prefilter, window Start-Early, two-pass k_cycle)"
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/m3_counters_legs.csv -k 'regex:k_compare|k_cluster|k_cycle|k_prof' python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-maxthr > gpurun_out/m3_counters_legs_bench.log 2>&1
python tools/ncu_counters.py gpurun_out/m3_counters_legs.csv 1000000 gpurun_out/m3_counters.json "r02 final, next-row legs" --legs
cp gpurun_out/m3_counters.json profiles/counters.json
python bench.py > gpurun_out/m3_bench_c3.json 2> gpurun_out/m3_bench_c3.err; echo c3 rc=$?
for c in 2 4 1; do python bench.py --config $c > gpurun_out/m3_bench_c$c.json 2> gpurun_out/m3_bench_c$c.err; echo c$c rc=$?; done
python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/m3_bench_c5.json 2> gpurun_out/m3_bench_c5.err; echo c5 rc=$?; python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/m3_bench_c5b.json 2>> gpurun_out/m3_bench_c5.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/m3_ref.json 2> gpurun_out/m3_ref.err; echo ref rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/m3_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-compare --no-below-knee --no-knee-probe --no-cluster --no-maxthr > gpurun_out/m3_launches_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k 'regex:k_prof_lane|k_cycle' -c 2 -o gpurun_out/m3_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-compare --no-below-knee --no-knee-probe --no-cluster --no-maxthr > gpurun_out/m3_full_bench.log 2>&1
ncu -i gpurun_out/m3_full.ncu-rep --page raw --csv > gpurun_out/m3_full_raw.csv 2>/dev/null
ncu -i gpurun_out/m3_full.ncu-rep --page details --csv > gpurun_out/m3_full_details.csv 2>/dev/null
rm -f gpurun_out/m3_full.ncu-rep
bash tools/prof_k4.sh k_ideal_sim m3_ki 4 20000
exit 0
