# Full ncu capture of the next-row leg kernels (k_cluster, k_compare) with source, for the per-line stall summary.
set -x
ncu --set full --import-source on --clock-control none -k 'regex:k_cluster|k_compare' -c 2 -o gpurun_out/full_legs python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-below-knee --no-knee-probe > gpurun_out/full_legs_bench.log 2>&1
ls -la gpurun_out/
