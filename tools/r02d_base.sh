#!/bin/bash
# Session re-entry check: GPU parity suite + config-3 bench line of HEAD
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/d_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/d_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/d_pytest.log
timeout 600 python bench.py > gpurun_out/d_bench_c3.json 2> gpurun_out/d_bench_c3.err; echo c3 rc=$?
tail -c 3000 gpurun_out/d_bench_c3.json
exit 0
