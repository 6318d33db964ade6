#!/bin/bash
# GPU: parity suite + the bench line of every BASELINE config (tag $1)
T=${1:-r02}
python -m pytest tests -q -m gpu -x > gpurun_out/${T}_pytest.log 2>&1; tail -3 gpurun_out/${T}_pytest.log
python bench.py > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err; echo c3 rc=$?
for c in 2 4 1; do
  python bench.py --config $c --no-compare --no-below-knee --no-knee-probe --no-cluster > gpurun_out/${T}_bench_c$c.json 2> gpurun_out/${T}_bench_c$c.err; echo c$c rc=$?
done
python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/${T}_bench_c5.json 2> gpurun_out/${T}_bench_c5.err; echo c5 rc=$?
exit 0
