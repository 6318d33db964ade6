# Round-end style validation on one B200: build, smoke, the GPU suite, the default bench line and the reference arm.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/fc_smoke.log 2>&1; echo smoke rc=$?
python -m pytest tests -q -m gpu > gpurun_out/fc_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/fc_pytest.log
python bench.py > gpurun_out/fc_bench.json 2> gpurun_out/fc_bench.err; echo bench rc=$?
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fc_ref.json 2> gpurun_out/fc_ref.err; echo ref rc=$?
tail -c 600 gpurun_out/fc_ref.json
