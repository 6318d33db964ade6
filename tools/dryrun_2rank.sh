#!/bin/bash
# 2-rank strong-scaling dry run on ONE GPU (gloo backend override; NCCL refuses two ranks on one device):
# the global aggregate (counts, histograms, position-free checksum) must equal the 1-rank run's.
N=${1:-200000}
O="--scen $N --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-compare --no-below-knee --no-knee-probe --no-cluster --no-maxthr"
python bench.py $O > gpurun_out/dry1.json 2> gpurun_out/dry1.err
DSTACK_BENCH_DEVICE=0 DSTACK_BENCH_BACKEND=gloo python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 $O > gpurun_out/dry2.json 2> gpurun_out/dry2.err
python - <<'PY'
import json
a = json.loads(open("gpurun_out/dry1.json").read().strip().splitlines()[-1])
b = json.loads(open("gpurun_out/dry2.json").read().strip().splitlines()[-1])
for k in ("checksum_rank0", "scen_status", "dnn_status", "bstar_hist_nonzero"):
    print(k, a["stats"][k] == b["stats"][k], a["stats"][k] if k == "checksum_rank0" else "")
print("mean_u", a["stats"]["mean_u"], b["stats"]["mean_u"])
print("shards", a["shards"], b["shards"], "values", a["value"], b["value"])
PY
