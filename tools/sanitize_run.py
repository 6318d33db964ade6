"""One small call of every libdstack entry point (configs 1-2 sized for compute-sanitizer).

Run under `compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck}`; tools/sanitize.sh drives it.
Only checks that every call returns OK and synchronises cleanly: parity is the job of tests/.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2304_13541_b200 import dstack as ds  # noqa: E402


def one(cfg, n, variant="default", **pk):
    sp, p = synth.config(cfg, num_scen=n, variant=variant)
    p = p.replace(**pk)
    pb = synth.generate_host(sp)
    dp = ds.from_host(pb, "cuda:0")
    o = ds.eval_batch(dp, p)
    ds.schedule_cycle(dp, p, o["demand"], o["batch"], o["alloc_q16"])
    ds.knee(dp, p, 4)
    ds.knee_probe(dp, p, 1)
    ds.batch_opt(dp, p)
    ds.wmaxmin(dp.scen_dnn_off, p.L, o["demand"])
    if not p.below_knee:   # O9 / F4 reject the F1 flag (dstack.h)
        ds.compare(dp, p, o["demand"], o["batch"], o["alloc_q16"])
        ds.cluster(dp, p, 4, o["demand"], o["batch"])
    torch.cuda.synchronize()
    print(f"cfg{cfg} {variant} {pk} ok", flush=True)
    return pb


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    one(1, 1)
    one(2, int(os.environ.get("SAN_N", "48")))
    one(2, 24, variant="batching")
    one(2, 24, below_knee=1, ideal=1)
    one(3, 24)
    one(4, 12)
    if which == "all":
        sp, p = synth.config(5, num_scen=16)
        pb = synth.generate_host(sp)
        dp = ds.from_host(pb, "cuda:0")
        ds.simulate(dp, p, 5, synth.SEED, 5)
        torch.cuda.synchronize()
        print("cfg5 sim ok", flush=True)


if __name__ == "__main__":
    main()
