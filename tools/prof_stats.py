"""Branch-and-bound counters of k_prof (needs the DSTACK_PROF_STATS=1 build in DSTACK_LIB)."""
import ctypes as C
import sys

import torch

import synth
from paper_2304_13541_b200 import dstack

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
sp, p = synth.config(cfg, num_scen=n)
g = synth.generate_device(sp, device="cuda")
dp = dstack.from_device_dict(g)
lib = dstack.lib()
buf = (C.c_ulonglong * 16)()
lib.dstack_debug_stats(buf, 1)
cbuf = (C.c_ulonglong * 16)()
lib.dstack_debug_stats_cycle(cbuf, 1)
out = dstack.eval_batch(dp, p)
torch.cuda.synchronize()
lib.dstack_debug_stats(buf, 1)
v = list(buf)
names = ["dnn_searched", "b_range>1", "jensen_surv", "run_surv", "better_exact_thr", "warp_best_exact", "bstar>blo", "rows", "fast_cold", "fast_band_exact"]
nd = max(v[0], 1)
for i, nm in enumerate(names):
    print(f"{nm:18s} {v[i]:14d}  per DNN {v[i]/nd:8.3f}")
lib.dstack_debug_stats_cycle(cbuf, 1)
c = list(cbuf)
cn = ["sessions", "static_jobs", "static_scan_chunks", "decision_times", "fill_candidates", "fill_placed",
      "fill_smaller_b", "fill_slice_short", "dec_with_cand", "early_tries", "late_tries"]
ns = max(c[0], 1)
for i, nm in enumerate(cn):
    print(f"{nm:18s} {c[i]:14d}  per session {c[i]/ns:8.3f}")
