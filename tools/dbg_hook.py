"""Debug: the hook-session parity case of tests/test_gpu_parity.py, counting mismatching scenarios per build."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle, synth
from synth import Params
from paper_2304_13541_b200 import dstack as ds

rng = np.random.default_rng(20261017)
S = 600
sizes = rng.integers(1, 33, S)
off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
D = int(off[-1])
L_of = rng.choice([1, 50, 100, 148, 255], S)
g = np.zeros(D, np.int32); d = np.zeros(D, np.int32); sl = np.zeros(D, np.int32)
for s_ in range(S):
    k0, k1 = off[s_], off[s_ + 1]
    T = int(rng.choice([40, 250, 1000, 1024, 1500, 4096]))
    n = k1 - k0
    sl[k0:k1] = np.maximum(1, T // rng.integers(1, 5, n))
    sl[k0 + rng.integers(0, n)] = T
    g[k0:k1] = rng.integers(1, L_of[s_] + 1, n)
    kind = rng.integers(0, 10, n)
    d[k0:k1] = np.where(kind < 5, rng.integers(1, 61, n), np.where(kind < 7, rng.integers(61, 125, n),
               np.where(kind < 9, rng.integers(125, 700, n), rng.integers(8191, 9001, n))))
    d[k0 + rng.integers(0, n)] = rng.choice([0, 1, 3]) if rng.random() < 0.2 else d[k0]
one = np.ones(D, np.int32)
pb = synth.make_problem(off, np.arange(D + 1), one, one, one, sl * 100, np.zeros(D, np.int32), one * 64, one, one,
                        np.zeros(D, np.int32))
dp = ds.from_host(pb, "cuda")
o_all = {}
for Lv in np.unique(L_of):
    p = Params(L=int(Lv), S_tot=148, slot_us=100)
    hook = dict(level=torch.from_numpy(g).cuda(), d_slots=torch.from_numpy(d).cuda())
    o = ds.schedule_cycle(dp, p, None, torch.ones(D, dtype=torch.uint8, device="cuda"), None, hook=hook)
    torch.cuda.synchronize()
    o_all[int(Lv)] = {k: v.cpu().numpy() for k, v in o.items() if v is not None}
bad = []
for s_ in range(S):
    k0, k1 = off[s_], off[s_ + 1]
    o = o_all[int(L_of[s_])]
    nslots = int(sl[k0:k1].max())
    njobs = int(sum(nslots // x for x in sl[k0:k1]))
    if njobs > 512:
        continue
    dt = np.zeros((k1 - k0, 64), np.int64); dt[:, 0] = d[k0:k1]
    want = oracle.cycle_direct(g[k0:k1], sl[k0:k1], np.ones(k1 - k0, np.int32), dt, 1, int(L_of[s_]), nslots)
    ok = (o["misses"][s_] == want["misses"] and np.array_equal(o["runs"][k0:k1].view(np.uint16), want["runs"])
          and o["u"][s_] == want["u"] and o["u_static"][s_] == want["u_static"])
    if not ok:
        dd = d[k0:k1]
        bad.append((s_, int(L_of[s_]), nslots, k1 - k0, int((dd == 0).sum()), int((dd > 124).sum()), int((dd >= 8191).sum()),
                    int(o["misses"][s_]), int(want["misses"])))
print(sys.argv[1] if len(sys.argv) > 1 else "", "bad", len(bad), bad[:6])
