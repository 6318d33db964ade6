"""Pins for F4, the multi-GPU cluster of §7.1 (4 T4 GPUs, "one T4 GPU for each
DNN model exclusively", "all 4 models in each GPU, temporally sharing the GPU", "D-STACK with the 4 DNN models",
"160% overall higher throughput than temporal sharing"; reading R23 in DESIGN.md §3.5).

The paper's T4 numbers come from measured models we do not have (its knees on T4 are unpublished), so the pins
are structural: G = 1 reduces every policy to the single-GPU schedulers (O9, pinned in test_oracle_compare.py);
the replicated policies are G times the single-GPU numbers; the placement policies equal an independent
composition of the pinned primitives (O4 WMAX-MIN, O5 sessions, O9 temporal) on the hand-placed subsets; one
model alone on a GPU has the closed-form back-to-back throughput.
"""
import numpy as np

import oracle
import synth
from synth import Params
from tests.helpers import multi_dnn_problem


def test_single_gpu_reduces_to_the_single_gpu_schedulers():
    sp, p = synth.config(2, num_scen=60, rows_pct=40)
    pb = synth.generate_host(sp)
    c = oracle.cluster(pb, p, 1)
    o = oracle.compare(pb, p)
    for col, ocol in ((0, 3), (1, 3), (2, 0), (3, 0)):   # G = 1: exclusive/temporal = temporal, D-STACK = D-STACK
        assert np.array_equal(c["u"][:, col], o["u"][:, ocol]), col
        assert np.array_equal(c["thr"][:, col], o["thr"][:, ocol]), col


def test_replicated_policies_scale_with_G():
    sp, p = synth.config(4, num_scen=30, rows_pct=40)
    pb = synth.generate_host(sp)
    o = oracle.compare(pb, p)
    for G in (2, 4, 8):
        c = oracle.cluster(pb, p, G)
        assert np.array_equal(c["u"][:, 1], o["u"][:, 3]) and np.array_equal(c["thr"][:, 1], G * o["thr"][:, 3])
        assert np.array_equal(c["u"][:, 2], o["u"][:, 0]) and np.array_equal(c["thr"][:, 2], G * o["thr"][:, 0])


def placement_ffd(dem, G, L):
    """First-fit decreasing by demand (desc, index), overflow to the least-loaded GPU (lowest index)."""
    load = [0] * G
    home = [-1] * len(dem)
    for j in sorted((j for j in range(len(dem)) if dem[j] > 0), key=lambda j: (-dem[j], j)):
        gi = next((i for i in range(G) if load[i] + dem[j] <= L), None)
        if gi is None:
            gi = min(range(G), key=lambda i: (load[i], i))
        home[j] = gi
        load[gi] += dem[j]
    return home


def test_placement_policies_compose_the_pinned_primitives():
    """c = 0 and c = 3 recomputed from O3 outputs, O4 (oracle.wmaxmin), O5 (oracle.cycle_direct) and O9 temporal
    (oracle.temporal_direct) on the subsets placed here, with run lengths from O1 (oracle.X)."""
    sp, p = synth.config(4, num_scen=8, rows_pct=40)
    pb = synth.generate_host(sp)
    G = 3
    c = oracle.cluster(pb, p, G)
    bo = oracle.batch_opt(pb, p)
    dem, bt, st = bo["demand"], bo["batch"], bo["status"]
    S_of = lambda l: -(-l * p.S_tot // p.L)
    for s in range(pb.num_scen):
        k0, k1 = int(pb.scen_dnn_off[s]), int(pb.scen_dnn_off[s + 1])
        d = [int(dem[k]) if st[k] == oracle.OK else 0 for k in range(k0, k1)]
        b = [max(int(bt[k]), 1) for k in range(k0, k1)]
        slo = [int(pb.slo_us[k]) for k in range(k0, k1)]
        sl = [v // p.slot_us for v in slo]
        M = [int(pb.mem_bw[k]) for k in range(k0, k1)]
        run = lambda j, l, bb: -(-oracle.X(pb, p, k0 + j, l, bb) // (S_of(l) * M[j] * p.slot_us))
        act = [j for j in range(k1 - k0) if d[j] > 0]
        if not act:
            assert not c["u"][s].any()
            continue
        home0 = {j: q % G for q, j in enumerate(act)}
        home3 = placement_ffd(d, G, p.L)
        u0 = t0 = u3 = t3 = 0.0
        for gi in range(G):
            sub = [j for j in act if home0[j] == gi]
            if sub:
                Ti = max(slo[j] for j in sub); ns = Ti // p.slot_us
                lvl = [d[j] if j in sub else 0 for j in range(k1 - k0)]
                dL = [run(j, p.L, b[j]) if j in sub else 0 for j in range(k1 - k0)]
                r = oracle.temporal_direct(lvl, sl, dL, ns)
                u0 += r["occ_num"] / (ns * p.L) / G
                t0 += sum(int(r["runs"][j]) * b[j] for j in sub) * 1e6 / Ti
            sub = [j for j in act if home3[j] == gi]
            if sub:
                Ti = max(slo[j] for j in sub); ns = Ti // p.slot_us
                alloc = oracle.wmaxmin([d[j] for j in sub], p.L)
                g = [0] * (k1 - k0)
                dtab = np.zeros((k1 - k0, 64), np.int64)
                for q, j in enumerate(sub):
                    g[j] = max(d[j], int(alloc[q]) >> 16)
                    for bb in range(p.b_min, b[j] + 1):
                        dtab[j, bb - 1] = run(j, g[j], bb)
                r = oracle.cycle_direct(g, sl, b, dtab, p.b_min, p.L, ns)
                u3 += r["occ_sum"] / (ns * p.L) / G
                t3 += r["served_total"] * 1e6 / Ti
        assert c["u"][s, 0] == u0 and c["thr"][s, 0] == t0, s
        assert c["u"][s, 3] == u3 and c["thr"][s, 3] == t3, s


def test_one_model_per_gpu_closed_form():
    """Exclusive with N <= G: model j alone owns a whole GPU for its SLO-long session and runs floor(nslots / d^L)
    back-to-back b* batches at 100%: throughput b* floor(nslots/d^L) 1e6 / SLO_j; idle GPUs count 0 in U."""
    dn = [dict(rows=[(30, 1, 10**5), (10, 2, 10**4)], t_p=40, t_np=5, M=50000, slo=20000, a=300, bmax=8),
          dict(rows=[(90, 1, 10**6)], t_p=60, t_np=4, M=50000, slo=40000, a=300, bmax=8)]
    pb = multi_dnn_problem(dn)
    p = Params(L=100, S_tot=148)
    G = 4
    c = oracle.cluster(pb, p, G)
    bo = oracle.batch_opt(pb, p)
    dem, bt = bo["demand"], bo["batch"]
    thr = 0.0
    u = 0.0
    for j, x in enumerate(dn):
        dL = -(-oracle.X(pb, p, j, p.L, int(bt[j])) // (p.S_tot * x["M"] * p.slot_us))
        ns = x["slo"] // p.slot_us
        thr += int(bt[j]) * (ns // dL) * 1e6 / x["slo"]
        u += ns * int(dem[j]) / (ns * p.L) / G   # the whole session slice at knee% accounting
    assert c["thr"][0, 0] == thr
    assert abs(c["u"][0, 0] - u) < 1e-15
    assert c["u"][0, 0] <= 2 / G   # two busy GPUs out of four
