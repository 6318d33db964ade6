"""Pins for F1, the below-knee fallback of the oracle's O5 session ("D-STACK's
scheduler can also schedule a model with GPU% lower than its Knee, albeit with high inference latency when
necessary. D-STACK also considers the additional latency of launching a new DNN model at lower GPU% into
the schedule"; reading R21 in DESIGN.md §3.3).

The paper prints no number for this mechanism, so the pins are a hand trace, an independent brute-force
replay of the rule on random sessions, and the special cases that reduce to O5 without the fallback.
"""
import numpy as np

import oracle
import synth


def hand_case(dlow_a):
    # L = 100, one 10-slot session; A: g = 60, d(b*) = 8; B: g = 60, d(b*) = 5; both SLO = session.
    g, sl, bs = [60, 60], [10, 10], [1, 1]
    dtab = [[8], [5]]
    dlow = np.zeros((2, 256), np.int64)
    dlow[0, 1:60] = dlow_a[1:60]
    return oracle.cycle_direct_bk(g, sl, bs, dtab, dlow, 1, 100, 10)


def test_hand_trace():
    """EDF with equal deadlines takes B first (shorter run): B [0, 5) at 60.  A's 8 slots at 60 cannot fit
    (slots 0-4 hold 60, only 5 free slots remain).  Below the knee A needs 9 slots at levels 41-59 (only
    slots 5-9 admit such a level) and 10 slots at 1-40: the first level that fits is 40, over [0, 10).
    Fill: t = 5 (B's end), B again over [5, 10).  U_static = (60*5 + 40*10) / 1000, U = 1."""
    dlow = np.zeros(256, np.int64)
    dlow[41:60] = 9
    dlow[1:41] = 10
    r = hand_case(dlow)
    tr = r["trace"]
    assert r["misses"] == 0 and r["below"] == 1 and r["status"] == oracle.OK
    st = [(int(tr["dnn"][i]), int(tr["start"][i]), int(tr["end"][i]), int(tr["kind"][i]), int(tr["level"][i]))
          for i in range(len(tr["dnn"]))]
    assert st == [(1, 0, 5, 0, 60), (0, 0, 10, 2, 40), (1, 5, 10, 1, 60)]
    assert r["occ_static_sum"] == 700 and r["occ_sum"] == 1000
    assert r["runs"].tolist() == [1, 2]


def test_hand_trace_without_fallback():
    """Same session, no usable level (launch latency pushes every run past the window): A is a miss, as in O5."""
    dlow = np.zeros(256, np.int64)
    dlow[1:60] = 11
    r = hand_case(dlow)
    base = oracle.cycle_direct([60, 60], [10, 10], [1, 1], [[8], [5]], 1, 100, 10)
    assert r["misses"] == 1 and r["below"] == 0 and r["status"] == oracle.OVERSUBSCRIBED
    for k in ("occ_static_sum", "occ_sum", "served_total", "misses"):
        assert r[k] == base[k], k
    assert r["occ_sum"] == 600


def replay(g, sl, bs, dtab, dlow, L, nslots):
    """Independent replay of the static pass (EDF order (deadline, d(b*), j, r), even repeats earliest /
    odd repeats latest start; on failure levels g-1 .. 1 with dlow).  Returns {(j, r): (start, d, level)}
    (None for a miss) and the static occupancy."""
    occ = np.zeros(nslots, np.int64)
    jobs = sorted((((r + 1) * sl[j], dtab[j][bs[j] - 1], j, r) for j in range(len(g)) if g[j] > 0
                   for r in range(nslots // sl[j])))
    out = {}
    for dl, d, j, r in jobs:
        rel = r * sl[j]
        placed = None
        for lvl, dd in [(g[j], d)] + [(l, int(dlow[j][l])) for l in range(g[j] - 1, 0, -1)]:
            if dd <= 0 or dd > dl - rel:
                continue
            starts = range(rel, dl - dd + 1) if r % 2 == 0 else range(dl - dd, rel - 1, -1)
            for s in starts:
                if all(occ[u] + lvl <= L for u in range(s, s + dd)):
                    placed = (s, dd, lvl)
                    break
            if placed:
                break
        if placed:
            s, dd, lvl = placed
            occ[s:s + dd] += lvl
        out[(j, r)] = placed
    return out, occ


def test_random_sessions_brute_force():
    rng = np.random.default_rng(21)
    n_below = 0
    for _ in range(300):
        n = int(rng.integers(2, 7)); L = int(rng.integers(10, 101))
        sl = [int(v) for v in rng.choice([10, 20, 40], n)]
        nslots = max(sl)
        g = [int(rng.integers(1, L + 1)) for _ in range(n)]
        bs = [1] * n
        dtab = [[int(rng.integers(1, s + 1))] for s in sl]
        dlow = np.zeros((n, 256), np.int64)
        for j in range(n):   # lower level -> longer run (plus a random launch latency)
            c = int(rng.integers(0, 3))
            for l in range(1, g[j]):
                dlow[j, l] = -(-dtab[j][0] * g[j] // l) + c
        r = oracle.cycle_direct_bk(g, sl, bs, dtab, dlow, 1, L, nslots)
        want, occ = replay(g, sl, bs, dtab, dlow, L, nslots)
        tr = r["trace"]
        got = {}
        for i in range(len(tr["dnn"])):
            if tr["kind"][i] in (0, 2):
                got[(int(tr["dnn"][i]), int(tr["rep"][i]))] = (int(tr["start"][i]), int(tr["end"][i] - tr["start"][i]),
                                                                int(tr["level"][i]))
        assert {k: v for k, v in want.items() if v} == got
        assert r["misses"] == sum(v is None for v in want.values())
        assert r["below"] == sum(1 for (j, _), v in want.items() if v and v[2] < g[j])
        assert r["occ_static_sum"] == int(occ.sum()) and occ.max(initial=0) <= L
        n_below += r["below"]
    assert n_below > 20   # the random sessions really exercise the fallback


def test_whole_path_flag_semantics():
    """Config 4 (oversubscribed): with the fallback some static jobs run below the knee; with a launch
    latency longer than every SLO nothing can, and every output equals the plain O5 path."""
    sp, p = synth.config(4, num_scen=40)
    pb = synth.generate_host(sp)
    base = oracle.evaluate(pb, p)
    on = oracle.evaluate(pb, p.replace(below_knee=1))
    assert on["below"].sum() > 0 and base["below"].sum() == 0
    off = oracle.evaluate(pb, p.replace(below_knee=1, reconf_us=10**8))
    for k in base:
        assert np.array_equal(off[k], base[k]), k
    # per-DNN a1-a4 outputs do not depend on the session rule
    for k in ("demand", "batch", "knee", "status", "alloc_q16", "level"):
        assert np.array_equal(on[k], base[k]), k
    # every scenario with a below-knee run had a miss without the fallback (the fallback runs only on misses;
    # EDF placements before the first miss coincide)
    assert np.all(base["misses"][on["below"] > 0] > 0)


def test_whole_path_glue_matches_direct_session():
    """eval's F1 session equals cycle_direct_bk fed with run lengths computed here from O1 (oracle.X, pinned in
    test_oracle_model.py): d_j(b) = ceil(X(g, b) / (S(g) M Delta)), dlow_j(l) = ceil(X(l, b*) / (S(l) M Delta)) +
    ceil(reconf_us / Delta)."""
    sp, p = synth.config(4, num_scen=6)
    p = p.replace(below_knee=1, reconf_us=250)
    pb = synth.generate_host(sp)
    on = oracle.evaluate(pb, p)
    c = -(-p.reconf_us // p.slot_us)
    S_of = lambda l: -(-l * p.S_tot // p.L)
    for s in range(pb.num_scen):
        k0, k1 = int(pb.scen_dnn_off[s]), int(pb.scen_dnn_off[s + 1])
        if on["T_us"][s] == 0:
            continue
        g = [int(v) for v in on["level"][k0:k1]]
        bs = [max(int(v), 1) for v in on["batch"][k0:k1]]
        sl = [int(pb.slo_us[k]) // p.slot_us for k in range(k0, k1)]
        dtab = np.zeros((k1 - k0, 64), np.int64)
        dlow = np.zeros((k1 - k0, 256), np.int64)
        for j, k in enumerate(range(k0, k1)):
            if g[j] == 0:
                continue
            M = int(pb.mem_bw[k])
            den = lambda l: S_of(l) * M * p.slot_us
            dtab[j, bs[j] - 1] = -(-oracle.X(pb, p, k, g[j], bs[j]) // den(g[j]))
            for l in range(1, g[j]):
                dlow[j, l] = -(-oracle.X(pb, p, k, l, bs[j]) // den(l)) + c
        r = oracle.cycle_direct_bk(g, sl, bs, dtab, dlow, 1, p.L, int(on["T_us"][s]) // p.slot_us)
        assert r["below"] == on["below"][s] and r["misses"] == on["misses"][s]
        assert r["occ_sum"] / (int(on["T_us"][s]) // p.slot_us * p.L) == on["u"][s]
