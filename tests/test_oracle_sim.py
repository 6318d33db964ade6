"""Pins for the oracle's O7 long-horizon simulation (config 5, DESIGN.md §3 O7)."""
import math

import numpy as np
import pytest

import oracle
import synth


def small_sim_problem(num_scen=4, rows_pct=10, lam=None):
    sp, p = synth.config(5, num_scen=num_scen, rows_pct=rows_pct)
    sp = sp.replace(ndnn_min=2, ndnn_max=5)
    pb = synth.generate_host(sp)
    if lam is not None:
        pb.lam_pct[:] = lam
    return sp, p, pb


def reference_sim(pb, p, s, cycles, seed, cfg_tag):
    """Independent re-implementation of the O7 loop (DESIGN.md §3 O7) on top of the pinned O3 (batch_opt),
    O4 (wmaxmin), O1 (X) and O5 (cycle_direct with scoreboard counts) plus the shared arrival sampler."""
    one = pb.scenario(s)
    bo = oracle.batch_opt(one, p)
    nd = one.num_dnn
    ok = bo["status"] == 0
    if not ok.any():
        return None
    T = int(max(one.slo_us[j] for j in range(nd) if ok[j]))
    nslots = T // p.slot_us

    class Stream:   # arrival times of one DNN, regenerated from the counter-based sampler
        def __init__(self, j, mean_q):
            self.j, self.mean_q, self.k, self.gaps, self.t = j, mean_q, 0, [], 0
            self.times = []

        def time(self, k):
            while len(self.times) <= k:
                g = synth.arrival_gaps(seed, cfg_tag, s, self.j, self.mean_q, len(self.times), 64)
                for x in g:
                    self.t += int(x)
                    self.times.append(self.t)
            return self.times[k]

        def count(self, t):   # arrivals with time <= t
            k = 0
            while self.time(k) <= t:
                k += 1
            return k

    streams = {}
    for j in range(nd):
        if not ok[j]:
            continue
        ls = max(1, int(bo["demand"][j]) - p.margin)
        S = -(-ls * p.S_tot // p.L)
        X = oracle.X(one, p, j, ls, int(bo["batch"][j]))
        M = int(one.mem_bw[j]) if p.mem_mode else 1
        lam = int(one.lam_pct[j])            # R25: no offered load -> infinite gap, capped below
        mq = ((X * 100) << 32) // (S * M * lam * int(bo["batch"][j])) if lam > 0 else 1 << 62
        streams[j] = Stream(j, min(mq, 1 << 62))
    served = [0] * nd
    ring = np.zeros((10, nd), np.int64)
    res = dict(in_slo=0, late=0, occ_sum=0, runs=0, misses=0, realloc=0)
    # per-cycle rows in dstack.h's DSTACK_SIM_* order: active, realloc, runs, served, in SLO, late, occ, misses
    res["series"] = np.zeros((cycles, 8), np.int64)
    prev = None
    for c in range(cycles):
        t0 = c * T
        dm = np.zeros(nd, np.uint16)
        for j in streams:
            if streams[j].count(t0) > served[j]:
                dm[j] = bo["demand"][j]
        act = tuple(int(x > 0) for x in dm)   # the active set; a change means a WMAX-MIN re-allocation
        row = res["series"][c]
        row[0] = sum(act)
        if prev is not None and act != prev:
            res["realloc"] += 1
            row[1] = 1
        prev = act
        al = oracle.wmaxmin(dm, p.L)
        g = np.zeros(nd, np.int32); dtab = np.zeros((nd, 64), np.int64)
        for j in range(nd):
            if dm[j] == 0:
                continue
            g[j] = max(int(dm[j]), int(al[j]) >> 16)
            S = -(-int(g[j]) * p.S_tot // p.L)
            M = int(one.mem_bw[j]) if p.mem_mode else 1
            for b in range(p.b_min, int(bo["batch"][j]) + 1):
                X = oracle.X(one, p, j, int(g[j]), b) if S == -(-int(g[j]) * p.S_tot // p.L) else None
                dtab[j, b - 1] = -(-X // (S * M * p.slot_us))
        sl = (one.slo_us // p.slot_us).astype(np.int32)
        cyc = oracle.cycle_direct(g, sl, bo["batch"].astype(np.int32), dtab, p.b_min, p.L, nslots,
                                  count0=ring.sum(axis=0))
        res["misses"] += cyc["misses"]
        row[7] = cyc["misses"]
        tr = cyc["trace"]
        order = sorted(range(len(tr["dnn"])), key=lambda q: (tr["dnn"][q], tr["start"][q]))
        cnt = np.zeros(nd, np.int64)
        for q in order:
            j, st, en, b = int(tr["dnn"][q]), int(tr["start"][q]), int(tr["end"][q]), int(tr["batch"][q])
            ts, te = t0 + st * p.slot_us, t0 + en * p.slot_us
            k = min(b, streams[j].count(ts) - served[j])
            if k <= 0:
                continue
            for i in range(served[j], served[j] + k):
                if te - streams[j].time(i) > int(one.slo_us[j]):
                    res["late"] += 1
                    row[5] += 1
                else:
                    res["in_slo"] += 1
                    row[4] += 1
            served[j] += k
            row[3] += k
            cnt[j] += 1
            res["occ_sum"] += int(g[j]) * (en - st)
            row[6] += int(g[j]) * (en - st)
            res["runs"] += 1
            row[2] += 1
        ring[c % 10] = cnt
    res["arrived"] = sum(streams[j].count(cycles * T) for j in streams)
    res["unserved"] = res["arrived"] - sum(served)
    return res


def test_sim_matches_independent_reimplementation():
    sp, p, pb = small_sim_problem(num_scen=4, rows_pct=10)
    cycles = 12
    o = oracle.simulate(pb, p, cycles, sp.seed, sp.cfg_tag, series=True)
    series = np.zeros((cycles, 8), np.int64)
    for s in range(pb.num_scen):
        want = reference_sim(pb, p, s, cycles, sp.seed, sp.cfg_tag)
        if want is None:
            continue
        for k in ("arrived", "in_slo", "late", "unserved", "occ_sum", "runs", "misses", "realloc"):
            assert int(o[k][s]) == want[k], (s, k, int(o[k][s]), want[k])
        series += want["series"]
    # the per-cycle aggregate series (dstack.h DSTACK_SIM_*), summed over the scenarios
    assert np.array_equal(o["series"].astype(np.int64), series)


def test_sim_zero_load():
    """R25: lam_pct <= 0 offers no requests. All-zero load: nothing arrives, runs or occupies a slot (every
    session is empty); a mix of zero and positive loads matches the independent re-implementation."""
    sp, p, pb = small_sim_problem(num_scen=6, rows_pct=10, lam=0)
    o = oracle.simulate(pb, p, 10, sp.seed, sp.cfg_tag, series=True)
    ok = o["status"] == oracle.OK
    assert ok.any()
    for k in ("arrived", "in_slo", "late", "unserved", "occ_sum", "runs", "realloc"):
        assert (o[k] == 0).all(), k
    pb.lam_pct[::2] = 0
    pb.lam_pct[1::2] = 90
    pb.lam_pct[3::4] = -5
    o = oracle.simulate(pb, p, 10, sp.seed, sp.cfg_tag)
    for s in range(pb.num_scen):
        want = reference_sim(pb, p, s, 10, sp.seed, sp.cfg_tag)
        if want is None:
            continue
        for k in ("arrived", "in_slo", "late", "unserved", "occ_sum", "runs", "misses", "realloc"):
            assert int(o[k][s]) == want[k], (s, k)
    assert o["arrived"].sum() > 0


def test_sim_conservation_and_determinism():
    sp, p, pb = small_sim_problem(num_scen=20, rows_pct=15)
    a = oracle.simulate(pb, p, 20, sp.seed, sp.cfg_tag)
    b = oracle.simulate(pb, p, 20, sp.seed, sp.cfg_tag, subset=range(5, 20, 3))
    assert np.array_equal(a["arrived"], a["in_slo"] + a["late"] + a["unserved"])
    for s in range(5, 20, 3):
        for k in a:
            assert a[k][s] == b[k][s]


def test_sim_load_sheds():
    # qualitative: raising the offered load cannot lower the violation share
    sp, p, pb = small_sim_problem(num_scen=6, rows_pct=15, lam=40)
    lo = oracle.simulate(pb, p, 15, sp.seed, sp.cfg_tag)
    pb.lam_pct[:] = 200
    hi = oracle.simulate(pb, p, 15, sp.seed, sp.cfg_tag)
    viol = lambda o: (o["late"] + o["unserved"]).sum() / max(o["arrived"].sum(), 1)
    assert viol(hi) > viol(lo)


def test_arrival_sampler_is_exponential():
    mean = 1000
    g = synth.arrival_gaps(0x230413541, 5, 123, 4, mean << 32, 0, 200_000).astype(np.float64)
    assert abs(g.mean() - mean) / mean < 0.01                      # E[gap] = mean (floor loses ~0.5)
    assert abs((g > mean).mean() - math.exp(-1)) < 0.005            # P(gap > mean) = e^-1
    assert abs((g > 3 * mean).mean() - math.exp(-3)) < 0.002
