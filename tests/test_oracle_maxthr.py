"""Pins for O9b, the max-throughput comparison scheduler of §6.3: "a schedule that maximizes the sum of the
throughput across all the models" (reading R24 in DESIGN.md §3.2): over one session, runs of a batch
b <= b*_j lasting d_j(b) slots at each model's level g_j, no self-overlap, summed level <= L at every slot, every
run inside the session; maximise the requests served.

Pins independent of oracle.c's memoised search: a hand trace, a brute-force enumeration of every schedule on tiny
instances (tests below, plain recursion without memoisation), closed forms (one model, models that always fit
together), and the invariant that D-STACK's own session (O5, a schedule of the same kind) never serves more.
"""
import functools

import numpy as np

import oracle


def brute(g, bs, d, L, nslots):
    """Every schedule, slot by slot: at slot t each idle model may start a run of any batch b <= b* that ends by
    the session end; occupancy at t = levels of the runs in progress.  Plain recursion (exponential)."""
    n = len(g)

    def rec(t, rem):
        if t == nslots:
            return 0
        best = -1
        idle = [j for j in range(n) if rem[j] == 0 and g[j] > 0]
        # every assignment of (no start | batch b) to the idle models
        choices = [[0] + [b for b in range(1, bs[j] + 1) if t + d[j][b - 1] <= nslots] for j in idle]
        for combo in _product(choices):
            r = list(rem)
            gain = 0
            for j, b in zip(idle, combo):
                if b:
                    r[j] = d[j][b - 1]; gain += b
            if sum(g[j] for j in range(n) if r[j] > 0) > L:
                continue
            best = max(best, gain + rec(t + 1, tuple(max(x - 1, 0) for x in r)))
        return best

    return rec(0, tuple([0] * n))


def _product(lists):
    if not lists:
        yield ()
        return
    for x in lists[0]:
        for rest in _product(lists[1:]):
            yield (x,) + rest


def dt(d):
    a = np.zeros((len(d), 64), np.int64)
    for j, row in enumerate(d):
        a[j, : len(row)] = row
    return a


def test_hand_trace():
    """L = 10, 5 slots.  A: level 6, b* = 2, d(1) = 2, d(2) = 3.  B: level 6, d(1) = 2.  A and B never overlap
    (12 > 10).  A alone: b = 2 over [0, 3) then b = 1 over [3, 5): 3 requests; A b=1, b=1 (4 slots) = 2; B alone 2;
    A b = 2 then B = 3.  Max = 3.  Adding C (level 4, d(1) = 1), which fits beside either (10 <= 10), adds one
    request per slot: 3 + 5 = 8."""
    assert oracle.maxthr_direct([6, 6], [2, 1], dt([[2, 3], [2]]), 1, 10, 5) == 3
    assert oracle.maxthr_direct([6, 6, 4], [2, 1, 1], dt([[2, 3], [2], [1]]), 1, 10, 5) == 8


def test_brute_force_tiny():
    rng = np.random.default_rng(2540)
    for _ in range(160):
        n = int(rng.integers(1, 4))
        L = int(rng.integers(3, 14))
        g = [int(rng.integers(1, L + 1)) for _ in range(n)]
        bs = [int(rng.integers(1, 3)) for _ in range(n)]
        d = []
        for j in range(n):
            v = int(rng.integers(1, 4))
            row = []
            for _ in range(bs[j]):
                row.append(v); v += int(rng.integers(0, 2))
            d.append(row)
        nslots = int(rng.integers(1, 8))
        assert oracle.maxthr_direct(g, bs, dt(d), 1, L, nslots) == brute(g, bs, d, L, nslots), (g, bs, d, L, nslots)


def test_closed_forms():
    # one model, b* = 1: floor(nslots / d) runs back to back
    for dd in (1, 2, 3, 7):
        for ns in (1, 6, 20):
            assert oracle.maxthr_direct([5], [1], dt([[dd]]), 1, 10, ns) == ns // dd
    # one model, batches: unbounded knapsack of value b and weight d(b) into nslots
    d = [2, 3, 5]   # b = 1, 2, 3
    for ns in range(0, 16):
        best = max(sum(c) for c in _knap(d, ns))
        assert oracle.maxthr_direct([5], [3], dt([d]), 1, 10, ns) == best
    # levels that always fit together: the models do not interact
    g, bs, d = [3, 4, 2], [1, 2, 1], [[2], [1, 3], [4]]
    solo = [oracle.maxthr_direct([g[j]], [bs[j]], dt([d[j]]), 1, 9, 13) for j in range(3)]
    assert oracle.maxthr_direct(g, bs, dt(d), 1, 9, 13) == sum(solo)
    # b_lo: batches below it are not allowed
    assert oracle.maxthr_direct([5], [2], dt([[1, 5]]), 2, 10, 10) == 4


def _knap(d, cap):
    """every multiset of batches (values b = index + 1, weights d) with total weight <= cap (as lists of values)"""
    out = [[]]
    for b, w in enumerate(d, start=1):
        new = []
        for base in out:
            k = 0
            while sum(d[x - 1] for x in base) + k * w <= cap:
                new.append(base + [b] * k)
                k += 1
        out = new
    return out


def test_dstack_never_beats_max_throughput():
    """D-STACK's session (O5) is a schedule of the same kind: it can never serve more than max-throughput."""
    rng = np.random.default_rng(7)
    for _ in range(120):
        n = int(rng.integers(1, 5))
        L = int(rng.integers(5, 30))
        g = [int(rng.integers(1, L + 1)) for _ in range(n)]
        sl = [int(rng.choice([6, 12])) for _ in range(n)]
        bs = [int(rng.integers(1, 3)) for _ in range(n)]
        d = []
        for j in range(n):
            v = int(rng.integers(1, 4)); row = []
            for _ in range(bs[j]):
                row.append(v); v += int(rng.integers(0, 2))
            d.append(row)
        ns = max(sl)
        o = oracle.cycle_direct(g, sl, bs, dt(d), 1, L, ns)
        m = oracle.maxthr_direct(g, bs, dt(d), 1, L, ns)
        assert m is not None and m >= o["served_total"], (g, sl, bs, d, L, m, o["served_total"])


def test_scenario_level_and_state_cap():
    """O9b on generated scenarios (config 2 mixes with 2.5 ms slots, so sessions are 10-40 slots): OK scenarios serve
    at least D-STACK's count; scenarios beyond the state-space cap (or > 8 active models) are INVALID."""
    import synth
    sp, p = synth.config(2, num_scen=40, rows_pct=20)
    sp = sp.replace(slot_us=2500, slo_min_slots=10, slo_max_slots=40, ndnn_max=5)
    p = p.replace(slot_us=2500)
    pb = synth.generate_host(sp)
    m = oracle.maxthr(pb, p)
    e = oracle.evaluate(pb, p)
    ok = m["status"] == oracle.OK
    assert ok.sum() >= 20
    dstack_served = np.rint(e["thr"] * e["T_us"] / 1e6).astype(np.int64)
    assert (m["served"][ok] >= dstack_served[ok]).all()
    assert np.array_equal(m["T_us"][ok], e["T_us"][ok].astype(np.int64))
    tight = oracle.maxthr(pb, p, max_states=2)
    assert (tight["status"] == oracle.INVALID).sum() > (m["status"] == oracle.INVALID).sum()
