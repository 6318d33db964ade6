"""Pins for the opportunistic fill of the O5 session when b* > 1 (Dynamic-schedule, Alg. 1 P:3547-3555;
§6.1.2): "the scheduler picks a batch size that can complete within the time slice",
"possibly with a smaller batch".  Readings R12/R13.

Two pins independent of `oracle.c`'s session loop:
  * hand traces (tests/golden/fill_hand_traces.json, each derived by hand in its `how` field);
  * `replay`, a re-implementation written from the readings with different data structures (a run list whose
    load at a slot is summed on demand, a heap of decision times, slices grown one slot at a time, the batch by an
    upward scan) on random sessions with b* in 2..8 and d(b) nondecreasing with plateaus; every run (start, end,
    batch, kind) is compared IN ORDER, so the fill's priority order, slice and batch choice are all checked.
A smallest-fitting-batch rule, a slice cut one slot short or a fill order other than (runs so far, index) fails
both (checked by hand against mutated oracle builds when this file was written; see the commit message).
"""
import heapq
import json
import os

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))


def replay(g, sl, bs, d, L, nslots, b_lo=1):
    """Independent session replay.  d[j][b-1] = run slots of batch b.  Returns the runs in placement order as
    (j, start, end, batch, kind) with kind 0 static / 1 fill, and the per-model served counts."""
    runs = []   # (j, start, end, batch, kind)

    def load(u):
        return sum(g[j] for (j, s, e, _, _) in runs if s <= u < e)

    def fits_run(j, s, dd):
        return all(load(u) + g[j] <= L for u in range(s, s + dd))

    active = [j for j in range(len(g)) if g[j] > 0]
    jobs = sorted(((r + 1) * sl[j], d[j][bs[j] - 1], j, r) for j in active for r in range(nslots // sl[j]))
    for (dl, dd, j, r) in jobs:
        rel = r * sl[j]
        starts = [s for s in range(rel, dl - dd + 1) if fits_run(j, s, dd)]
        if starts:
            s = starts[0] if r % 2 == 0 else starts[-1]
            runs.append((j, s, s + dd, bs[j], 0))
    heap = [0] + [e for (_, _, e, _, _) in runs if e < nslots]
    heapq.heapify(heap)
    seen = set()
    while heap:
        t = heapq.heappop(heap)
        if t in seen or t >= nslots:
            continue
        seen.add(t)
        count = {j: sum(1 for x in runs if x[0] == j) for j in active}
        for j in sorted(active, key=lambda j: (count[j], j)):
            mine = [x for x in runs if x[0] == j]
            if any(s <= t < e for (_, s, e, _, _) in mine):
                continue
            if load(t) + g[j] > L:
                continue
            nxt = min([s for (_, s, _, _, _) in mine if s > t], default=nslots)
            k = 0
            while t + k < nxt and load(t + k) + g[j] <= L:
                k += 1
            b = 0
            for bb in range(b_lo, bs[j] + 1):
                if d[j][bb - 1] <= k:
                    b = bb
            if b == 0:
                continue
            runs.append((j, t, t + d[j][b - 1], b, 1))
            if t + d[j][b - 1] < nslots:
                heapq.heappush(heap, t + d[j][b - 1])
    served = [sum(x[3] for x in runs if x[0] == j) for j in range(len(g))]
    return runs, served


def oracle_runs(o):
    tr = o["trace"]
    return [(int(tr["dnn"][i]), int(tr["start"][i]), int(tr["end"][i]), int(tr["batch"][i]), int(tr["kind"][i]))
            for i in range(len(tr["dnn"]))]


def dtab_of(d):
    dt = np.zeros((len(d), 64), np.int64)
    for j, row in enumerate(d):
        dt[j, : len(row)] = row
    return dt


def load_golden():
    with open(os.path.join(HERE, "golden", "fill_hand_traces.json")) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("case", load_golden(), ids=lambda c: c["name"])
def test_fill_hand_traces(case):
    o = oracle.cycle_direct(case["g"], case["sl"], case["bstar"], dtab_of(case["d"]), 1, case["L"], case["nslots"])
    want = [tuple(r) for r in case["runs"]]
    assert oracle_runs(o) == want
    assert o["served"].tolist() == case["served"]
    assert o["occ_static_sum"] == case["occ_static_sum"] and o["occ_sum"] == case["occ_sum"]
    # the independent replay agrees with the hand trace too
    runs, served = replay(case["g"], case["sl"], case["bstar"], case["d"], case["L"], case["nslots"])
    assert runs == want and served == case["served"]


def random_session(rng):
    n = int(rng.integers(1, 6))
    L = int(rng.integers(8, 40))
    g = [int(rng.integers(1, L + 1)) for _ in range(n)]
    sl = [int(rng.choice([12, 16, 24, 48])) for _ in range(n)]
    bs = [int(rng.integers(2, 9)) for _ in range(n)]
    d = []
    for j in range(n):
        v = int(rng.integers(1, max(2, sl[j] // 3)))
        row = []
        for _ in range(bs[j]):
            row.append(v)
            v += int(rng.choice([0, 0, 1, 1, 2, 4]))   # nondecreasing, with plateaus
        d.append(row)
    return g, sl, bs, d, L, max(sl)


def test_fill_random_replay_b_star_above_one():
    """Every run (static and fill, in placement order) of 400 random sessions with b* in 2..8 equals the
    independent replay; the sample must exercise reduced batches and slices cut by a blocking slot and by the
    model's own next start."""
    rng = np.random.default_rng(20304)
    reduced = cut_by_own = 0
    for _ in range(400):
        g, sl, bs, d, L, nslots = random_session(rng)
        b_lo = 1 if rng.random() < 0.8 else 2
        o = oracle.cycle_direct(g, sl, bs, dtab_of(d), b_lo, L, nslots)
        runs, served = replay(g, sl, bs, d, L, nslots, b_lo)
        assert oracle_runs(o) == runs
        assert o["served"].tolist() == served
        for (j, s, e, b, kind) in runs:
            if kind == 1 and b < bs[j]:
                reduced += 1
                nxt = min([x[1] for x in runs if x[0] == j and x[1] > s], default=nslots)
                if e <= nxt and d[j][b] > nxt - s:
                    cut_by_own += 1
    assert reduced >= 200 and cut_by_own >= 20, (reduced, cut_by_own)


def test_fill_batch_is_largest_fitting_not_smallest():
    """Direct statement of the rule on the first golden case: the fill batch is the largest b <= b* whose run fits
    the 3-slot residual (b = 2, d = 3), not the smallest (b = 1) and not b* (d = 5 > 3)."""
    c = load_golden()[0]
    o = oracle.cycle_direct(c["g"], c["sl"], c["bstar"], dtab_of(c["d"]), 1, c["L"], c["nslots"])
    fill = [r for r in oracle_runs(o) if r[4] == 1]
    assert fill == [(0, 9, 12, 2, 1)]
