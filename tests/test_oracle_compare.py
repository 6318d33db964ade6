"""Pins for the oracle's O9 comparison schedulers (§6.3 of the paper; readings in
DESIGN.md §3.2): Max-Min fair fill, max-throughput fill, temporal sharing, GSLICE-style static spatial sharing."""
import json
import os

import numpy as np
import pytest

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "table4.json")


def table4():
    with open(GOLDEN) as f:
        return json.load(f)["models"]


def hand_case(fill_order):
    # L = 10 levels, 10 slots, one window each; g = (6, 3, 4), d(b*=1) = (2, 4, 1) slots
    dt = np.zeros((3, 64), np.int64)
    dt[:, 0] = [2, 4, 1]
    return oracle.cycle_direct([6, 3, 4], [10, 10, 10], [1, 1, 1], dt, 1, 10, 10, fill_order=fill_order)


@pytest.mark.parametrize("order,runs,occ,busy", [
    # hand traces (tests/golden/README.md "O9 hand traces"): static EDF placement M2 [0,1), M0 [0,2), M1 [1,5)
    (0, [4, 2, 4], 88, [8, 8, 4]),    # D-STACK: fewest runs first
    (1, [1, 2, 9], 72, [2, 8, 9]),    # Max-Min fair: smallest GPU% first
    (2, [3, 1, 9], 84, [6, 4, 9]),    # max-throughput: shortest run first
])
def test_fill_orders_hand_trace(order, runs, occ, busy):
    r = hand_case(order)
    assert r["runs"].tolist() == runs
    assert r["occ_sum"] == occ
    assert r["busy"].tolist() == busy
    assert r["misses"] == 0


def test_temporal_table4_pin():
    """slices proportional to SLO for Alexnet, ResNet-50, VGG-19 give 'mean GPU utilization of
    44%' = sum knee*SLO / sum SLO = 7750/175 % (exact when the slices are whole slots)."""
    t = table4()
    names = ["Alexnet", "ResNet-50", "VGG-19"]
    lvl = [t[m]["knee"] for m in names]
    sl = [t[m]["slo_ms"] * 10 for m in names]            # slots of 100 us
    r = oracle.temporal_direct(lvl, sl, [80, 280, 550], 1750)
    assert r["slice"].tolist() == [250, 500, 1000]
    assert r["occ_num"] / (1750 * 100) == pytest.approx(7750 / 17500, abs=0)
    assert round(100 * r["occ_num"] / (1750 * 100)) == 44
    assert r["runs"].tolist() == [250 // 80, 500 // 280, 1000 // 550]
    # T = 100 ms (1000 slots): floors lose < 1 slot per model
    r2 = oracle.temporal_direct(lvl, sl, [80, 280, 550], 1000)
    assert abs(r2["occ_num"] / 1e5 - 0.442857) < 3 * 50 / 1e5


def test_gslice_p1112_pin():
    """knees of Alexnet, Mobilenet, ResNet-50, VGG-19 exceed 100% together; 'VGG-19 in the first time
    slot, ResNet-50 in the second, along with Alexnet and Mobilenet concurrently in both time slots'."""
    t = table4()
    names = ["Alexnet", "Mobilenet", "ResNet-50", "VGG-19"]
    r = oracle.gslice_direct([t[m]["knee"] for m in names], [8, 10, 28, 55], 2000, 100)
    home = dict(zip(names, r["home"].tolist()))
    assert r["nbins"] == 2
    assert home["Alexnet"] == -1 and home["Mobilenet"] == -1
    assert {home["VGG-19"], home["ResNet-50"]} == {0, 1}
    assert home["VGG-19"] == 0                            # the first slot (first-fit decreasing)
    # residents run in both 1000-slot slots, the others in one
    assert r["runs"].tolist() == [2 * (1000 // 8), 2 * (1000 // 10), 1000 // 28, 1000 // 55]


def test_gslice_all_fit_is_one_slot():
    r = oracle.gslice_direct([20, 30, 40], [7, 9, 11], 500, 100)
    assert r["nbins"] == 1 and r["home"].tolist() == [-1, -1, -1]
    assert r["occ_num"] == sum(lv * (500 // d) * d for lv, d in zip([20, 30, 40], [7, 9, 11]))


def ref_temporal(lvl, sl, dL, nslots):
    tot = sum(s for lv, s in zip(lvl, sl) if lv > 0)
    sl_ = [nslots * s // tot if lv > 0 else 0 for lv, s in zip(lvl, sl)]
    return sl_, [x // d if d else 0 for x, d in zip(sl_, dL)]


def ref_gslice(lvl, dk, nslots, L):
    act = [j for j in range(len(lvl)) if lvl[j] > 0]
    asc = sorted(act, key=lambda j: (lvl[j], j))
    npre = max(p for p in range(len(asc) + 1)
               if sum(lvl[j] for j in asc[:p]) + (max(lvl[j] for j in asc) if p < len(asc) else 0) <= L)
    res = set(asc[:npre])
    cap = L - sum(lvl[j] for j in res)
    bins, home = [], {}
    for j in sorted(set(act) - res, key=lambda j: (-lvl[j], j)):
        for b, r in enumerate(bins):
            if r >= lvl[j]:
                bins[b] -= lvl[j]; home[j] = b
                break
        else:
            bins.append(cap - lvl[j]); home[j] = len(bins) - 1
    K = max(1, len(bins)); w = nslots // K
    runs = [0] * len(lvl)
    for j in act:
        runs[j] = (K if j in res else 1) * (w // dk[j])
    return K, runs


def test_temporal_and_gslice_vs_reference_random():
    rng = np.random.default_rng(7)
    for _ in range(300):
        n = int(rng.integers(1, 9))
        lvl = rng.integers(0, 101, n).tolist()
        lvl[0] = max(lvl[0], 1)
        sl = rng.integers(1, 60, n).tolist()
        d = rng.integers(1, 30, n).tolist()
        nslots = int(rng.integers(1, 400))
        r = oracle.temporal_direct(lvl, sl, d, nslots)
        s_, runs = ref_temporal(lvl, sl, d, nslots)
        assert r["slice"].tolist() == s_ and r["runs"].tolist() == runs
        g = oracle.gslice_direct(lvl, d, nslots, 100)
        K, runs = ref_gslice(lvl, d, nslots, 100)
        assert g["nbins"] == K and g["runs"].tolist() == runs


def test_compare_dstack_column_is_the_eval_path():
    sp, p = synth.config(2, num_scen=40, rows_pct=15)
    pb = synth.generate_host(sp)
    c = oracle.compare(pb, p)
    e = oracle.evaluate(pb, p)
    assert np.array_equal(c["u"][:, 0], e["u"]) and np.array_equal(c["thr"][:, 0], e["thr"])
    ok = e["T_us"] > 0
    assert ok.any()
    j = c["jain"][ok]
    assert np.all((j > 0) & (j <= 1 + 1e-12))
    # the fill variants only add runs to the same static placement
    assert np.all(c["u"][ok, 1:3] >= e["u_static"][ok, None] - 1e-12)


def test_jain_hand_value():
    sp, p = synth.config(1)
    pb = synth.generate_host(sp)
    c = oracle.compare(pb, p)
    assert c["jain"].shape == (1, 5)
    busy = hand_case(0)["busy"]
    assert busy.sum() ** 2 / (3 * (busy ** 2).sum()) == pytest.approx(400 / 432)
