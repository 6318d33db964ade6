"""Pins for the oracle's O1 (latency, Eqs. 1-5), O2 (knee, Eq. 6) and O3 (batch/GPU%, Eqs. 7-12).

Each test ties the oracle to something other than itself: a value printed in PAPER.md or a
SPEC.md worked example (cited), a closed form, a special case, or an independent brute force
written per kernel with exact rationals (tests/helpers.py) -- never the oracle's integer X.
"""
from fractions import Fraction as F

import numpy as np
import pytest

import oracle
from synth import Params
from tests.helpers import S_of, eq1_rows, f_L, multi_dnn_problem, random_dnn, single_dnn_problem


def fl_oracle(pb, p, dnn, l, b, M=1):
    """f_L from the oracle's X = E_t * S * M."""
    M = 1 if p.mem_mode == 0 else M
    return F(oracle.X(pb, p, dnn, l, b), S_of(p, l) * M)


# ---------------------------------------------------------------- O1 -------

def test_eq1_spec_examples():
    # SPEC S:49-51 (Eq. 1): (K=50, p=20, b=1): N_1 = 20, N_2 = floor(20 - 0.4) = 19, N_50 = 0.
    N = eq1_rows(50, 20, 1)
    assert N[0] == 20 and N[1] == 19 and N[49] == 0
    assert all(N[i] >= N[i + 1] >= 0 for i in range(49))


def test_eq2_spec_examples():
    # SPEC S:58-60 (Eq. 2): N_i = 20, t_p = 40: s = 10 -> 80; s = 20 -> 40; N_i = 0 -> 0.
    p = Params(L=20, S_tot=20, mem_mode=0, b_max=1)
    pb = single_dnn_problem([(20, 1, 0)], t_p=40, t_np=0)
    assert fl_oracle(pb, p, 0, 10, 1) == 80
    assert fl_oracle(pb, p, 0, 20, 1) == 40
    pb0 = single_dnn_problem([(0, 1, 0)], t_p=40, t_np=0)
    assert fl_oracle(pb0, p, 0, 7, 1) == 0


def test_eq3_spec_examples():
    # SPEC S:67-69 (Eq. 3): d = 100, s = 4, M = 50: verbatim E_m = d s / M = 8; bandwidth mode d/(M s) = 0.5.
    pb = single_dnn_problem([(0, 1, 100)], t_p=1, t_np=0, M=50)
    assert fl_oracle(pb, Params(L=4, S_tot=4, mem_mode=2), 0, 4, 1, M=50) == 8
    assert fl_oracle(pb, Params(L=4, S_tot=4, mem_mode=1), 0, 4, 1, M=50) == F(1, 2)
    assert fl_oracle(pb, Params(L=4, S_tot=4, mem_mode=0), 0, 4, 1, M=50) == 0


def test_eq4_spec_examples():
    # SPEC S:76-78 (Eq. 4): K = 50, R = 1, t_np = 10, E_m = 0: b = 1 -> 500; b = 2 -> 1000; t_np = 0 -> 0.
    p = Params(L=8, S_tot=8, mem_mode=0)
    pb = single_dnn_problem([(0, 1, 0)] * 50, t_p=1, t_np=10)
    assert fl_oracle(pb, p, 0, 3, 1) == 500
    assert fl_oracle(pb, p, 0, 3, 2) == 1000
    pb0 = single_dnn_problem([(0, 1, 0)] * 50, t_p=1, t_np=0)
    assert fl_oracle(pb0, p, 0, 3, 1) == 0


def test_eq5_spec_examples():
    # SPEC S:86 (Eq. 5): Fig. 3 DNN (K=50, p=20, t_p=40, t_np=10, b=1) at s=1: 500 + 40 * sum_i N_i.
    # S:85's s=1000 formula is wrong: with s >= N_1 every non-empty kernel takes t_p,
    # so E_t = 500 + 40 * #{N_i >= 1} = 500 + 40*20 = 1300.
    N = eq1_rows(50, 20, 1)
    pb = single_dnn_problem([(n, 1, 0) for n in N], t_p=40, t_np=10)
    p = Params(L=1000, S_tot=256, mem_mode=0)   # S(L) = 256 >= N_1
    assert fl_oracle(pb, Params(L=256, S_tot=256, mem_mode=0), 0, 1, 1) == 500 + 40 * sum(N)
    assert fl_oracle(pb, Params(L=256, S_tot=256, mem_mode=0), 0, 256, 1) == 1300
    # monotone check S:87: E_t(s=5) >= E_t(s=40) with the memory term off
    pp = Params(L=50, S_tot=50, mem_mode=0)
    assert fl_oracle(pb, pp, 0, 5, 1) >= fl_oracle(pb, pp, 0, 40, 1)
    del p


@pytest.mark.parametrize("mode", [(0, 0, 0), (1, 0, 0), (2, 0, 0), (1, 1, 0), (1, 0, 1), (2, 1, 1), (0, 1, 1)])
def test_X_matches_per_kernel_rational_sum(mode):
    """O1 vs Eqs. 2-5 summed per kernel with exact rationals (independent of the integer scaling)."""
    mem, par, wse = mode
    rng = np.random.default_rng(11 + mem + 3 * par + 5 * wse)
    for _ in range(40):
        x = random_dnn(rng, threads=bool(par))
        L = int(rng.integers(3, 20)); S_tot = int(rng.integers(1, 40))
        p = Params(L=L, S_tot=S_tot, mem_mode=mem, par_mode=par, wse_mode=wse)
        pb = multi_dnn_problem([x])
        for _ in range(6):
            l = int(rng.integers(1, L + 1)); b = int(rng.integers(1, 9))
            want = f_L(x["rows"], x["t_p"], x["t_np"], x["M"], p, S_of(p, l), b)
            assert fl_oracle(pb, p, 0, l, b, M=x["M"]) == want


def test_latency_invariants():
    # saturation E_t(s) = E_t(N_1) for s >= N_1 (memory off); non-increasing in s
    # (off / bw); E_t(b=2) >= E_t(b=1).
    rng = np.random.default_rng(5)
    for _ in range(30):
        x = random_dnn(rng, n_max=12)
        pb = multi_dnn_problem([x])
        for mem in (0, 1):
            p = Params(L=32, S_tot=32, mem_mode=mem)
            f = [fl_oracle(pb, p, 0, l, 1, M=x["M"]) for l in range(1, 33)]
            assert all(f[i] >= f[i + 1] for i in range(31))
            f2 = [fl_oracle(pb, p, 0, l, 2, M=x["M"]) for l in range(1, 33)]
            assert all(a >= c for a, c in zip(f2, f))
        p = Params(L=32, S_tot=32, mem_mode=0)
        nmax = max(r[0] for r in x["rows"])
        if 1 <= nmax <= 31:
            sat = fl_oracle(pb, p, 0, nmax, 1)
            assert all(fl_oracle(pb, p, 0, l, 1) == sat for l in range(nmax, 33))


# ---------------------------------------------------------------- O2 -------

@pytest.mark.parametrize("smax", [50, 60, 80])
def test_fig3_knee_N1_20_is_9(golden, smax):
    """PAPER.md P:1627 (§4.3, Fig. 3): K_max=50, t_p=40, t_np=10, N_1=20 -> knee at 9 SMs."""
    g = golden("fig3.json")
    N = eq1_rows(g["K_max"], 20, 1)
    pb = single_dnn_problem([(n, 1, 0) for n in N], t_p=g["t_p"], t_np=g["t_np"])
    k, st = oracle.knee(pb, Params(L=smax, S_tot=smax, mem_mode=0), 1)
    assert st[0] == oracle.OK and int(k[0]) == g["pinned"][0]["knee"]


def test_fig3_unpinned_values_documented(golden):
    """N_1 = 40 / 60: the paper prints 24 / 31, the printed equations give 20 / 28
    (parity unpinned -- DESIGN.md §5). Cross-check against the survey's numbers."""
    g = golden("fig3.json")
    for u in g["unpinned"]:
        N = eq1_rows(g["K_max"], u["N1"], 1)
        pb = single_dnn_problem([(n, 1, 0) for n in N], t_p=g["t_p"], t_np=g["t_np"])
        k, _ = oracle.knee(pb, Params(L=80, S_tot=80, mem_mode=0), 1)
        assert int(k[0]) == u["equations_give"] != u["paper_knee"]


def _g(S, X):
    return F(S, X * X)


def test_knee_single_kernel_closed_form():
    """One kernel (K=1, R=1, n), memory off, b=1: for S < n, X = M(t_np S + t_p n) so g = S/X^2 peaks at
    S* = t_p n / t_np; for S >= n, X = M S (t_np + t_p) so g decreases.  Knee = best of
    {floor(S*), ceil(S*)} n [1, n-1] plus n (if n <= S_max), by exact comparison of the closed form."""
    rng = np.random.default_rng(3)
    for _ in range(200):
        n = int(rng.integers(1, 120)); t_p = int(rng.integers(1, 50)); t_np = int(rng.integers(1, 50))
        smax = int(rng.integers(1, 150))
        X = lambda S: (t_np * S + t_p * n) if S < n else S * (t_np + t_p)
        s_star = F(t_p * n, t_np)
        cands = {c for c in (int(s_star), int(s_star) + 1) if 1 <= c <= min(n - 1, smax)}
        cands |= {min(n, smax), 1}
        best = max(sorted(cands), key=lambda S: (_g(S, X(S)), -S))
        pb = single_dnn_problem([(n, 1, 0)], t_p=t_p, t_np=t_np)
        k, st = oracle.knee(pb, Params(L=smax, S_tot=smax, mem_mode=0), 1)
        assert int(k[0]) == best, (n, t_p, t_np, smax)


def test_knee_special_cases():
    # t_np = 0, one kernel -> knee = min(b n, S_max)
    for n, b, smax in [(10, 1, 40), (10, 3, 40), (50, 1, 40), (7, 2, 100)]:
        pb = single_dnn_problem([(n, 1, 0)], t_p=9, t_np=0)
        k, _ = oracle.knee(pb, Params(L=smax, S_tot=smax, mem_mode=0), b)
        assert int(k[0]) == min(b * n, smax)
    # flat latency curve (all N_i = 0: E_t = b t_np sum R, constant) -> knee = 1 (SPEC S:173 analogue)
    pb = single_dnn_problem([(0, 2, 0), (0, 1, 0)], t_p=5, t_np=7)
    assert int(oracle.knee(pb, Params(L=64, S_tot=64, mem_mode=0), 1)[0][0]) == 1
    # E_t = c / S (t_np = 0, every kernel wider than S_max, memory off) -> knee = S_max
    pb = single_dnn_problem([(500, 1, 0), (300, 2, 0)], t_p=5, t_np=0)
    assert int(oracle.knee(pb, Params(L=64, S_tot=64, mem_mode=0), 1)[0][0]) == 64


def test_knee_scale_invariance():
    # scaling t_p and t_np together leaves the knee unchanged (argmax of 1/(c^2 f^2 S))
    rng = np.random.default_rng(9)
    for _ in range(40):
        x = random_dnn(rng, n_max=60)
        c = int(rng.integers(2, 7))
        y = dict(x, t_p=x["t_p"] * c, t_np=x["t_np"] * c)
        p = Params(L=60, S_tot=60, mem_mode=0)
        k1 = oracle.knee(multi_dnn_problem([x]), p, 1)[0][0]
        k2 = oracle.knee(multi_dnn_problem([y]), p, 1)[0][0]
        assert k1 == k2


@pytest.mark.parametrize("mode", [(0, 0, 0), (1, 0, 0), (2, 0, 0), (1, 1, 1), (2, 1, 0), (1, 0, 1)])
def test_knee_brute_force_rational(mode):
    """O2 vs argmax over l of 1/(f_L^2 S(l)) with f_L from the per-kernel rational sum; L != S_tot too."""
    mem, par, wse = mode
    rng = np.random.default_rng(21 + mem + 7 * par + 13 * wse)
    for _ in range(40):
        x = random_dnn(rng, threads=bool(par))
        L = int(rng.integers(2, 24)); S_tot = int(rng.integers(1, 40))
        p = Params(L=L, S_tot=S_tot, mem_mode=mem, par_mode=par, wse_mode=wse)
        b = int(rng.integers(1, 6))
        vals = []
        for l in range(1, L + 1):
            f = f_L(x["rows"], x["t_p"], x["t_np"], x["M"], p, S_of(p, l), b)
            vals.append((1 / (f * f * S_of(p, l)) if f > 0 else None, l))
        if any(v is None for v, _ in vals):
            continue
        best = max(vals, key=lambda t: (t[0], -t[1]))[1]
        k, st = oracle.knee(multi_dnn_problem([x]), p, b)
        assert st[0] == oracle.OK and int(k[0]) == best


# ---------------------------------------------------------------- O3 -------

def brute_batch(x, p: Params):
    """Eqs. 9-12 by exhaustive enumeration with exact rationals: feasible iff b_lo <= b <= b_hi,
    f_L + b a <= SLO, f_L <= SLO/2; eta = b / (f_L^2 * S/S_tot); ties -> smaller l, then smaller b."""
    b_hi = min(p.b_max, x.get("bmax", 64))
    best = None
    for l in range(1, p.L + 1):
        S = S_of(p, l)
        for b in range(p.b_min, b_hi + 1):
            f = f_L(x["rows"], x["t_p"], x["t_np"], x["M"], p, S, b)
            if f + b * x["a"] > x["slo"] or f > F(x["slo"], 2):
                continue
            eta = F(b) / (f * f * F(S, p.S_tot))
            if best is None or eta > best[0]:
                best = (eta, l, b)
    return best


@pytest.mark.parametrize("mode", [(0, 0, 0), (1, 0, 0), (2, 0, 0), (1, 1, 0), (1, 0, 1), (1, 1, 1), (2, 1, 1)])
def test_batch_opt_brute_force_rational(mode):
    """North-star pin: 'brute-force enumeration of batch sizes on tiny scenarios'."""
    mem, par, wse = mode
    rng = np.random.default_rng(101 + mem + 7 * par + 13 * wse)
    seen_b = set()
    for _ in range(40):
        x = random_dnn(rng, threads=bool(par), n_max=20)
        L = int(rng.integers(2, 14)); S_tot = int(rng.integers(1, 24))
        p = Params(L=L, S_tot=S_tot, mem_mode=mem, par_mode=par, wse_mode=wse, b_min=1, b_max=6,
                   margin=int(rng.integers(0, 3)))
        slo_scale = int(rng.integers(1, 6))
        f1 = f_L(x["rows"], x["t_p"], x["t_np"], x["M"], p, S_of(p, L), 1)
        x["slo"] = max(1, int(f1 * 2 * slo_scale) + int(rng.integers(0, 50)))
        x["a"] = int(rng.integers(0, 30))
        x["slot"] = 1
        p = p.replace(slot_us=1)
        o = oracle.batch_opt(multi_dnn_problem([x]), p)
        best = brute_batch(x, p)
        if best is None:
            assert o["status"][0] == oracle.INFEASIBLE
            continue
        assert o["status"][0] == oracle.OK
        assert int(o["batch"][0]) == best[2]
        assert int(o["demand"][0]) == min(L, best[1] + p.margin)
        seen_b.add(best[2])
        # knee at b* (O2 at the chosen batch)
        assert int(o["knee"][0]) == int(oracle.knee(multi_dnn_problem([x]), p, best[2])[0][0])
    del seen_b


def test_eq12_boundary_and_spec_feasibility():
    # SPEC S:238 (Eqs. 11-12): f_L = 28 ms with SLO 50 ms is infeasible (28 > 25).  A DNN of one empty
    # kernel with t_np = 28 ms has f_L = b * 28 ms at every GPU% (Eq. 4 per_request).
    x = dict(rows=[(0, 1, 0)], t_p=1, t_np=28000, M=1, slo=50000, a=481)
    p = Params(L=10, S_tot=10, mem_mode=0, slot_us=1000)
    assert oracle.batch_opt(multi_dnn_problem([x]), p)["status"][0] == oracle.INFEASIBLE
    # boundary: SLO = 56 ms -> f_L = SLO/2 exactly (Eq. 12 is <=) and 28 + 0.481 <= 56 (Eq. 11): feasible, b = 1
    x["slo"] = 56000
    o = oracle.batch_opt(multi_dnn_problem([x]), p)
    assert o["status"][0] == oracle.OK and o["batch"][0] == 1 and o["demand"][0] == 1
    # f_L = 20 ms at b = 16, C = 16 * 481 us ~ 7.7 ms, SLO 50 -> feasible
    y = dict(rows=[(0, 1, 0)], t_p=1, t_np=1250, M=1, slo=50000, a=481)
    o = oracle.batch_opt(multi_dnn_problem([y]), Params(L=10, S_tot=10, mem_mode=0, slot_us=1000, b_min=16, b_max=16))
    assert o["status"][0] == oracle.OK and o["batch"][0] == 16


def test_batch_relaxation_monotone():
    # removing (relaxing) a constraint never decreases the optimum eta.
    rng = np.random.default_rng(77)
    for _ in range(30):
        x = random_dnn(rng, n_max=20)
        p = Params(L=10, S_tot=16, mem_mode=1, b_max=6, slot_us=1)
        f1 = f_L(x["rows"], x["t_p"], x["t_np"], x["M"], p, 16, 1)
        x["a"] = int(rng.integers(0, 20))
        etas = []
        for k in (1, 2, 3, 5):
            x["slo"] = int(f1 * 2 * k) + 1
            best = brute_batch(x, p)
            o = oracle.batch_opt(multi_dnn_problem([x]), p)
            if best is None:
                assert o["status"][0] == oracle.INFEASIBLE
                etas.append(F(0))
                continue
            assert (int(o["demand"][0]), int(o["batch"][0])) == (best[1], best[2])
            etas.append(best[0])
        assert all(etas[i] <= etas[i + 1] for i in range(len(etas) - 1))


def test_validation_statuses():
    p = Params(L=10, S_tot=10, mem_mode=1, slot_us=100)
    base = dict(rows=[(3, 1, 10)], t_p=5, t_np=2, M=10, slo=10000, a=10)
    ok = oracle.batch_opt(multi_dnn_problem([base]), p)["status"][0]
    assert ok == oracle.OK
    bad = [dict(base, t_p=0), dict(base, slo=10050), dict(base, rows=[(3, 0, 10)]), dict(base, M=0),
           dict(base, rows=[(0, 1, 0)], t_np=0), dict(base, a=-1), dict(base, bmax=0)]
    for b in bad:
        assert oracle.batch_opt(multi_dnn_problem([b]), p)["status"][0] == oracle.INVALID, b
    huge = dict(base, rows=[(4_000_000_000, 65535, 4_000_000_000)] * 3, t_p=2**30)
    assert oracle.batch_opt(multi_dnn_problem([huge]), p)["status"][0] == oracle.OVERFLOW
    assert oracle.batch_opt(multi_dnn_problem([dict(base, bmax=3)]), p.replace(b_min=4))["status"][0] == oracle.INFEASIBLE
