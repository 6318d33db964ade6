"""Pins for F3, online knee discovery ("our platform initially provides it a
nominal, 30%, GPU. The GPU% is then readjusted using Dynamic GPU resource reconfiguration to find the knee
based on the inference latency using a simple binary search"; reading R22 in DESIGN.md §3.4).

The paper prints no probe sequence or result, so the pins are: an independent re-trace of the search with
latencies from the per-kernel rational model (tests/helpers.py, not the oracle's integer X); the closed-form
single-kernel knee (a unimodal objective, where a binary search must find the exact Eq. 6 argmax); the
local-maximum property and the step bound on random DNNs; equality with O2 whenever the objective is unimodal.
"""
from fractions import Fraction as F
from math import ceil, log2

import numpy as np
import pytest

import oracle
from synth import Params
from tests.helpers import S_of, f_L, multi_dnn_problem, random_dnn, single_dnn_problem


def objective(x, p, b):
    """Eq. 6's objective g(l) = 1/(f_L(l,b)^2 S(l)) over l = 1..L from the rational per-kernel model."""
    g = [None]
    for l in range(1, p.L + 1):
        S = S_of(p, l)
        f = f_L(x["rows"], x["t_p"], x["t_np"], x["M"], p, S, b)
        g.append(1 / (f * f * S))
    return g


def retrace(g, L):
    """The search of P:1194 as read in R22, written out: start at ceil(0.3 L), then midpoints."""
    lo, hi, trace = 1, L, []
    while lo < hi:
        m = ceil(F(3 * L, 10)) if not trace else (lo + hi) // 2
        m = min(max(m, lo), hi - 1)
        trace.append(m)
        if g[m + 1] > g[m]:
            lo = m + 1
        else:
            hi = m
    return lo, trace


@pytest.mark.parametrize("mode", [(0, 0, 0), (1, 0, 0), (2, 0, 0), (1, 1, 1), (1, 0, 1)])
def test_retrace_random_dnns(mode):
    mem, par, wse = mode
    rng = np.random.default_rng(5 + mem + 3 * par + 11 * wse)
    unimodal = 0
    for _ in range(60):
        x = random_dnn(rng, threads=bool(par))
        if all(r[0] == 0 for r in x["rows"]) and x["t_np"] == 0 and mem == 0:
            continue   # latency identically 0: INVALID
        L = int(rng.integers(1, 60)); S_tot = int(rng.integers(L, 80))   # L <= S_tot: S(l) strictly increasing
        p = Params(L=L, S_tot=S_tot, mem_mode=mem, par_mode=par, wse_mode=wse)
        b = int(rng.integers(1, 5))
        pb = multi_dnn_problem([x])
        k, steps, st, tr = oracle.knee_probe(pb, p, b, trace=True)
        if st[0] != oracle.OK:
            continue
        g = objective(x, p, b)
        want, trace = retrace(g, L)
        assert int(k[0]) == want and int(steps[0]) == len(trace) and tr[0][:len(trace)].tolist() == trace
        # local maximum of the objective; at most ceil(log2 L) + 1 steps (two latency probes each)
        kk = int(k[0])
        assert kk == 1 or g[kk] > g[kk - 1]
        assert kk == L or g[kk + 1] <= g[kk]
        assert len(trace) <= (ceil(log2(L)) + 1 if L > 1 else 0)
        if L > 1:
            assert trace[0] == min(max(ceil(F(3 * L, 10)), 1), L - 1)   # the nominal 30% start
        # where the objective is unimodal over the levels the probe finds Eq. 6's exact argmax (O2)
        d = [g[l + 1] > g[l] for l in range(1, L)]
        if all(d[i] or not d[i + 1] for i in range(len(d) - 1)):
            unimodal += 1
            assert kk == int(oracle.knee(pb, p, b)[0][0])
    assert unimodal >= 10


def test_single_kernel_closed_form():
    """One kernel, memory off, b = 1: g(S) = S/X^2 with X = t_np S + t_p n (S < n), S (t_np + t_p) (S >= n)
    is unimodal, so the binary search lands on the closed-form knee (test_oracle_model.py's construction)."""
    rng = np.random.default_rng(17)
    for _ in range(200):
        n = int(rng.integers(1, 120)); t_p = int(rng.integers(1, 50)); t_np = int(rng.integers(1, 50))
        smax = int(rng.integers(1, 150))
        X = lambda S: (t_np * S + t_p * n) if S < n else S * (t_np + t_p)
        s_star = F(t_p * n, t_np)
        cands = {c for c in (int(s_star), int(s_star) + 1) if 1 <= c <= min(n - 1, smax)}
        cands |= {min(n, smax), 1}
        best = max(sorted(cands), key=lambda S: (F(S, X(S) ** 2), -S))
        pb = single_dnn_problem([(n, 1, 0)], t_p=t_p, t_np=t_np)
        k, steps, st = oracle.knee_probe(pb, Params(L=smax, S_tot=smax, mem_mode=0), 1)
        assert st[0] == oracle.OK and int(k[0]) == best, (n, t_p, t_np, smax)


def test_statuses_match_knee():
    """Validation is the knee's (dstack_knee): INVALID / OVERFLOW DNNs get knee 0 and no probes."""
    x = dict(rows=[(10, 1, 100)], t_p=20, t_np=3, M=100)
    bad = dict(rows=[(10, 0, 100)], t_p=20, t_np=3, M=100)          # R = 0: INVALID
    big = dict(rows=[(4_000_000_000, 65535, 0)] * 2, t_p=2**30, t_np=3, M=100)   # OVERFLOW
    pb = multi_dnn_problem([x, bad, big])
    p = Params(L=100, S_tot=148)
    k, steps, st = oracle.knee_probe(pb, p, 1)
    _, st2 = oracle.knee(pb, p, 1)
    assert st.tolist() == st2.tolist() == [oracle.OK, oracle.INVALID, oracle.OVERFLOW]
    assert k.tolist()[1:] == [0, 0] and steps.tolist()[1:] == [0, 0] and steps[0] > 0
