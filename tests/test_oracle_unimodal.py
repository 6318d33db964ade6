"""Pins for the structure the a2/a3 searches of k_prof_lane rely on ("a2/a3 by search").

The paper's objective at b = 1 (Eq. 6; R5): maximise 1 / (f_L(S)^2 S), i.e. S / X(S)^2 with
X = E_t S M (O1).  Per kernel (Eqs. 2-5), E_i S = t_p max(N_i, S) for N_i >= 1, so X is a sum of convex functions
of S and the objective is unimodal in S.  The kernel replaces the scan of every width by a binary search that
keeps the left candidate on ties; these tests check, with exact rationals evaluated kernel by kernel from the
equations (tests/helpers.f_L, independent of the oracle's integer X), that

  * the objective never rises again after it has fallen (at most two maxima, adjacent),
  * the binary search returns the leftmost maximum (the oracle's tie rule: smaller S),
  * the b >= 2 certificate's segment supremum is attained in the first segment whose
    right end is past the peak, as the kernel's search assumes (each segment's supremum taken exactly at its
    end points and its stationary point).
"""
from fractions import Fraction as F

import numpy as np
import pytest

from synth import Params
from tests.helpers import f_L, random_dnn


def objective(dnn, p, S):
    Et = f_L(dnn["rows"], dnn["t_p"], dnn["t_np"], dnn["M"], p, S, 1)
    return F(1) / (Et * Et * S) if Et != 0 else None


def leftmost_max_by_search(vals):
    """The kernel's knee search on a list indexed 1..N (vals[0] unused)."""
    lo, hi = 1, len(vals) - 1
    while lo < hi:
        mid = (lo + hi) // 2
        if vals[mid] >= vals[mid + 1]:
            hi = mid
        else:
            lo = mid + 1
    return lo


def rand_profiles(seed, count, S_tot):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        dnn = random_dnn(rng, K_max=8, n_max=2 * S_tot, d_max=10 ** 6)
        if rng.random() < 0.25:
            dnn["t_np"] = 0          # C1 = 0: flat stretches of X, the tie-prone case
        out.append(dnn)
    return out


@pytest.mark.parametrize("mem_mode", [0, 1, 2])
def test_b1_objective_is_unimodal_and_search_finds_leftmost_max(mem_mode):
    S_tot = 24
    p = Params(L=S_tot, S_tot=S_tot, mem_mode=mem_mode)
    checked = 0
    for dnn in rand_profiles(100 + mem_mode, 120, S_tot):
        vals = [None] + [objective(dnn, p, S) for S in range(1, S_tot + 1)]
        if any(v is None for v in vals[1:]):
            continue   # E_t = 0 (no work at all): INVALID before a2
        fell = False
        for S in range(1, S_tot):
            if vals[S + 1] < vals[S]:
                fell = True
            elif vals[S + 1] > vals[S]:
                assert not fell, f"objective rises again at S={S + 1}: {dnn}"
        best = max(vals[1:])
        argmaxes = [S for S in range(1, S_tot + 1) if vals[S] == best]
        assert len(argmaxes) <= 2 and argmaxes[-1] - argmaxes[0] <= 1, (argmaxes, dnn)
        assert leftmost_max_by_search(vals) == argmaxes[0]
        checked += 1
    assert checked > 100


def test_unimodal_on_coarse_levels():
    """L < S_tot: the candidates are the widths S(l) = ceil(l S_tot / L) (a subsequence), still unimodal."""
    S_tot, L = 30, 11
    p = Params(L=L, S_tot=S_tot, mem_mode=1)
    for dnn in rand_profiles(7, 80, S_tot):
        Ss = [None] + [-(-l * S_tot // L) for l in range(1, L + 1)]
        vals = [None] + [objective(dnn, p, Ss[l]) for l in range(1, L + 1)]
        if any(v is None for v in vals[1:]):
            continue
        best = max(vals[1:])
        assert leftmost_max_by_search(vals) == min(l for l in range(1, L + 1) if vals[l] == best)


def test_certificate_peak_segment():
    """The b >= 2 bound of DESIGN.md §6: on segment m (s in [m, m+1)) eta <= s / (alpha_m s + beta_m)^2 with
    alpha_m = 2 C1 + Mtp PA[m], beta_m = Mtp (Q[m] + W>) + mem.  Its supremum over (0, S_tot / 2] lies in the
    first segment m with alpha_m (m + 1) >= beta_m (else the last)."""
    S_tot = 40
    half = F(S_tot, 2)
    rng = np.random.default_rng(11)
    for _ in range(150):
        dnn = random_dnn(rng, K_max=8, n_max=2 * S_tot, d_max=10 ** 6)
        M, t_p, t_np = dnn["M"], dnn["t_p"], dnn["t_np"]
        RT = sum(R for (_, R, _) in dnn["rows"])
        C1 = t_np * M * RT
        Mtp = M * t_p
        Wgt = sum(R * n for (n, R, _) in dnn["rows"] if n > S_tot)
        mem = sum(R * d for (_, R, d) in dnn["rows"])   # the bw term (mem_mode 1)

        def ab(m):
            PA = sum(R for (n, R, _) in dnn["rows"] if 1 <= n <= m)
            Q = sum(R * n for (n, R, _) in dnn["rows"] if m < n <= S_tot)
            return 2 * C1 + Mtp * PA, Mtp * (Q + Wgt) + mem

        mh = S_tot // 2
        if ab(mh)[1] == 0:
            continue   # beta = 0 at S_tot / 2: a bound of 1 / (alpha^2 m), not the tested case

        def seg_sup(m):
            a, b = ab(m)
            lo, hi = F(m), min(F(m + 1), half)
            pts = [lo, hi] + ([F(b, a)] if a and lo <= F(b, a) <= hi else [])
            return max((s / (a * s + b) ** 2 for s in pts if s > 0), default=F(0))

        m0 = next((m for m in range(mh + 1) if ab(m)[0] * (m + 1) >= ab(m)[1]), mh)
        sups = [seg_sup(m) for m in range(mh + 1)]
        assert sups[m0] == max(sups), (m0, sups.index(max(sups)), dnn)
