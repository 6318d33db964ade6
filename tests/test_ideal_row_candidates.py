"""The candidate rule k_ideal_rows uses for a row's knee (ideal.cu, DSTACK_IDEAL_ROW_CANDIDATES): each latency
regime's end levels plus the levels next to the regime's real maximum of S / X^2 contain the exact argmax over all
L levels (ties to the smaller level).  Checked here against the brute-force scan with exact rationals on random
one-row DNNs in every model mode and with L < S_tot, L = S_tot and L > S_tot; the GPU parity tests check the
kernel itself against the oracle."""
import math
from fractions import Fraction as F

import numpy as np


def candidate_levels(L, St, N, wC, Mtp, m1, vb):
    """The levels the kernel evaluates (before mapping each to the smallest level with the same S)."""
    cands = []
    lmax = (min(N - 1, St) * L // St) if N >= 1 else 0
    for seg in (0, 1):
        l0, l1 = (1, lmax) if seg == 0 else (lmax + 1, L)
        if l0 > l1:
            continue
        cands += [l0, l1]
        beta = wC + (Mtp if seg == 1 and N >= 1 else 0)
        gamma = m1 + (Mtp * N if seg == 0 else 0)
        if vb > 0:
            sst = (-beta + math.sqrt(beta * beta + 12.0 * vb * gamma)) / (6.0 * vb)
        elif beta > 0:
            sst = gamma / beta
        else:
            sst = St
        sst = min(max(sst, 0.0), St + 4.0)
        if L <= St:
            lc = math.floor(sst * L / St)
            cands += [l for l in range(lc - 2, lc + 4) if l0 <= l <= l1]
        else:
            sc = math.floor(sst)
            for S in range(sc - 2, sc + 4):
                if 1 <= S <= St:
                    l = (S - 1) * L // St + 1
                    if l0 <= l <= l1:
                        cands.append(l)
    return cands


def test_row_knee_candidates_contain_the_argmax():
    rng = np.random.default_rng(3)
    tot = 0
    for _ in range(400):
        L = int(rng.choice([37, 64, 100, 148, 200, 255])); St = int(rng.choice([40, 64, 80, 148, 256]))
        mem = int(rng.integers(0, 3)); par = int(rng.integers(0, 2)); wse = int(rng.integers(0, 2))
        b = int(rng.integers(1, 65)); tp = int(rng.integers(1, 60)); tnp = int(rng.integers(0, 20))
        M = 1 if mem == 0 else int(rng.integers(1, 100000))
        n = int(rng.integers(0, 4 * St)) if par == 0 else int(rng.integers(0, 4 * St * 2048))
        dd = int(rng.integers(0, 10**7))
        N = b * n if par == 0 else -(-(b * n) // 2048)
        wC = (b if wse == 0 else 1) * tnp * M

        def s_of(l):
            return -(-l * St // L)

        def X(S):
            x = wC * S + (M * tp * max(N, S) if N >= 1 else 0)
            if mem == 1:
                x += b * dd
            elif mem == 2:
                x += b * dd * S * S
            return x

        if X(1) == 0:
            continue

        def key(l):
            S = s_of(l)
            return (F(S, X(S) ** 2), -l)

        brute = max(range(1, L + 1), key=key)
        cands = candidate_levels(L, St, N, wC, M * tp, b * dd if mem == 1 else 0, b * dd if mem == 2 else 0)
        got = max([(s_of(l) - 1) * L // St + 1 for l in cands], key=key)
        assert got == brute, dict(L=L, St=St, mem=mem, par=par, wse=wse, b=b, N=N)
        tot += 1
    assert tot > 300
