"""Test-only helpers: independent exact (Fraction) evaluations written directly from the paper's
equations, per kernel, un-multiplied -- a different code path from the oracle's integer X."""
from __future__ import annotations

from fractions import Fraction as F
from math import ceil, floor

import numpy as np

from synth import Params, make_problem


def S_of(p: Params, l: int) -> int:
    return -(-l * p.S_tot // p.L)


def N_of(p: Params, n: int, b: int) -> int:
    return b * n if p.par_mode == 0 else -(-(b * n) // 2048)


def f_L(rows, t_p, t_np, M, p: Params, S: int, b: int) -> F:
    """E_t (Eq. 5) for S SMs and batch b, evaluated per kernel with exact rationals:
    Eq. 2 E_i = N_i t_p / max(1, min(S, N_i)); Eq. 3 E_m = d S / M (verbatim) or d / (M S) (bw);
    Eq. 4 W_se = b sum R (t_np + E_m) (per_request) or sum R t_np + b sum R E_m (per_launch)."""
    M = 1 if p.mem_mode == 0 else M
    Et = F(0)
    for (n, R, d) in rows:
        N = N_of(p, n, b)
        Ei = F(N * t_p, max(1, min(S, N)))
        Em = F(0) if p.mem_mode == 0 else (F(d, M * S) if p.mem_mode == 1 else F(d * S, M))
        if p.wse_mode == 0:
            Wse = b * R * (t_np + Em)
        else:
            Wse = R * t_np + b * R * Em
        Et += Wse + R * Ei
    return Et


def eq1_rows(K: int, p: int, b: int = 1):
    """Eq. 1: N_1 = p b, N_i = floor(N_{i-1} - p b / K), clamped at 0, exact rationals."""
    N = [F(p * b)]
    for _ in range(1, K):
        N.append(F(max(0, floor(N[-1] - F(p * b, K)))))
    return [int(x) for x in N]


def single_dnn_problem(rows, t_p, t_np, M=1, slo=10**8, a=0, bmax=64):
    n = [x[0] for x in rows]; r = [x[1] for x in rows]; d = [x[2] for x in rows]
    return make_problem([0, 1], [0, len(rows)], [t_p], [t_np], [M], [slo], [a], [bmax], n, r, d)


def multi_dnn_problem(dnns, scen_sizes=None):
    """dnns: list of dict(rows=[(n,R,d)], t_p, t_np, M, slo, a, bmax). One scenario unless scen_sizes."""
    if scen_sizes is None:
        scen_sizes = [len(dnns)]
    off = np.concatenate([[0], np.cumsum(scen_sizes)])
    roff = np.concatenate([[0], np.cumsum([len(x["rows"]) for x in dnns])])
    cols = lambda k, default=None: [x.get(k, default) for x in dnns]
    n = [r[0] for x in dnns for r in x["rows"]]
    R = [r[1] for x in dnns for r in x["rows"]]
    d = [r[2] for x in dnns for r in x["rows"]]
    return make_problem(off, roff, cols("t_p"), cols("t_np"), cols("M", 1), cols("slo", 10**8), cols("a", 0),
                        cols("bmax", 64), n, R, d)


def random_dnn(rng: np.random.Generator, K_max=6, n_max=30, d_max=5000, threads=False):
    K = int(rng.integers(1, K_max + 1))
    rows = []
    for _ in range(K):
        n = int(rng.integers(0, n_max + 1))
        if threads:
            n = int(rng.integers(0, n_max * 2048 + 1))
        rows.append((n, int(rng.integers(1, 4)), int(rng.integers(0, d_max + 1))))
    return dict(rows=rows, t_p=int(rng.integers(1, 60)), t_np=int(rng.integers(0, 20)), M=int(rng.integers(1, 200)))
