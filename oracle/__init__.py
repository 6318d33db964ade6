"""CPU ORACLE -- test infrastructure only.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
(``paper_2304_13541_b200``) never imports it.  Plain C definitions live in
``oracle/oracle.c`` (exact integer arithmetic, brute force); this file is a
ctypes shim over ``oracle/liboracle.so``.

Parity status per function (DESIGN.md §5 lists the pins):
  X (O1), knee (O2), batch_opt (O3), wmaxmin (O4), cycle (O5), ideal (O6):
  pinned by tests/test_oracle_*.py (paper values, closed forms, brute force).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from synth import Params, Problem

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "liboracle.so")

OK, INFEASIBLE, OVERFLOW, INVALID, OVERSUBSCRIBED = 0, 1, 2, 3, 4


class OrProblem(C.Structure):
    _fields_ = [("num_scen", C.c_int32), ("num_dnn", C.c_int32),
                ("scen_dnn_off", C.c_void_p), ("dnn_row_off", C.c_void_p),
                ("t_p", C.c_void_p), ("t_np", C.c_void_p), ("mem_bw", C.c_void_p), ("slo_us", C.c_void_p),
                ("asm_us", C.c_void_p), ("bmax", C.c_void_p),
                ("n", C.c_void_p), ("r", C.c_void_p), ("d", C.c_void_p)]


class OrParams(C.Structure):
    _fields_ = [(k, C.c_int32) for k in
                ("L", "S_tot", "slot_us", "mem_mode", "margin", "par_mode", "wse_mode", "b_min", "b_max", "ideal",
                 "below_knee", "reconf_us")]


class OrOut(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in
                ("demand", "batch", "knee", "status", "alloc_q16", "level", "runs", "served",
                 "scen_status", "T_us", "u_static", "u", "thr", "misses", "u_ideal", "thr_ideal", "below")]


class OrCycSum(C.Structure):
    _fields_ = [("occ_static_sum", C.c_int64), ("occ_sum", C.c_int64), ("served_total", C.c_int64),
                ("misses", C.c_int32), ("status", C.c_int32), ("trace_n", C.c_int32), ("below", C.c_int32)]


class OrSimOut(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ("status", "T_us", "arrived", "in_slo", "late", "unserved", "occ_sum", "runs",
                                          "misses", "realloc", "series")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise RuntimeError(f"{LIB} missing: run __graft_entry__.build()")
        L = C.CDLL(LIB)
        P = C.POINTER
        L.oracle_X.argtypes = [P(OrProblem), P(OrParams), C.c_int64, C.c_int32, C.c_int32,
                               P(C.c_uint64), P(C.c_uint64)]
        L.oracle_knee.argtypes = [P(OrProblem), P(OrParams), C.c_int32, C.c_void_p, C.c_void_p]
        L.oracle_knee_probe.argtypes = [P(OrProblem), P(OrParams), C.c_int32] + [C.c_void_p] * 4
        L.oracle_batch_opt.argtypes = [P(OrProblem), P(OrParams)] + [C.c_void_p] * 4
        L.oracle_wmaxmin.argtypes = [C.c_int32, C.c_void_p, C.c_int32, C.c_void_p]
        L.oracle_cycle_direct.argtypes = ([C.c_int32] + [C.c_void_p] * 4 + [C.c_int32] * 3 + [C.c_void_p] * 4
                                          + [P(OrCycSum), C.c_int32] + [C.c_void_p] * 6)
        L.oracle_cycle_direct_ex.argtypes = ([C.c_int32] + [C.c_void_p] * 4 + [C.c_int32] * 3 + [C.c_void_p]
                                             + [C.c_int32] + [C.c_void_p] * 4 + [P(OrCycSum), C.c_int32]
                                             + [C.c_void_p] * 6)
        L.oracle_cycle_direct_bk.argtypes = ([C.c_int32] + [C.c_void_p] * 5 + [C.c_int32] * 3 + [C.c_void_p] * 3
                                             + [P(OrCycSum), C.c_int32] + [C.c_void_p] * 7)
        L.oracle_temporal_direct.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32] + [C.c_void_p] * 3
        L.oracle_gslice_direct.argtypes = ([C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32]
                                           + [C.c_void_p] * 5)
        L.oracle_compare.argtypes = [P(OrProblem), P(OrParams)] + [C.c_void_p] * 4 + [C.c_int64, C.c_int32]
        L.oracle_maxthr_direct.argtypes = ([C.c_int32] + [C.c_void_p] * 3 + [C.c_int32] * 3 + [C.c_int64, C.c_void_p])
        L.oracle_maxthr.argtypes = ([P(OrProblem), P(OrParams), C.c_int64] + [C.c_void_p] * 4 + [C.c_int64, C.c_int32])
        L.oracle_cluster.argtypes = [P(OrProblem), P(OrParams), C.c_int32] + [C.c_void_p] * 3 + [C.c_int64, C.c_int32]
        L.oracle_simulate.argtypes = [P(OrProblem), P(OrParams), C.c_void_p, C.c_int32, C.c_uint64, C.c_int32,
                                      C.c_int64, P(OrSimOut), C.c_void_p, C.c_int64, C.c_int32]
        L.oracle_ideal_direct.argtypes = ([C.c_int32] + [C.c_void_p] * 6 + [C.c_int32, C.c_int64]
                                          + [C.c_void_p] * 3)
        L.oracle_ideal_rows.argtypes = [P(OrProblem), P(OrParams), C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]
        L.oracle_eval.argtypes = [P(OrProblem), P(OrParams), P(OrOut), C.c_int32]
        L.oracle_eval_subset.argtypes = [P(OrProblem), P(OrParams), P(OrOut), C.c_void_p, C.c_int64, C.c_int32]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _problem(pb: Problem) -> OrProblem:
    return OrProblem(pb.num_scen, pb.num_dnn, _p(pb.scen_dnn_off), _p(pb.dnn_row_off), _p(pb.t_p), _p(pb.t_np),
                     _p(pb.mem_bw), _p(pb.slo_us), _p(pb.asm_us), _p(pb.bmax), _p(pb.n), _p(pb.r), _p(pb.d))


def _params(p: Params) -> OrParams:
    return OrParams(p.L, p.S_tot, p.slot_us, p.mem_mode, p.margin, p.par_mode, p.wse_mode, p.b_min, p.b_max,
                    p.ideal, p.below_knee, p.reconf_us)


def X(pb: Problem, p: Params, dnn: int, l: int, b: int) -> int:
    """O1: X(l, b) = E_t * S(l) * M (exact Python int)."""
    lo, hi = C.c_uint64(), C.c_uint64()
    rc = lib().oracle_X(C.byref(_problem(pb)), C.byref(_params(p)), dnn, l, b, C.byref(lo), C.byref(hi))
    assert rc == 0
    return (hi.value << 64) | lo.value


def knee(pb: Problem, p: Params, b: int):
    """O2: (knee[num_dnn] uint16, status[num_dnn] uint8) at batch b."""
    k = np.zeros(pb.num_dnn, np.uint16); st = np.zeros(pb.num_dnn, np.uint8)
    assert lib().oracle_knee(C.byref(_problem(pb)), C.byref(_params(p)), b, _p(k), _p(st)) == 0
    return k, st


def knee_probe(pb: Problem, p: Params, b: int, trace: bool = False):
    """F3: binary-search knee from the nominal 30%. Returns (knee, probes, status[, trace[D, 16]])."""
    D = pb.num_dnn
    k = np.zeros(D, np.uint16); pr = np.zeros(D, np.uint8); st = np.zeros(D, np.uint8)
    tr = np.full((D, 16), -1, np.int32) if trace else None
    assert lib().oracle_knee_probe(C.byref(_problem(pb)), C.byref(_params(p)), b, _p(k), _p(pr), _p(st), _p(tr)) == 0
    return (k, pr, st, tr) if trace else (k, pr, st)


def batch_opt(pb: Problem, p: Params):
    """O3: dict(demand, batch, knee, status) per DNN."""
    D = pb.num_dnn
    o = dict(demand=np.zeros(D, np.uint16), batch=np.zeros(D, np.uint8), knee=np.zeros(D, np.uint16),
             status=np.zeros(D, np.uint8))
    assert lib().oracle_batch_opt(C.byref(_problem(pb)), C.byref(_params(p)), _p(o["demand"]), _p(o["batch"]),
                                  _p(o["knee"]), _p(o["status"])) == 0
    return o


def wmaxmin(demand, L: int) -> np.ndarray:
    """O4: Q16.16 allocations."""
    d = np.ascontiguousarray(demand, np.uint16)
    a = np.zeros(d.shape[0], np.uint32)
    assert lib().oracle_wmaxmin(d.shape[0], _p(d), L, _p(a)) == 0
    return a


def cycle_direct(g, sl_slots, bstar, dtab, b_lo: int, L: int, nslots: int, trace_cap: int = 4096, count0=None,
                 fill_order: int = 0):
    """O5 with direct per-DNN inputs. dtab: array [n, 64], dtab[j, b-1] = d_j(b) slots.
    fill_order (O9): 0 D-STACK (runs so far), 1 Max-Min fair (smallest GPU% first), 2 max-throughput (shortest
    run first); ties by index.  Returns also busy[j] = slots covered by j's runs."""
    g = np.ascontiguousarray(g, np.int32); sl = np.ascontiguousarray(sl_slots, np.int32)
    bs = np.ascontiguousarray(bstar, np.int32)
    n = g.shape[0]
    dt = np.zeros((n, 64), np.int64)
    dtab = np.asarray(dtab, np.int64)
    dt[:, : dtab.shape[1]] = dtab
    runs = np.zeros(n, np.int32); served = np.zeros(n, np.int64); jm = np.zeros(n, np.int32)
    s = OrCycSum()
    tr = [np.zeros(trace_cap, np.int32) for _ in range(6)]
    c0 = None if count0 is None else np.ascontiguousarray(count0, np.int64)
    busy = np.zeros(n, np.int64)
    rc = lib().oracle_cycle_direct_ex(n, _p(g), _p(sl), _p(bs), _p(dt), b_lo, L, nslots, _p(c0), fill_order, _p(runs),
                                      _p(served), _p(jm), _p(busy), C.byref(s), trace_cap, *[_p(t) for t in tr])
    assert rc == 0
    k = s.trace_n
    trace = dict(dnn=tr[0][:k], start=tr[1][:k], end=tr[2][:k], batch=tr[3][:k], kind=tr[4][:k], rep=tr[5][:k])
    return dict(occ_static_sum=s.occ_static_sum, occ_sum=s.occ_sum, served_total=s.served_total,
                misses=s.misses, status=s.status, runs=runs, served=served, jmiss=jm, trace=trace, busy=busy,
                u_static=s.occ_static_sum / (nslots * L) if nslots else 0.0,
                u=s.occ_sum / (nslots * L) if nslots else 0.0)


def cycle_direct_bk(g, sl_slots, bstar, dtab, dlow, b_lo: int, L: int, nslots: int, trace_cap: int = 4096):
    """O5 + F1 below-knee fallback. dlow: array [n, 256], dlow[j, l] = run slots of j's b*
    batch at level l < g_j including the launch latency (0 = unusable). Trace kind 2 = below-knee static run,
    trace level = the run's GPU% level."""
    g = np.ascontiguousarray(g, np.int32); sl = np.ascontiguousarray(sl_slots, np.int32)
    bs = np.ascontiguousarray(bstar, np.int32)
    n = g.shape[0]
    dt = np.zeros((n, 64), np.int64)
    dtab = np.asarray(dtab, np.int64)
    dt[:, : dtab.shape[1]] = dtab
    dl = np.zeros((n, 256), np.int64)
    dlow = np.asarray(dlow, np.int64)
    dl[:, : dlow.shape[1]] = dlow
    runs = np.zeros(n, np.int32); served = np.zeros(n, np.int64); jm = np.zeros(n, np.int32)
    s = OrCycSum()
    tr = [np.zeros(trace_cap, np.int32) for _ in range(7)]
    rc = lib().oracle_cycle_direct_bk(n, _p(g), _p(sl), _p(bs), _p(dt), _p(dl), b_lo, L, nslots, _p(runs),
                                      _p(served), _p(jm), C.byref(s), trace_cap, *[_p(t) for t in tr])
    assert rc == 0
    k = s.trace_n
    trace = dict(dnn=tr[0][:k], start=tr[1][:k], end=tr[2][:k], batch=tr[3][:k], kind=tr[4][:k], rep=tr[5][:k],
                 level=tr[6][:k])
    return dict(occ_static_sum=s.occ_static_sum, occ_sum=s.occ_sum, served_total=s.served_total,
                misses=s.misses, status=s.status, below=s.below, runs=runs, served=served, jmiss=jm, trace=trace,
                u_static=s.occ_static_sum / (nslots * L) if nslots else 0.0,
                u=s.occ_sum / (nslots * L) if nslots else 0.0)


def temporal_direct(lvl, sl_slots, dL, nslots: int):
    """O9 temporal sharing with direct inputs: slices proportional to SLO, back-to-back runs at 100% GPU."""
    lv = np.ascontiguousarray(lvl, np.int32); sl = np.ascontiguousarray(sl_slots, np.int32)
    d = np.ascontiguousarray(dL, np.int64)
    n = lv.shape[0]
    slice_, runs = np.zeros(n, np.int64), np.zeros(n, np.int64)
    occ = C.c_int64()
    assert lib().oracle_temporal_direct(n, _p(lv), _p(sl), _p(d), nslots, _p(slice_), _p(runs), C.byref(occ)) == 0
    return dict(slice=slice_, runs=runs, occ_num=occ.value)


def gslice_direct(lvl, dk, nslots: int, L: int):
    """O9 static spatial sharing (GSLICE CSS) with direct inputs; home[j] = -1 resident, slot index, -2 idle."""
    lv = np.ascontiguousarray(lvl, np.int32); d = np.ascontiguousarray(dk, np.int64)
    n = lv.shape[0]
    home = np.zeros(n, np.int32); runs, busy = np.zeros(n, np.int64), np.zeros(n, np.int64)
    K = C.c_int32(); occ = C.c_int64()
    assert lib().oracle_gslice_direct(n, _p(lv), _p(d), nslots, L, _p(home), C.byref(K), _p(runs), _p(busy),
                                      C.byref(occ)) == 0
    return dict(home=home, nbins=K.value, runs=runs, busy=busy, occ_num=occ.value)


CMP_NAMES = ("dstack", "maxmin", "srf_struck", "temporal", "gslice")


def compare(pb: Problem, p: Params, nthreads: int = 0, subset=None):
    """O9: U, throughput and Jain fairness of the five schedulers per scenario, arrays [num_scen, 5] in the
    order of CMP_NAMES (subset: scenario indices, others left zero)."""
    S = pb.num_scen
    u, thr, jain = (np.zeros((S, 5), np.float64) for _ in range(3))
    idx = None if subset is None else np.ascontiguousarray(np.asarray(list(subset)), np.int64)
    rc = lib().oracle_compare(C.byref(_problem(pb)), C.byref(_params(p)), _p(u), _p(thr), _p(jain), _p(idx),
                              0 if idx is None else idx.shape[0], nthreads)
    assert rc == 0
    return dict(u=u, thr=thr, jain=jain)


MAXTHR_STATES = 8192   # state-space cap shared with the CUDA path (R24)


def maxthr_direct(g, bstar, dtab, b_lo: int, L: int, nslots: int, max_states: int = 1 << 22):
    """O9b max-throughput with direct inputs: the largest number of requests any session schedule serves (runs of
    batch b <= b*_j lasting dtab[j, b-1] slots at level g_j, capacity L); None if the state space exceeds
    max_states."""
    g = np.ascontiguousarray(g, np.int32); bs = np.ascontiguousarray(bstar, np.int32)
    n = g.shape[0]
    dt = np.zeros((n, 64), np.int64)
    dtab = np.asarray(dtab, np.int64)
    if n:
        dt[:, : dtab.shape[1]] = dtab
    best = C.c_int64()
    rc = lib().oracle_maxthr_direct(n, _p(g), _p(bs), _p(dt), b_lo, L, nslots, max_states, C.byref(best))
    return None if rc != 0 else int(best.value)


def maxthr(pb: Problem, p: Params, max_states: int = MAXTHR_STATES, nthreads: int = 0, subset=None):
    """O9b per scenario on the eval path's quantities: dict(served int64, status u8, T_us int64) [scenarios of
    `subset` in order, or all]."""
    idx = None if subset is None else np.ascontiguousarray(np.asarray(list(subset)), np.int64)
    n = pb.num_scen if idx is None else idx.shape[0]
    served = np.zeros(n, np.int64); st = np.zeros(n, np.uint8); T = np.zeros(n, np.int64)
    rc = lib().oracle_maxthr(C.byref(_problem(pb)), C.byref(_params(p)), max_states, _p(served), _p(st), _p(T),
                             _p(idx), 0 if idx is None else n, nthreads)
    assert rc == 0
    return dict(served=served, status=st, T_us=T)


CLUSTER_NAMES = ("exclusive", "temporal", "dstack", "dstack_ffd")


def cluster(pb: Problem, p: Params, G: int, nthreads: int = 0, subset=None):
    """F4: multi-GPU cluster policies of §7.1 over G modelled GPUs; dict u, thr of shape [num_scen, 4]
    (columns CLUSTER_NAMES)."""
    S = pb.num_scen
    u = np.zeros((S, 4), np.float64); thr = np.zeros((S, 4), np.float64)
    idx = None if subset is None else np.ascontiguousarray(np.asarray(list(subset)), np.int64)
    rc = lib().oracle_cluster(C.byref(_problem(pb)), C.byref(_params(p)), G, _p(u), _p(thr), _p(idx),
                              0 if idx is None else idx.shape[0], nthreads)
    assert rc == 0
    return dict(u=u, thr=thr)


def ideal_direct(chains, slo_us, active, L: int, T_us: int, bstar=None):
    """O6 with direct chains: chains[j] = list of (g_e, tau_e). Returns dict(util, completed, events)."""
    n = len(chains)
    off = np.zeros(n + 1, np.int64)
    for j, ch in enumerate(chains):
        off[j + 1] = off[j] + len(ch)
    E = int(off[-1])
    eg = np.zeros(max(E, 1), np.int32); et = np.zeros(max(E, 1), np.int64)
    for j, ch in enumerate(chains):
        for q, (gg, tt) in enumerate(ch):
            eg[off[j] + q] = gg; et[off[j] + q] = tt
    slo = np.ascontiguousarray(slo_us, np.int64)
    bs = np.ascontiguousarray(bstar if bstar is not None else np.ones(n), np.int32)
    act = np.ascontiguousarray(active, np.uint8)
    util = C.c_int64(); ev = C.c_int64()
    comp = np.zeros(n, np.int64)
    rc = lib().oracle_ideal_direct(n, _p(off), _p(eg), _p(et), _p(slo), _p(bs), _p(act), L, T_us, C.byref(util),
                                   _p(comp), C.byref(ev))
    assert rc == 0
    return dict(util=util.value, completed=comp, events=ev.value)


def ideal_rows(pb: Problem, p: Params, dnn: int, b: int):
    K = int(pb.dnn_row_off[dnn + 1] - pb.dnn_row_off[dnn])
    g = np.zeros(K, np.int32); tau = np.zeros(K, np.int64)
    assert lib().oracle_ideal_rows(C.byref(_problem(pb)), C.byref(_params(p)), dnn, b, _p(g), _p(tau)) == 0
    return g, tau


def out_arrays(num_scen: int, num_dnn: int):
    D, S = num_dnn, num_scen
    return dict(demand=np.zeros(D, np.uint16), batch=np.zeros(D, np.uint8), knee=np.zeros(D, np.uint16),
                status=np.zeros(D, np.uint8), alloc_q16=np.zeros(D, np.uint32), level=np.zeros(D, np.uint16),
                runs=np.zeros(D, np.uint16), served=np.zeros(D, np.uint32),
                scen_status=np.zeros(S, np.uint8), T_us=np.zeros(S, np.uint32), u_static=np.zeros(S, np.float64),
                u=np.zeros(S, np.float64), thr=np.zeros(S, np.float64), misses=np.zeros(S, np.uint32),
                u_ideal=np.zeros(S, np.float64), thr_ideal=np.zeros(S, np.float64), below=np.zeros(S, np.uint32))


def evaluate(pb: Problem, p: Params, nthreads: int = 0, subset=None):
    """Whole path a1-a6. subset: optional iterable of scenario indices (others left zero)."""
    o = out_arrays(pb.num_scen, pb.num_dnn)
    oo = OrOut(*[_p(o[k]) for k, _ in OrOut._fields_])
    if subset is None:
        rc = lib().oracle_eval(C.byref(_problem(pb)), C.byref(_params(p)), C.byref(oo), nthreads)
    else:
        idx = np.ascontiguousarray(np.asarray(list(subset)), np.int64)
        rc = lib().oracle_eval_subset(C.byref(_problem(pb)), C.byref(_params(p)), C.byref(oo), _p(idx),
                                      idx.shape[0], nthreads)
    assert rc == 0, rc
    return o


def simulate(pb: Problem, p: Params, cycles: int, seed: int, cfg_tag: int, scen_base: int = 0, subset=None,
             nthreads: int = 0, series: bool = False):
    """O7 long-horizon simulation; per-scenario dict (subset: scenario indices, others left zero).  series: also
    the per-cycle aggregate series, uint64 [cycles, 8] (dstack.h DSTACK_SIM_* order)."""
    S = pb.num_scen
    o = dict(status=np.zeros(S, np.uint8), T_us=np.zeros(S, np.uint32),
             **{k: np.zeros(S, np.uint64) for k in ("arrived", "in_slo", "late", "unserved", "occ_sum", "runs",
                                                     "misses", "realloc")})
    if series:
        o["series"] = np.zeros((max(cycles, 1), 8), np.uint64)
    oo = OrSimOut(*[(_p(o[k]) if k in o else None) for k, _ in OrSimOut._fields_])
    lam = np.ascontiguousarray(pb.lam_pct, np.int32)
    idx = None if subset is None else np.ascontiguousarray(np.asarray(list(subset)), np.int64)
    rc = lib().oracle_simulate(C.byref(_problem(pb)), C.byref(_params(p)), _p(lam), cycles, seed, cfg_tag, scen_base,
                               C.byref(oo), _p(idx), 0 if idx is None else idx.shape[0], nthreads)
    assert rc == 0
    return o
