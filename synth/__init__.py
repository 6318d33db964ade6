"""Seeded synthetic D-STACK workloads (shared by oracle tests and the CUDA path).

This module only DRAWS INPUTS: it holds none of the method's arithmetic.
The generator core is ``synth/synth_core.h`` (integer-only Philox4x32-10),
compiled twice: ``libdstack_synth_host.so`` (gcc, numpy arrays) and
``libdstack_synth_dev.so`` (nvcc sm_100a, torch CUDA tensors).  Both give
byte-identical arrays for the same spec and global scenario index, so a
scenario drawn on the GPU for the bench can be re-drawn on the host for the
oracle.  Workload recipes: SURVEY.md §8(d), restated in DESIGN.md §4.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
HOST_LIB = os.path.join(_HERE, "libdstack_synth_host.so")
DEV_LIB = os.path.join(_HERE, "libdstack_synth_dev.so")

SEED = 0x230413541
SHAPES = ("mobilenet", "resnet50", "vgg19", "bert")


class SynthSpec(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64), ("scen_base", C.c_int64), ("num_scen", C.c_int32), ("cfg_tag", C.c_int32),
        ("S_tot", C.c_int32), ("ndnn_min", C.c_int32), ("ndnn_max", C.c_int32), ("shape_mask", C.c_int32),
        ("paper_mix", C.c_int32), ("slot_us", C.c_int32), ("slo_min_slots", C.c_int32),
        ("slo_max_slots", C.c_int32), ("asm_min_us", C.c_int32), ("asm_max_us", C.c_int32),
        ("bmax", C.c_int32), ("mem_bw", C.c_int32), ("threads", C.c_int32), ("rows_pct", C.c_int32),
        ("heavy", C.c_int32),
    ]


@dataclass
class Spec:
    seed: int = SEED
    scen_base: int = 0
    num_scen: int = 1
    cfg_tag: int = 0
    S_tot: int = 148
    ndnn_min: int = 2
    ndnn_max: int = 8
    shape_mask: int = 0xF
    paper_mix: int = 0
    slot_us: int = 100
    slo_min_slots: int = 250
    slo_max_slots: int = 1000
    asm_min_us: int = 240
    asm_max_us: int = 1920
    bmax: int = 64
    mem_bw: int = 50000
    threads: int = 0
    rows_pct: int = 100
    heavy: int = 0

    def c(self) -> SynthSpec:
        return SynthSpec(**dataclasses.asdict(self))

    def replace(self, **kw) -> "Spec":
        return dataclasses.replace(self, **kw)


@dataclass
class Params:
    """Evaluation parameters (the product's dstack_params_t / the oracle's or_params_t)."""
    L: int = 100
    S_tot: int = 148
    slot_us: int = 100
    mem_mode: int = 1      # 0 off, 1 bw (default), 2 verbatim
    margin: int = 0
    par_mode: int = 0      # 0 linear, 1 threads
    wse_mode: int = 0      # 0 per_request (printed Eq. 4), 1 per_launch
    b_min: int = 1
    b_max: int = 64
    ideal: int = 0
    below_knee: int = 0    # F1 below-knee fallback
    reconf_us: int = 100   # F1 launch latency of a lower-GPU% instance (P:2821 switchover)

    def replace(self, **kw) -> "Params":
        return dataclasses.replace(self, **kw)


@dataclass
class Problem:
    """Structure-of-arrays problem set, CSR-indexed (numpy, host)."""
    scen_dnn_off: np.ndarray   # int32 [S+1]
    dnn_row_off: np.ndarray    # int64 [D+1]
    t_p: np.ndarray            # int32 [D]
    t_np: np.ndarray
    mem_bw: np.ndarray
    slo_us: np.ndarray
    asm_us: np.ndarray
    bmax: np.ndarray
    n: np.ndarray              # uint32 [R] (padded: len >= R + 8)
    r: np.ndarray              # uint16 [R]
    d: np.ndarray              # uint32 [R]
    shape: np.ndarray = field(default=None)  # int32 [D] (reporting only)
    lam_pct: np.ndarray = field(default=None)  # int32 [D] config-5 offered load, % of standalone capacity

    @property
    def num_scen(self) -> int:
        return int(self.scen_dnn_off.shape[0] - 1)

    @property
    def num_dnn(self) -> int:
        return int(self.dnn_row_off.shape[0] - 1)

    @property
    def num_rows(self) -> int:
        return int(self.dnn_row_off[-1])

    def nbytes_rows(self) -> int:
        return self.num_rows * 10

    def scenario(self, s: int) -> "Problem":
        """Problem holding only scenario s (copies)."""
        return self.subset([s])

    def subset(self, scen) -> "Problem":
        scen = [int(s) for s in scen]
        offs = [0]; dnn_rows = [0]
        tp, tnp, mb, slo, asm, bm, shp, ns, rs, ds, lp = ([] for _ in range(11))
        for s in scen:
            k0, k1 = int(self.scen_dnn_off[s]), int(self.scen_dnn_off[s + 1])
            offs.append(offs[-1] + (k1 - k0))
            for k in range(k0, k1):
                r0, r1 = int(self.dnn_row_off[k]), int(self.dnn_row_off[k + 1])
                dnn_rows.append(dnn_rows[-1] + r1 - r0)
                ns.append(self.n[r0:r1]); rs.append(self.r[r0:r1]); ds.append(self.d[r0:r1])
            tp.append(self.t_p[k0:k1]); tnp.append(self.t_np[k0:k1]); mb.append(self.mem_bw[k0:k1])
            slo.append(self.slo_us[k0:k1]); asm.append(self.asm_us[k0:k1]); bm.append(self.bmax[k0:k1])
            if self.shape is not None:
                shp.append(self.shape[k0:k1])
            if self.lam_pct is not None:
                lp.append(self.lam_pct[k0:k1])
        cat = lambda xs, dt: (np.concatenate(xs).astype(dt) if xs else np.zeros(0, dt))
        return make_problem(
            np.asarray(offs, np.int32), np.asarray(dnn_rows, np.int64), cat(tp, np.int32), cat(tnp, np.int32),
            cat(mb, np.int32), cat(slo, np.int32), cat(asm, np.int32), cat(bm, np.int32),
            cat(ns, np.uint32), cat(rs, np.uint16), cat(ds, np.uint32),
            cat(shp, np.int32) if shp else None, cat(lp, np.int32) if lp else None)


def _pad(a: np.ndarray, extra: int = 8) -> np.ndarray:
    out = np.zeros(a.shape[0] + extra, a.dtype)
    out[: a.shape[0]] = a
    return out


def make_problem(scen_dnn_off, dnn_row_off, t_p, t_np, mem_bw, slo_us, asm_us, bmax, n, r, d, shape=None,
                 lam_pct=None) -> Problem:
    """Build a Problem from explicit arrays (hand-written test instances)."""
    R = int(np.asarray(dnn_row_off)[-1])
    n = np.asarray(n, np.uint32)[:R]; r = np.asarray(r, np.uint16)[:R]; d = np.asarray(d, np.uint32)[:R]
    return Problem(
        np.ascontiguousarray(scen_dnn_off, np.int32), np.ascontiguousarray(dnn_row_off, np.int64),
        np.ascontiguousarray(t_p, np.int32), np.ascontiguousarray(t_np, np.int32),
        np.ascontiguousarray(mem_bw, np.int32), np.ascontiguousarray(slo_us, np.int32),
        np.ascontiguousarray(asm_us, np.int32), np.ascontiguousarray(bmax, np.int32),
        _pad(n), _pad(r), _pad(d), None if shape is None else np.ascontiguousarray(shape, np.int32),
        None if lam_pct is None else np.ascontiguousarray(lam_pct, np.int32))


_host = None


def _host_lib():
    global _host
    if _host is None:
        if not os.path.exists(HOST_LIB):
            raise RuntimeError(f"{HOST_LIB} missing: run __graft_entry__.build()")
        lib = C.CDLL(HOST_LIB)
        P = C.POINTER
        lib.synth_host_ndnn.argtypes = [P(SynthSpec), C.c_void_p]
        lib.synth_host_headers.argtypes = [P(SynthSpec)] + [C.c_void_p] * 10
        lib.synth_host_rows.argtypes = [P(SynthSpec)] + [C.c_void_p] * 5
        lib.synth_host_arrival_gaps.argtypes = [C.c_uint64, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_uint32,
                                                C.c_uint32, C.c_void_p]
        _host = lib
    return _host


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def generate_host(spec: Spec) -> Problem:
    lib = _host_lib()
    cs = spec.c()
    S = spec.num_scen
    ndnn = np.zeros(S, np.int32)
    assert lib.synth_host_ndnn(C.byref(cs), _ptr(ndnn)) == 0
    off = np.zeros(S + 1, np.int32)
    np.cumsum(ndnn, out=off[1:])
    D = int(off[-1])
    hdr = [np.zeros(D, np.int32) for _ in range(9)]
    assert lib.synth_host_headers(C.byref(cs), _ptr(off), *[_ptr(h) for h in hdr]) == 0
    nrows, t_p, t_np, mem_bw, slo, asm, bmax, shape, lam = hdr
    roff = np.zeros(D + 1, np.int64)
    np.cumsum(nrows.astype(np.int64), out=roff[1:])
    R = int(roff[-1])
    n = np.zeros(R + 8, np.uint32); r = np.zeros(R + 8, np.uint16); d = np.zeros(R + 8, np.uint32)
    assert lib.synth_host_rows(C.byref(cs), _ptr(off), _ptr(roff), _ptr(n), _ptr(r), _ptr(d)) == 0
    return Problem(off, roff, t_p, t_np, mem_bw, slo, asm, bmax, n, r, d, shape, lam)


_dev = None


def _dev_lib():
    global _dev
    if _dev is None:
        if not os.path.exists(DEV_LIB):
            raise RuntimeError(f"{DEV_LIB} missing: run __graft_entry__.build()")
        lib = C.CDLL(DEV_LIB)
        P = C.POINTER
        lib.synth_dev_ndnn.argtypes = [P(SynthSpec), C.c_void_p, C.c_void_p]
        lib.synth_dev_headers.argtypes = [P(SynthSpec)] + [C.c_void_p] * 11
        lib.synth_dev_rows.argtypes = [P(SynthSpec)] + [C.c_void_p] * 6
        _dev = lib
    return _dev


def generate_device(spec: Spec, device="cuda"):
    """Draw the same problem directly into device memory. Returns a dict of torch tensors
    with the Problem field names (row arrays padded by 8 elements)."""
    import torch
    lib = _dev_lib()
    cs = spec.c()
    dev = torch.device(device)
    stream = torch.cuda.current_stream(dev).cuda_stream
    S = spec.num_scen
    i32 = dict(dtype=torch.int32, device=dev)
    ndnn = torch.zeros(S, **i32)
    assert lib.synth_dev_ndnn(C.byref(cs), C.c_void_p(ndnn.data_ptr()), C.c_void_p(stream)) == 0
    off = torch.zeros(S + 1, **i32)
    off[1:] = torch.cumsum(ndnn, 0, dtype=torch.int32)
    D = int(off[-1].item())
    hdr = [torch.zeros(max(D, 1), **i32) for _ in range(9)]
    assert lib.synth_dev_headers(C.byref(cs), C.c_void_p(off.data_ptr()),
                                 *[C.c_void_p(h.data_ptr()) for h in hdr], C.c_void_p(stream)) == 0
    hdr = [h[:D] for h in hdr]
    nrows, t_p, t_np, mem_bw, slo, asm, bmax, shape, lam = hdr
    roff = torch.zeros(D + 1, dtype=torch.int64, device=dev)
    roff[1:] = torch.cumsum(nrows.to(torch.int64), 0)
    R = int(roff[-1].item())
    # row arrays: +8 elements of slack so 16-byte vector / bulk loads never run off the end
    n = torch.zeros(R + 8, dtype=torch.int32, device=dev)     # reinterpreted as u32
    r = torch.zeros(R + 8, dtype=torch.int16, device=dev)     # reinterpreted as u16
    d = torch.zeros(R + 8, dtype=torch.int32, device=dev)     # reinterpreted as u32
    assert lib.synth_dev_rows(C.byref(cs), C.c_void_p(off.data_ptr()), C.c_void_p(roff.data_ptr()),
                              C.c_void_p(n.data_ptr()), C.c_void_p(r.data_ptr()), C.c_void_p(d.data_ptr()),
                              C.c_void_p(stream)) == 0
    return dict(scen_dnn_off=off, dnn_row_off=roff, t_p=t_p, t_np=t_np, mem_bw=mem_bw, slo_us=slo,
                asm_us=asm, bmax=bmax, n=n, r=r, d=d, shape=shape, lam_pct=lam)


# ---------------------------------------------------------------- configs ---
# BASELINE.json "configs" (SURVEY §8(d) per-config table).

def config(k: int, num_scen: int | None = None, rows_pct: int = 100, scen_base: int = 0, variant: str = "default"):
    """Return (Spec, Params) for BASELINE config k (1..5)."""
    if k == 1:
        # one scenario = the paper's C-4 mix: ResNet-50, VGG-19, BERT, MobileNet; S_tot 80
        # (V100), L = 100, a = 481 us, batches 1..64, Delta = 100 us, ideal on.
        sp = Spec(num_scen=num_scen or 1, cfg_tag=1, S_tot=80, paper_mix=1, rows_pct=rows_pct, scen_base=scen_base)
        pr = Params(L=100, S_tot=80, ideal=1)
    elif k == 2:
        sp = Spec(num_scen=num_scen or 10_000, cfg_tag=2, S_tot=148, ndnn_min=2, ndnn_max=8,
                  rows_pct=rows_pct, scen_base=scen_base)
        pr = Params(L=100, S_tot=148, ideal=1)
    elif k == 3:
        sp = Spec(num_scen=num_scen or 1_000_000, cfg_tag=3, S_tot=148, ndnn_min=4, ndnn_max=16,
                  rows_pct=rows_pct, scen_base=scen_base)
        pr = Params(L=148, S_tot=148, ideal=0)
    elif k == 4:
        sp = Spec(num_scen=num_scen or 100_000, cfg_tag=4, S_tot=148, ndnn_min=8, ndnn_max=16, heavy=1,
                  rows_pct=rows_pct, scen_base=scen_base)
        pr = Params(L=100, S_tot=148, ideal=1)
    elif k == 5:
        sp = Spec(num_scen=num_scen or 100_000, cfg_tag=5, S_tot=148, ndnn_min=4, ndnn_max=16,
                  rows_pct=rows_pct, scen_base=scen_base)
        pr = Params(L=148, S_tot=148, ideal=0)
    else:
        raise ValueError(k)
    if variant == "batching":  # labelled batching-aware variant: threads + per_launch
        sp = sp.replace(threads=1)
        pr = pr.replace(par_mode=1, wse_mode=1)
    return sp, pr


def concat(problems) -> Problem:
    """Concatenate problems scenario-wise (e.g. a stratified sample drawn one scenario at a time)."""
    problems = list(problems)
    offs, roffs = [np.zeros(1, np.int32)], [np.zeros(1, np.int64)]
    d0, r0 = 0, 0
    cols = {k: [] for k in ("t_p", "t_np", "mem_bw", "slo_us", "asm_us", "bmax", "shape", "lam_pct")}
    rows = {k: [] for k in ("n", "r", "d")}
    for pb in problems:
        offs.append(pb.scen_dnn_off[1:] + d0)
        roffs.append(pb.dnn_row_off[1:] + r0)
        for k in cols:
            v = getattr(pb, k)
            cols[k].append(v if v is not None else np.zeros(pb.num_dnn, np.int32))
        R = pb.num_rows
        for k in rows:
            rows[k].append(getattr(pb, k)[:R])
        d0 += pb.num_dnn
        r0 += R
    return make_problem(np.concatenate(offs), np.concatenate(roffs), *[np.concatenate(cols[k]) for k in
                        ("t_p", "t_np", "mem_bw", "slo_us", "asm_us", "bmax")],
                        *[np.concatenate(rows[k]) for k in ("n", "r", "d")], np.concatenate(cols["shape"]),
                        np.concatenate(cols["lam_pct"]))


def sample(spec: Spec, indices) -> Problem:
    """Scenarios at the given local indices of `spec`, drawn one by one on the host (stratified samples
    of device-generated workloads: same bytes as the device draw)."""
    return concat(generate_host(spec.replace(scen_base=spec.scen_base + int(i), num_scen=1)) for i in indices)


def arrival_gaps(seed: int, cfg_tag: int, gscen: int, dnn: int, mean_q32: int, k0: int, count: int) -> np.ndarray:
    """Gaps (us) of arrivals k0.. of one Poisson stream (config 5), from the shared integer sampler."""
    out = np.zeros(count, np.uint64)
    assert _host_lib().synth_host_arrival_gaps(seed, cfg_tag, gscen, dnn, mean_q32, k0, count, _ptr(out)) == 0
    return out
