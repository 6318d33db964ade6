"""Thin ctypes binding of libdstack (include/dstack.h): argument marshalling only.

Every step of the path runs in the sm_100a kernels of ``libdstack.so``; this module allocates
device tensors with torch (plumbing: memory, streams) and passes raw pointers.  There is no CPU
fallback: if the shared library is missing the import fails, and without a CUDA device every
compute call raises ``DstackError`` (the library returns DSTACK_ELAUNCH).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DSTACK_LIB") or os.path.join(_HERE, "libdstack.so")   # DSTACK_LIB: A/B builds

DSTACK_OK, DSTACK_EINVAL, DSTACK_EWORKSPACE, DSTACK_ELAUNCH = 0, -1, -2, -3
ST_OK, ST_INFEASIBLE, ST_OVERFLOW, ST_INVALID, ST_OVERSUBSCRIBED = 0, 1, 2, 3, 4
FLAG_IDEAL = 1
FLAG_BELOW_KNEE = 2
MAX_BATCH = 64


class DstackError(RuntimeError):
    pass


class CProblem(C.Structure):
    _fields_ = [("num_scen", C.c_int32), ("num_dnn", C.c_int32), ("num_rows", C.c_int64),
                ("scen_dnn_off", C.c_void_p), ("dnn_row_off", C.c_void_p), ("t_p", C.c_void_p),
                ("t_np", C.c_void_p), ("mem_bw", C.c_void_p), ("slo_us", C.c_void_p), ("asm_us", C.c_void_p),
                ("bmax", C.c_void_p), ("n", C.c_void_p), ("r", C.c_void_p), ("d", C.c_void_p)]


class CParams(C.Structure):
    _fields_ = [("L", C.c_int32), ("S_tot", C.c_int32), ("slot_us", C.c_int32), ("mem_mode", C.c_int32),
                ("margin", C.c_int32), ("par_mode", C.c_int32), ("wse_mode", C.c_int32), ("b_min", C.c_int32),
                ("b_max", C.c_int32), ("flags", C.c_uint32), ("reconf_us", C.c_int32)]


class CAgg(C.Structure):
    _fields_ = ([(k, C.c_double) for k in ("sum_u_static", "sum_u", "sum_thr", "sum_u_ideal", "sum_thr_ideal")] +
                [(k, C.c_uint64) for k in ("n_scen", "n_scen_scheduled", "n_dnn", "n_dnn_ok")] +
                [("n_st", C.c_uint64 * 5), ("n_scen_st", C.c_uint64 * 5)] +
                [(k, C.c_uint64) for k in ("misses", "runs", "served")] +
                [("batch_hist", C.c_uint64 * (MAX_BATCH + 1)), ("demand_hist", C.c_uint64 * 256),
                 ("checksum", C.c_uint64)])


AGG_WORDS = C.sizeof(CAgg) // 8

_OUT_FIELDS = ("demand", "batch", "knee", "status", "alloc_q16", "level", "runs", "served",
               "scen_status", "T_us", "u_static", "u", "thr", "misses", "u_ideal", "thr_ideal", "agg", "below")


class COut(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in _OUT_FIELDS]


_SIM_FIELDS = ("status", "T_us", "arrived", "in_slo", "late", "unserved", "occ_sum", "runs", "misses", "realloc")


SIM_SERIES = ("active", "realloc", "runs", "served", "in_slo", "late", "occ", "misses")   # DSTACK_SIM_* columns


class CSimOut(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in _SIM_FIELDS] + [("series", C.c_void_p)]


class CHook(C.Structure):
    _fields_ = [("level", C.c_void_p), ("d_slots", C.c_void_p)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() (no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH)
    P = C.POINTER
    lib.dstack_workspace_size.argtypes = [P(CProblem), P(CParams)]
    lib.dstack_workspace_size.restype = C.c_size_t
    lib.dstack_knee.argtypes = [P(CProblem), P(CParams), C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_size_t, C.c_void_p]
    lib.dstack_knee_probe.argtypes = [P(CProblem), P(CParams), C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_size_t, C.c_void_p]
    lib.dstack_batch_opt.argtypes = [P(CProblem), P(CParams)] + [C.c_void_p] * 5 + [C.c_size_t, C.c_void_p]
    lib.dstack_wmaxmin.argtypes = [C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.dstack_schedule_cycle.argtypes = [P(CProblem), P(CParams), C.c_void_p, C.c_void_p, C.c_void_p, P(CHook),
                                          P(COut), C.c_void_p, C.c_size_t, C.c_void_p]
    lib.dstack_eval_batch.argtypes = [P(CProblem), P(CParams), P(COut), C.c_void_p, C.c_size_t, C.c_void_p]
    lib.dstack_aggregate.argtypes = [P(CProblem), P(CParams), P(COut), C.c_void_p, C.c_size_t, C.c_void_p]
    lib.dstack_sim_workspace_size.argtypes = [P(CProblem), P(CParams)]
    lib.dstack_sim_workspace_size.restype = C.c_size_t
    lib.dstack_simulate.argtypes = [P(CProblem), P(CParams), C.c_void_p, C.c_int32, C.c_uint64, C.c_int32, C.c_int64,
                                    P(CSimOut), C.c_void_p, C.c_size_t, C.c_void_p]
    lib.dstack_compare.argtypes = [P(CProblem), P(CParams)] + [C.c_void_p] * 7 + [C.c_size_t, C.c_void_p]
    lib.dstack_cluster.argtypes = [P(CProblem), P(CParams), C.c_int32] + [C.c_void_p] * 5 + [C.c_size_t, C.c_void_p]
    lib.dstack_unpack_nr.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.dstack_unpack_w5.argtypes = [C.c_int64] + [C.c_void_p] * 6
    lib.dstack_max_throughput.argtypes = [P(CProblem), P(CParams)] + [C.c_void_p] * 6 + [C.c_size_t, C.c_void_p]
    lib.dstack_ideal_stats.argtypes = [P(CProblem), P(CParams), C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]
    lib.dstack_profile_start.argtypes = [C.c_int32]
    lib.dstack_profile_stop.argtypes = [C.c_void_p, C.c_void_p]
    lib.dstack_status_str.restype = C.c_char_p
    lib.dstack_last_launch_count.restype = C.c_int
    return lib


_lib = _load()

# every symbol include/dstack.h declares (checked by tests/test_abi.py)
EXPORTS = ("dstack_workspace_size", "dstack_knee", "dstack_knee_probe", "dstack_batch_opt", "dstack_wmaxmin", "dstack_schedule_cycle",
           "dstack_eval_batch", "dstack_aggregate", "dstack_sim_workspace_size", "dstack_simulate",
           "dstack_compare", "dstack_cluster", "dstack_max_throughput", "dstack_unpack_nr", "dstack_unpack_w5", "dstack_profile_start", "dstack_profile_stop",
           "dstack_last_launch_count", "dstack_ideal_stats", "dstack_status_str", "dstack_version")


def lib():
    return _lib


def _check(rc: int, what: str):
    if rc != DSTACK_OK:
        raise DstackError(f"{what}: {_lib.dstack_status_str(rc).decode()} ({rc})")


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(device):
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


@dataclass
class DeviceProblem:
    """The SoA problem set resident in device memory (torch tensors used as plain buffers)."""
    num_scen: int
    num_dnn: int
    num_rows: int
    scen_dnn_off: torch.Tensor   # int32
    dnn_row_off: torch.Tensor    # int64
    t_p: torch.Tensor
    t_np: torch.Tensor
    mem_bw: torch.Tensor
    slo_us: torch.Tensor
    asm_us: torch.Tensor
    bmax: torch.Tensor
    n: torch.Tensor              # int32 storage of u32 (+ >= 16 B slack)
    r: torch.Tensor              # int16 storage of u16
    d: torch.Tensor              # int32 storage of u32
    lam_pct: torch.Tensor | None = None   # int32 [num_dnn], config-5 offered load (dstack_simulate only)

    @property
    def device(self):
        return self.n.device

    def c(self) -> CProblem:
        return CProblem(self.num_scen, self.num_dnn, self.num_rows, self.scen_dnn_off.data_ptr(),
                        self.dnn_row_off.data_ptr(), self.t_p.data_ptr(), self.t_np.data_ptr(),
                        self.mem_bw.data_ptr(), self.slo_us.data_ptr(), self.asm_us.data_ptr(),
                        self.bmax.data_ptr(), self.n.data_ptr(), self.r.data_ptr(), self.d.data_ptr())

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in (self.scen_dnn_off, self.dnn_row_off, self.t_p, self.t_np,
                                                         self.mem_bw, self.slo_us, self.asm_us, self.bmax, self.n,
                                                         self.r, self.d))


def from_host(pb, device="cuda", pin=False) -> DeviceProblem:
    """Copy a host problem (numpy arrays with the synth.Problem field names) to the device."""
    dev = torch.device(device)

    def t(a, dt):
        x = torch.from_numpy(np.ascontiguousarray(a).view(dt))
        if pin:
            x = x.pin_memory()
        return x.to(dev, non_blocking=pin)
    R = int(pb.dnn_row_off[-1])
    pad = lambda a: a if a.shape[0] >= R + 8 else np.concatenate([a, np.zeros(R + 8 - a.shape[0], a.dtype)])
    return DeviceProblem(int(pb.scen_dnn_off.shape[0] - 1), int(pb.dnn_row_off.shape[0] - 1), R,
                         t(pb.scen_dnn_off, np.int32), t(pb.dnn_row_off, np.int64), t(pb.t_p, np.int32),
                         t(pb.t_np, np.int32), t(pb.mem_bw, np.int32), t(pb.slo_us, np.int32), t(pb.asm_us, np.int32),
                         t(pb.bmax, np.int32), t(pad(pb.n), np.int32), t(pad(pb.r), np.int16), t(pad(pb.d), np.int32),
                         None if getattr(pb, "lam_pct", None) is None else t(pb.lam_pct, np.int32))


def from_device_dict(g: dict) -> DeviceProblem:
    """Wrap the dict returned by synth.generate_device()."""
    S = g["scen_dnn_off"].numel() - 1
    D = g["dnn_row_off"].numel() - 1
    R = int(g["dnn_row_off"][-1].item())
    return DeviceProblem(S, D, R, g["scen_dnn_off"], g["dnn_row_off"], g["t_p"], g["t_np"], g["mem_bw"],
                         g["slo_us"], g["asm_us"], g["bmax"], g["n"], g["r"], g["d"], g.get("lam_pct"))


def cparams(p) -> CParams:
    flags = (FLAG_IDEAL if getattr(p, "ideal", 0) else 0) | (FLAG_BELOW_KNEE if getattr(p, "below_knee", 0) else 0)
    return CParams(p.L, p.S_tot, p.slot_us, p.mem_mode, p.margin, p.par_mode, p.wse_mode, p.b_min, p.b_max, flags,
                   getattr(p, "reconf_us", 100))


def workspace_size(dp: DeviceProblem, p) -> int:
    return int(_lib.dstack_workspace_size(C.byref(dp.c()), C.byref(cparams(p))))


class Workspace:
    """Caller-owned scratch (no call allocates device memory)."""

    def __init__(self, nbytes: int, device):
        self.buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        self.nbytes = int(nbytes)

    def ptr(self):
        return C.c_void_p(self.buf.data_ptr()) if self.nbytes > 0 else None


def knee(dp: DeviceProblem, p, batch: int):
    """dstack_knee: (knee[num_dnn] int16-storage u16, status[num_dnn] u8) device tensors."""
    dev = dp.device
    k = torch.zeros(max(dp.num_dnn, 1), dtype=torch.int16, device=dev)
    st = torch.zeros(max(dp.num_dnn, 1), dtype=torch.uint8, device=dev)
    _check(_lib.dstack_knee(C.byref(dp.c()), C.byref(cparams(p)), batch, _ptr(k), _ptr(st), None, 0,
                            _stream(dev)), "dstack_knee")
    return k[: dp.num_dnn], st[: dp.num_dnn]


def knee_probe(dp: DeviceProblem, p, batch: int):
    """dstack_knee_probe (F3, online knee discovery): (knee u16-in-int16, probes u8, status u8) device tensors."""
    dev = dp.device
    k = torch.zeros(max(dp.num_dnn, 1), dtype=torch.int16, device=dev)
    pr = torch.zeros(max(dp.num_dnn, 1), dtype=torch.uint8, device=dev)
    st = torch.zeros(max(dp.num_dnn, 1), dtype=torch.uint8, device=dev)
    ws = Workspace(workspace_size(dp, p), dev)
    _check(_lib.dstack_knee_probe(C.byref(dp.c()), C.byref(cparams(p)), batch, _ptr(k), _ptr(pr), _ptr(st), ws.ptr(),
                                  ws.nbytes, _stream(dev)), "dstack_knee_probe")
    return k[: dp.num_dnn], pr[: dp.num_dnn], st[: dp.num_dnn]


def batch_opt(dp: DeviceProblem, p, out=None):
    """dstack_batch_opt into out (dict with demand/batch/knee/status tensors) or fresh tensors."""
    dev = dp.device
    o = out if out is not None else alloc_outputs(dp, agg=False)
    _check(_lib.dstack_batch_opt(C.byref(dp.c()), C.byref(cparams(p)), _ptr(o["demand"]), _ptr(o["batch"]),
                                 _ptr(o["knee"]), _ptr(o["status"]), None, 0, _stream(dev)), "dstack_batch_opt")
    if out is not None:
        return o
    return {k: o[k][: dp.num_dnn] for k in ("demand", "batch", "knee", "status")}


def wmaxmin(scen_dnn_off: torch.Tensor, L: int, demand: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    dev = demand.device
    a = out if out is not None else torch.zeros(max(demand.numel(), 1), dtype=torch.int32, device=dev)
    _check(_lib.dstack_wmaxmin(scen_dnn_off.numel() - 1, _ptr(scen_dnn_off), L, _ptr(demand), _ptr(a), _stream(dev)),
           "dstack_wmaxmin")
    return a if out is not None else a[: demand.numel()]


def aggregate(dp: DeviceProblem, p, out: dict, ws: "Workspace"):
    _check(_lib.dstack_aggregate(C.byref(dp.c()), C.byref(cparams(p)), C.byref(_cout(out)), ws.ptr(), ws.nbytes,
                                 _stream(dp.device)), "dstack_aggregate")
    return out["agg"]


def alloc_outputs(dp: DeviceProblem, agg=True):
    dev = dp.device
    D, S = max(dp.num_dnn, 1), max(dp.num_scen, 1)
    z = lambda n, dt: torch.zeros(n, dtype=dt, device=dev)
    o = dict(demand=z(D, torch.int16), batch=z(D, torch.uint8), knee=z(D, torch.int16), status=z(D, torch.uint8),
             alloc_q16=z(D, torch.int32), level=z(D, torch.int16), runs=z(D, torch.int16), served=z(D, torch.int32),
             scen_status=z(S, torch.uint8), T_us=z(S, torch.int32), u_static=z(S, torch.float64),
             u=z(S, torch.float64), thr=z(S, torch.float64), misses=z(S, torch.int32), u_ideal=z(S, torch.float64),
             thr_ideal=z(S, torch.float64), below=z(S, torch.int32))
    if agg:
        o["agg"] = z(AGG_WORDS, torch.int64)
    return o


def _cout(o: dict) -> COut:
    return COut(*[(o[k].data_ptr() if o.get(k) is not None else None) for k in _OUT_FIELDS])


def schedule_cycle(dp: DeviceProblem, p, demand, batch, alloc_q16, hook=None, out=None, ws: Workspace | None = None):
    dev = dp.device
    o = out if out is not None else alloc_outputs(dp, agg=False)
    if ws is None:
        ws = Workspace(workspace_size(dp, p), dev)
    h = None
    if hook is not None:
        h = C.byref(CHook(hook["level"].data_ptr(), hook["d_slots"].data_ptr()))
    _check(_lib.dstack_schedule_cycle(C.byref(dp.c()), C.byref(cparams(p)), _ptr(demand), _ptr(batch),
                                      _ptr(alloc_q16), h, C.byref(_cout(o)), ws.ptr(), ws.nbytes, _stream(dev)),
           "dstack_schedule_cycle")
    return o


def eval_batch(dp: DeviceProblem, p, out=None, ws: Workspace | None = None, agg=True):
    """dstack_eval_batch: the whole path a1-a6 + a8 on the current stream. Returns the output dict."""
    dev = dp.device
    o = out if out is not None else alloc_outputs(dp, agg=agg)
    if ws is None:
        ws = Workspace(workspace_size(dp, p), dev)
    _check(_lib.dstack_eval_batch(C.byref(dp.c()), C.byref(cparams(p)), C.byref(_cout(o)), ws.ptr(), ws.nbytes,
                                  _stream(dev)), "dstack_eval_batch")
    return o


CMP_NAMES = ("dstack", "maxmin", "srf_struck", "temporal", "gslice")   # DSTACK_CMP_* order
CLU_NAMES = ("exclusive", "temporal", "dstack", "dstack_ffd")         # DSTACK_CLU_* order


def pack_nr(n, r):
    """Host side of the compact row transport: nr = n | R << 12 (u16 torch tensor), or None when some row does not
    fit (n >= 4096 or R outside 1..15) and the rows must travel wide.  n, r: int32 / int16 storage of the ABI's
    u32 / u16 rows (CPU tensors)."""
    nn = n.to(torch.int64) & 0xFFFFFFFF
    rr = r.to(torch.int64) & 0xFFFF
    if nn.numel() and (int(nn.max()) >= 4096 or int(rr.min()) < 1 or int(rr.max()) > 15):
        return None
    return (nn | (rr << 12)).to(torch.int32).to(torch.int16)


def unpack_nr(nr, n_out, r_out, num_rows: int):
    """dstack_unpack_nr: expand the compact rows on the device into the problem's n / r arrays."""
    _check(_lib.dstack_unpack_nr(num_rows, _ptr(nr), _ptr(n_out), _ptr(r_out), _stream(nr.device)), "dstack_unpack_nr")


def unpack_w5(w, lo, n_out, r_out, d_out, num_rows: int):
    """dstack_unpack_w5: expand 5-byte rows (w = d | (R - 1) << 26 | (n >> 8) << 28, lo = n & 255) on the device."""
    _check(_lib.dstack_unpack_w5(num_rows, _ptr(w), _ptr(lo), _ptr(n_out), _ptr(r_out), _ptr(d_out), _stream(w.device)),
           "dstack_unpack_w5")


def cluster(dp: DeviceProblem, p, gpus: int, demand, batch, out=None, ws: Workspace | None = None):
    """dstack_cluster (F4): U and throughput of the CLU_NAMES policies on `gpus` modelled GPUs, f64 tensors
    [num_scen, 4], from the a3 outputs (demand, batch)."""
    dev = dp.device
    if out is None:
        out = {k: torch.zeros((max(dp.num_scen, 1), len(CLU_NAMES)), dtype=torch.float64, device=dev)
               for k in ("u", "thr")}
    if ws is None:
        ws = Workspace(workspace_size(dp, p), dev)
    _check(_lib.dstack_cluster(C.byref(dp.c()), C.byref(cparams(p)), gpus, _ptr(demand), _ptr(batch), _ptr(out["u"]),
                               _ptr(out["thr"]), ws.ptr(), ws.nbytes, _stream(dev)), "dstack_cluster")
    return {k: v[: dp.num_scen] for k, v in out.items()}


def compare(dp: DeviceProblem, p, demand, batch, alloc_q16, out=None, ws: Workspace | None = None):
    """dstack_compare (O9): U, throughput and Jain fairness of the five schedulers of CMP_NAMES per scenario,
    f64 tensors [num_scen, 5], from the a3/a4 outputs (e.g. eval_batch's demand, batch, alloc_q16)."""
    dev = dp.device
    if out is None:
        out = {k: torch.zeros((dp.num_scen, len(CMP_NAMES)), dtype=torch.float64, device=dev)
               for k in ("u", "thr", "jain")}
    if ws is None:
        ws = Workspace(workspace_size(dp, p), dev)
    _check(_lib.dstack_compare(C.byref(dp.c()), C.byref(cparams(p)), _ptr(demand), _ptr(batch), _ptr(alloc_q16),
                               _ptr(out["u"]), _ptr(out["thr"]), _ptr(out["jain"]), ws.ptr(), ws.nbytes,
                               _stream(dev)), "dstack_compare")
    return out


def max_throughput(dp: DeviceProblem, p, demand, batch, alloc_q16, ws: "Workspace | None" = None):
    """dstack_max_throughput (O9b): (served u32-in-int32 [num_scen], status u8 [num_scen]) device tensors."""
    dev = dp.device
    S = max(dp.num_scen, 1)
    served = torch.zeros(S, dtype=torch.int32, device=dev)
    st = torch.zeros(S, dtype=torch.uint8, device=dev)
    if ws is None:
        ws = Workspace(workspace_size(dp, p), dev)
    _check(_lib.dstack_max_throughput(C.byref(dp.c()), C.byref(cparams(p)), _ptr(demand), _ptr(batch), _ptr(alloc_q16),
                                      _ptr(served), _ptr(st), ws.ptr(), ws.nbytes, _stream(dev)),
           "dstack_max_throughput")
    return served[: dp.num_scen], st[: dp.num_scen]


PROF_SLOTS = ("k_prof", "k_wmaxmin", "k_cycle", "k_ideal", "k_agg")


def profile_start(max_calls: int):
    """Record CUDA events between the kernels of the next eval_batch calls on this thread."""
    _check(_lib.dstack_profile_start(max_calls), "dstack_profile_start")


def profile_stop() -> tuple[dict, int]:
    """Synchronise the recorded events: (summed ms per kernel slot, number of profiled calls)."""
    ms = (C.c_double * len(PROF_SLOTS))()
    calls = C.c_int32()
    _check(_lib.dstack_profile_stop(ms, C.byref(calls)), "dstack_profile_stop")
    return {k: ms[i] for i, k in enumerate(PROF_SLOTS)}, calls.value


def simulate(dp: DeviceProblem, p, cycles: int, seed: int, cfg_tag: int, scen_base: int = 0, series: bool = False):
    """dstack_simulate (a7, config 5): per-scenario counters as device tensors (uint64 stored as int64); series:
    also the per-cycle aggregate series [cycles, 8] (columns SIM_SERIES)."""
    dev = dp.device
    S = max(dp.num_scen, 1)
    o = dict(status=torch.zeros(S, dtype=torch.uint8, device=dev), T_us=torch.zeros(S, dtype=torch.int32, device=dev),
             **{k: torch.zeros(S, dtype=torch.int64, device=dev) for k in _SIM_FIELDS[2:]})
    ser = torch.zeros((max(cycles, 1), len(SIM_SERIES)), dtype=torch.int64, device=dev) if series else None
    wsz = int(_lib.dstack_sim_workspace_size(C.byref(dp.c()), C.byref(cparams(p))))
    ws = Workspace(wsz, dev)
    cout = CSimOut(*[o[k].data_ptr() for k in _SIM_FIELDS], ser.data_ptr() if ser is not None else None)
    _check(_lib.dstack_simulate(C.byref(dp.c()), C.byref(cparams(p)), _ptr(dp.lam_pct), cycles, seed, cfg_tag,
                                scen_base, C.byref(cout), ws.ptr(), ws.nbytes, _stream(dev)), "dstack_simulate")
    r = {k: v[: dp.num_scen] for k, v in o.items()}
    if ser is not None:
        r["series"] = ser[:cycles]
    return r


IDEAL_STATS = ("events", "reselections", "sel_all_fit", "sel_enumeration", "sel_meet_in_middle", "sel_dp", "scenarios")


def ideal_stats(dp: DeviceProblem, p, ws: "Workspace") -> dict:
    """dstack_ideal_stats: a6 work counters of the last IDEAL call that used `ws`."""
    out = (C.c_uint64 * 8)()
    _check(_lib.dstack_ideal_stats(C.byref(dp.c()), C.byref(cparams(p)), ws.ptr(), ws.nbytes, out,
                                   _stream(dp.device)), "dstack_ideal_stats")
    return {k: int(out[i]) for i, k in enumerate(IDEAL_STATS)}


def last_launch_count() -> int:
    return int(_lib.dstack_last_launch_count())


def agg_to_dict(agg_tensor: torch.Tensor) -> dict:
    raw = agg_tensor.detach().cpu().numpy().tobytes()
    a = CAgg.from_buffer_copy(raw)
    out = {}
    for k, t in CAgg._fields_:
        v = getattr(a, k)
        out[k] = list(v) if hasattr(v, "__len__") else v
    return out


_U = {torch.int16: np.uint16, torch.int32: np.uint32}


def to_numpy(o: dict, num_scen: int, num_dnn: int) -> dict:
    """Host copies with the ABI's unsigned dtypes (oracle-comparable)."""
    per_dnn = ("demand", "batch", "knee", "status", "alloc_q16", "level", "runs", "served")
    res = {}
    for k, v in o.items():
        if k == "agg":
            continue
        n = num_dnn if k in per_dnn else num_scen
        a = v[:n].cpu().numpy()
        if v.dtype in _U:
            a = a.view(_U[v.dtype])
        res[k] = a
    return res
