"""Workload selection for BASELINE config 4 ("oversubscribed mixes (sum of knees 2-5x maxGPU%)").

The generator (synth_core.h) draws every scenario from its global index and holds none of the method's
arithmetic.  Config 4 keeps only the scenarios whose summed demand lies in [2, 5] x L; the demands come from
the CALLER's a3 (the product's dstack_batch_opt on the device), so the selection is harness logic applied to the
product's outputs, and the oracle re-checks the ratio on every sampled scenario (tests/test_gpu_fullsize.py).
Selection is deterministic: the first `need` qualifying global indices in ascending order.
"""
from __future__ import annotations

import numpy as np

from . import Spec, generate_device

RATIO_BINS = (0.0, 1.0, 2.0, 3.0, 4.0, 5.0, 6.0, 8.0, 1e9)


def _gather(g: dict, sel, device):
    """Device problem dict holding only the scenarios `sel` (int64 tensor of local indices) of `g`."""
    import torch
    off = g["scen_dnn_off"].to(torch.int64)
    roff = g["dnn_row_off"]
    nd = off[sel + 1] - off[sel]
    new_off = torch.zeros(sel.numel() + 1, dtype=torch.int64, device=device)
    new_off[1:] = torch.cumsum(nd, 0)
    D = int(new_off[-1].item())
    rep = torch.repeat_interleave(torch.arange(sel.numel(), device=device), nd)
    dnn = off[sel][rep] + (torch.arange(D, device=device) - new_off[:-1][rep])
    nr = roff[dnn + 1] - roff[dnn]
    new_roff = torch.zeros(D + 1, dtype=torch.int64, device=device)
    new_roff[1:] = torch.cumsum(nr, 0)
    R = int(new_roff[-1].item())
    rrep = torch.repeat_interleave(torch.arange(D, device=device), nr)
    rows = roff[dnn][rrep] + (torch.arange(R, device=device) - new_roff[:-1][rrep])
    out = {"scen_dnn_off": new_off.to(torch.int32), "dnn_row_off": new_roff}
    for k in ("t_p", "t_np", "mem_bw", "slo_us", "asm_us", "bmax", "shape", "lam_pct"):
        out[k] = g[k][dnn]
    for k in ("n", "r", "d"):
        v = torch.zeros(R + 8, dtype=g[k].dtype, device=device)
        v[:R] = g[k][rows]
        out[k] = v
    return out


def _concat(parts: list, device):
    import torch
    if len(parts) == 1:
        return parts[0]
    offs, roffs = [torch.zeros(1, dtype=torch.int64, device=device)], [torch.zeros(1, dtype=torch.int64, device=device)]
    d0 = r0 = 0
    for q in parts:
        offs.append(q["scen_dnn_off"][1:].to(torch.int64) + d0)
        roffs.append(q["dnn_row_off"][1:] + r0)
        d0 += int(q["dnn_row_off"].numel() - 1)
        r0 += int(q["dnn_row_off"][-1].item())
    out = {"scen_dnn_off": torch.cat(offs).to(torch.int32), "dnn_row_off": torch.cat(roffs)}
    for k in ("t_p", "t_np", "mem_bw", "slo_us", "asm_us", "bmax", "shape", "lam_pct"):
        out[k] = torch.cat([q[k] for q in parts])
    for k in ("n", "r", "d"):
        R = [int(q["dnn_row_off"][-1].item()) for q in parts]
        v = torch.zeros(sum(R) + 8, dtype=parts[0][k].dtype, device=device)
        v[: sum(R)] = torch.cat([q[k][:n] for q, n in zip(parts, R)])
        out[k] = v
    return out


def select_by_demand_ratio(spec: Spec, L: int, a3, need: int, lo: float = 2.0, hi: float = 5.0,
                           chunk: int = 200_000, device="cuda", max_pool: int = 50_000_000, gather_range=None):
    """Scan spec's scenario stream (global indices spec.scen_base, +1, ...) in chunks; a3(device_dict) -> demand
    (u16 per DNN, the caller's product a3) decides which scenarios have sum(demand) / L in [lo, hi].
    Returns (global_indices int64 numpy [need], device dict of the selected scenarios gather_range = [b, e) of the
    selection (default all), stats).  Raises if the pool runs out."""
    import torch
    sel_glob, parts, hist_pool = [], [], np.zeros(len(RATIO_BINS) - 1, np.int64)
    b, e = gather_range if gather_range is not None else (0, need)
    base, found, scanned = spec.scen_base, 0, 0
    while found < need:
        if scanned >= max_pool:
            raise RuntimeError(f"config-4 selection: only {found} of {need} in {scanned} scenarios")
        g = generate_device(spec.replace(scen_base=base, num_scen=chunk), device)
        dem = a3(g).to(torch.int64)
        off = g["scen_dnn_off"].to(torch.int64)
        cs = torch.zeros(dem.numel() + 1, dtype=torch.int64, device=device)
        cs[1:] = torch.cumsum(dem, 0)
        tot = cs[off[1:]] - cs[off[:-1]]
        ratio = tot.to(torch.float64) / float(L)
        hist_pool += np.histogram(ratio.cpu().numpy(), bins=RATIO_BINS)[0]
        ok = torch.nonzero((ratio >= lo) & (ratio <= hi)).flatten()
        take = ok[: need - found]
        # the part of this chunk's selection that falls in [b, e) of the whole selection
        lo_i, hi_i = max(b - found, 0), min(e - found, take.numel())
        if hi_i > lo_i:
            parts.append(_gather(g, take[lo_i:hi_i], device))
        sel_glob.append(take.cpu().numpy() + base)
        found += take.numel()
        scanned += chunk
        base += chunk
        del g, dem
    glob = np.concatenate(sel_glob)[:need]
    dd = _concat(parts, device) if parts else None
    stats = {"pool_scanned": scanned, "selected": need, "ratio_bins": list(RATIO_BINS[:-1]) + ["inf"],
             "ratio_hist_pool": hist_pool.tolist(), "selected_frac_of_pool": need / scanned,
             "rule": f"sum(demand)/L in [{lo}, {hi}] (demand = the product's a3), first {need} global indices"}
    return glob, dd, stats
