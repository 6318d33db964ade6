"""bench.py's reference arm (the CPU oracle, this tier's reference) prints the contract's JSON line (CPU, small)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1",
                        "--ref-per-step", "8"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in line["config"]


def test_kcycle_algorithmic_bytes_count_raised_rows():
    """k_cycle's algorithmic bytes add the rows (10 B each) and RT, D, row offsets (20 B) of exactly the DNNs whose
    session level WMAX-MIN raised above the demand (level > 0, demand > 0, level != demand)."""
    import types

    import torch
    sys.path.insert(0, ROOT)
    import bench
    off = torch.tensor([0, 3, 10, 10, 14, 20], dtype=torch.int64)           # rows per DNN: 3, 7, 0, 4, 6
    dp = types.SimpleNamespace(dnn_row_off=off, num_rows=20, num_dnn=5, num_scen=2)
    out = {"level": torch.tensor([5, 9, 0, 4, 7], dtype=torch.int16),       # raised: DNN 1 (7 rows), DNN 4 (6 rows)
           "demand": torch.tensor([5, 6, 0, 0, 3], dtype=torch.int16)}      # DNN 3: demand 0 -> not counted
    assert bench.raised_rows(dp, out) == (2, 13)
    base = bench.algorithmic_bytes(dp, None)
    ab = bench.algorithmic_bytes(dp, None, out)
    assert ab["k_cycle"] - base["k_cycle"] == 10 * 13 + 2 * 20
    assert {k: v for k, v in ab.items() if k != "k_cycle"} == {k: v for k, v in base.items() if k != "k_cycle"}


def test_strong_and_weak_shards():
    """bench.shard_of: strong scaling splits the config's scenarios into contiguous global-index shards
    (SURVEY §8(e)); weak scaling gives every rank the config's size at its own global offset."""
    import types
    sys.path.insert(0, ROOT)
    import bench
    import synth
    sp0, _ = synth.config(3, num_scen=1_000_003)
    for world in (1, 2, 4, 8):
        got = [bench.shard_of(types.SimpleNamespace(scaling="strong"), sp0, r, world) for r in range(world)]
        assert all(g[1] == 1_000_003 for g in got)
        assert got[0][0].scen_base == 0 and sum(g[2] for g in got) == 1_000_003
        assert all(got[i][0].scen_base + got[i][2] == got[i + 1][0].scen_base for i in range(world - 1))
        assert all(g[0].num_scen == g[2] for g in got)
        weak = [bench.shard_of(types.SimpleNamespace(scaling="weak"), sp0, r, world) for r in range(world)]
        assert all(w[0].scen_base == r * 1_000_003 and w[2] == 1_000_003 and w[1] == 1_000_003 * world
                   for r, w in enumerate(weak))


def test_selection_gather_equals_host_draw():
    """synth.select._gather (config-4 workload assembly) on CPU tensors: the gathered scenarios are byte-identical
    to the generator's host re-draw of the same global indices."""
    import numpy as np
    import torch
    import synth
    from synth.select import _concat, _gather
    sp, _ = synth.config(4, num_scen=40, rows_pct=10)
    pb = synth.generate_host(sp)
    g = {k: torch.from_numpy(np.ascontiguousarray(getattr(pb, k)).view(
        {np.uint32: np.int32, np.uint16: np.int16}.get(getattr(pb, k).dtype.type, getattr(pb, k).dtype)))
         for k in ("scen_dnn_off", "dnn_row_off", "t_p", "t_np", "mem_bw", "slo_us", "asm_us", "bmax", "shape",
                   "lam_pct", "n", "r", "d")}
    sel = [3, 4, 11, 12, 13, 30, 39]
    parts = [_gather(g, torch.tensor(sel[:3]), "cpu"), _gather(g, torch.tensor(sel[3:]), "cpu")]
    got = _concat(parts, "cpu")
    want = synth.sample(sp, sel)
    R = want.num_rows
    for k in ("scen_dnn_off", "dnn_row_off", "t_p", "t_np", "mem_bw", "slo_us", "asm_us", "bmax"):
        assert np.array_equal(got[k].numpy(), getattr(want, k)), k
    for k, dt in (("n", np.uint32), ("r", np.uint16), ("d", np.uint32)):
        assert np.array_equal(got[k][:R].numpy().view(dt), getattr(want, k)[:R]), k
