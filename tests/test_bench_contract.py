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
