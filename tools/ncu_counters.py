"""Per-scenario kernel counters from an ncu --csv metrics log (the bench launch configuration).

  ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file gpurun_out/counters.csv python bench.py --steps 1 --warmup 3 ...
  python tools/ncu_counters.py gpurun_out/counters.csv 1000000 profiles/counters.json "<label>"

Kernels are grouped into the bench's profiling slots (k_prof*, k_wmaxmin, k_cycle, k_agg*); every value is
the per-launch mean of the slot's kernels summed, divided by the scenarios per launch."""
import csv
import json
import sys
from collections import defaultdict

SLOTS = (("k_prof", "k_prof"), ("k_wmaxmin", "k_wmaxmin"), ("k_cycle", "k_cycle"), ("k_agg", "k_agg"),
         ("k_ideal", "k_ideal"))
# the next-row legs' kernels (bench.py compare / below_knee / knee_probe / cluster legs), counted in a separate run
LEG_SLOTS = (("k_compare", "k_compare"), ("k_cluster", "k_cluster"), ("k_cycle<1,", "k_cycle_bk"), ("k_cycle<1>", "k_cycle_bk"),
             ("k_cycle<true,", "k_cycle_bk"), ("k_cycle<true>", "k_cycle_bk"), ("k_prof<0>", "k_knee_probe"))


def slot_of(name, legs=False):
    for key, slot in (LEG_SLOTS if legs else SLOTS):
        if key in name:
            return slot
    return None


def main(path, nscen, out, label, legs=False):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    per = defaultdict(lambda: defaultdict(float))     # (slot, kernel) -> metric -> sum
    launches = defaultdict(set)
    for r in rows:
        sl = slot_of(r["Kernel Name"], legs)
        if sl is None:
            continue
        name = r["Kernel Name"].split("(")[0]
        launches[(sl, name)].add(r["ID"])
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        if r["Metric Name"] == "gpu__time_duration.sum":
            v = v * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1e-6)
        elif r["Metric Name"].startswith("dram__bytes"):
            v = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        per[(sl, name)][r["Metric Name"]] += v
    res = {}
    for (sl, name), m in per.items():
        n = len(launches[(sl, name)])
        d = res.setdefault(sl, {"kernels": [], "warp_inst": 0.0, "dram_bytes": 0.0, "ncu_ms": 0.0})
        d["kernels"].append(name)
        d["warp_inst"] += m["smsp__inst_executed.sum"] / n / nscen
        d["dram_bytes"] += (m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]) / n / nscen
        d["ncu_ms"] += m["gpu__time_duration.sum"] / n
    src = (f"{label}: ncu --metrics smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
           f"gpu__time_duration.sum --clock-control none over bench.py (per launch / {nscen} scenarios)")
    if legs:   # merge into an existing counters file under "legs"
        with open(out) as f:
            doc = json.load(f)
        doc["legs"] = res
        doc["_source_legs"] = src
    else:
        doc = {"_source": src, "per_scenario": res}
    with open(out, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else "",
         legs=len(sys.argv) > 5 and sys.argv[5] == "--legs")
