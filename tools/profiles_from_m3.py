"""Copy a tools/measure_r02c.sh run (gpurun_out/m3_*) into profiles/ (bench lines, counters, launch list, full-capture
metrics).  Usage: python tools/profiles_from_m3.py <label> [config-5 file suffix]"""
import csv
import json
import shutil
import sys

WANT = ("gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__occupancy_limit", "launch__registers_per_thread", "smsp__average_warp_latency_per_inst_issued.ratio",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__grid_size", "launch__block_size",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__average_warps_issue_stalled_", "launch__shared_mem_per_block")


def grab(path, kernel):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        if not any(kernel in c for c in r[:12]):
            continue
        out = {}
        for i, h in enumerate(hdr):
            if h.startswith(WANT):
                if h.startswith("smsp__average_warps_issue_stalled_") and not (
                        h.endswith("per_issue_active.ratio") and float((r[i] or "0").replace(",", "")) > 0.05):
                    continue
                out[h] = (r[i] + (" " + units[i] if units[i] else "")).strip()
        return out


def main(label, c5="c5w1"):
    d = {"_source": f"{label}: ncu --set full --clock-control none; bench.py config 3 launch configuration (1M scenarios) "
                    "and config 4 (k_ideal_sim; 20k scenarios); units as ncu prints them",
         "k_prof_lane": grab("gpurun_out/m3_full_raw.csv", "k_prof_lane"),
         "k_cycle": grab("gpurun_out/m3_full_raw.csv", "k_cycle"),
         "k_ideal_sim(config4,20k)": grab("gpurun_out/m3_ki_raw.csv", "k_ideal_sim")}
    json.dump(d, open("profiles/r02_ncu_full_metrics.json", "w"), indent=1)
    shutil.copy("gpurun_out/m3_counters.json", "profiles/counters.json")
    shutil.copy("gpurun_out/m3_launches.csv", "profiles/r02_launches.csv")
    for c in (1, 2, 3, 4):
        shutil.copy(f"gpurun_out/m3_bench_c{c}.json", f"profiles/r02_bench_config{c}.json")
    shutil.copy(f"gpurun_out/m3_bench_{c5}.json", "profiles/r02_bench_config5.json")
    shutil.copy("gpurun_out/m3_ref.json", "profiles/r02_bench_reference_arm.json")


if __name__ == "__main__":
    main(sys.argv[1], *(sys.argv[2:3]))
