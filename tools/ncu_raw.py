"""Selected raw metrics of an ncu --page raw --csv export (first kernel row)."""
import csv
import sys

WANT = ("gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__occupancy_limit", "launch__registers_per_thread", "smsp__average_warp_latency_per_inst_issued.ratio",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__grid_size", "launch__block_size",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__average_warps_issue_stalled_")


def main(path, kernel=None):
    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    for r in rows[2:]:
        if kernel and not any(kernel in c for c in r[:12]):
            continue
        for i, h in enumerate(hdr):
            if h.startswith(WANT) and (not h.startswith("smsp__average_warps_issue_stalled_") or
                                       (h.endswith("per_issue_active.ratio") and float(r[i] or 0) > 0.05)):
                print(f"{h} {r[i]}")
        break


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
