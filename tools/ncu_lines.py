"""Per-source-line summary of an ncu source page export (--page source --csv --print-source cuda,sass)."""
import csv
import sys


def main(path, top=40):
    rows, fname = [], None
    with open(path) as f:
        for rec in csv.reader(f):
            if not rec:
                continue
            if rec[0] == "File Path":
                fname = rec[1].rsplit("/", 1)[-1]
                continue
            if rec[0].isdigit() and len(rec) > 8 and rec[2] == "-":
                try:
                    samp, inst = int(rec[4]), int(rec[7])
                except ValueError:
                    continue
                rows.append((samp, inst, f"{fname}:{rec[0]}", rec[1][:90]))
    ts = sum(r[0] for r in rows) or 1
    ti = sum(r[1] for r in rows) or 1
    print(f"total samples {ts}  total warp-instr {ti:.3e}")
    for samp, inst, loc, src in sorted(rows, reverse=True)[:top]:
        print(f"{100*samp/ts:5.1f}% samp {100*inst/ti:5.1f}% inst  {loc:18s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
