"""Warp-instructions per unit by source line (ncu --page source --csv export), in source order."""
import csv
import sys


def load(path):
    rows, fname = {}, None
    for rec in csv.reader(open(path)):
        if not rec:
            continue
        if rec[0] == "File Path":
            fname = rec[1].rsplit("/", 1)[-1]
            continue
        if rec[0].isdigit() and len(rec) > 11 and rec[2] == "-":
            try:
                inst = int(rec[7])
            except ValueError:
                continue
            if inst:
                rows[(fname, int(rec[0]))] = (inst, rec[1][:90])
    return rows


if __name__ == "__main__":
    rows = load(sys.argv[1])
    units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    tot = sum(v[0] for v in rows.values())
    print(f"total {tot/units:.0f} per unit")
    for (f, ln), (inst, src) in sorted(rows.items()):
        if inst / units >= float(sys.argv[3] if len(sys.argv) > 3 else 20):
            print(f"{f:14s}:{ln:4d} {inst/units:8.0f}  {src}")
