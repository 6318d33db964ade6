"""SASS in address order with per-instruction executed counts and the source line each maps to
(ncu --page source --csv --print-source cuda,sass export)."""
import csv
import sys


def main(path, min_count=0, scale=1.0):
    rows, fname, line = [], None, None
    for rec in csv.reader(open(path)):
        if not rec:
            continue
        if rec[0] == "File Path":
            fname = rec[1].rsplit("/", 1)[-1]
            continue
        if rec[0].isdigit():
            line = f"{fname}:{rec[0]}"
            continue
        if rec[0] == "" and len(rec) > 8 and rec[2].startswith("0x"):
            try:
                inst, thr = int(rec[7]), int(rec[8])
            except ValueError:
                continue
            rows.append((int(rec[2], 16), rec[3].strip(), inst, thr, line))
    rows.sort()
    base = rows[0][0] if rows else 0
    for addr, sass, inst, thr, loc in rows:
        if inst >= min_count:
            print(f"{addr - base:6x} {inst * scale:10.2f} {thr / max(inst, 1):5.1f}  {loc:22s} {sass}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0, float(sys.argv[3]) if len(sys.argv) > 3 else 1.0)
