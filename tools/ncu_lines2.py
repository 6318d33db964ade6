"""Per-source-line summary with average active / predicated-on threads (ncu --page source --csv export)."""
import csv
import sys


def main(path, top=40, fname_filter=None):
    rows, fname = [], None
    for rec in csv.reader(open(path)):
        if not rec:
            continue
        if rec[0] == "File Path":
            fname = rec[1].rsplit("/", 1)[-1]
            continue
        if rec[0].isdigit() and len(rec) > 11 and rec[2] == "-":
            try:
                samp, inst, thr, pthr = int(rec[6]), int(rec[7]), int(rec[8]), int(rec[9])
            except ValueError:
                continue
            rows.append((inst, samp, thr, pthr, f"{fname}:{rec[0]}", rec[1][:80]))
    ti = sum(r[0] for r in rows) or 1
    tt = sum(r[2] for r in rows) or 1
    tp = sum(r[3] for r in rows) or 1
    ts = sum(r[1] for r in rows) or 1
    print(f"warp-instr {ti:.3e}  thread-instr {tt:.3e} ({tt/ti:.2f}/warp-instr)  predicated-on {tp:.3e} ({tp/ti:.2f})")
    for inst, samp, thr, pthr, loc, src in sorted(rows, reverse=True)[:top]:
        print(f"{100*inst/ti:5.1f}% inst {100*samp/ts:5.1f}% samp  thr {thr/max(inst,1):5.1f} pred {pthr/max(inst,1):5.1f}  {loc:18s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
