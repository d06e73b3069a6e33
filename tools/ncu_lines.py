"""Top source lines of an ncu --page source --csv --print-source cuda,sass export by warp-stall samples."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
h = rows[hi]
si = h.index("Warp Stall Sampling (All Samples)")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
lines = []
tot = 0
for r in rows[hi + 1:]:
    if r and r[0] and len(r) > si:
        try:
            s = int(r[si])
        except ValueError:
            continue
        tot += s
        det = {c: int(r[h.index(c)]) for c in cols if r[h.index(c)] not in ("", "0", "-")}
        lines.append((s, r[0], r[1][:70], det))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print("total samples", tot)
for s, ln, src, det in sorted(lines, key=lambda x: -x[0])[:n]:
    top = sorted(det.items(), key=lambda x: -x[1])[:3]
    print(f"{s:6d} {100*s/tot:5.1f}% L{ln:>4} {src:70s} {top}")
