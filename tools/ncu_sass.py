"""Top SASS instructions of an `ncu --page source --csv --print-source sass` export by warp-stall samples,
with a window of preceding instructions for context."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
si = h.index("Warp Stall Sampling (All Samples)")
ei = h.index("Instructions Executed")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ins = []
for r in rows[hi + 1:]:
    if len(r) <= si:
        continue
    det = {c: int(r[h.index(c)]) for c in cols if r[h.index(c)] not in ("", "0", "-")}
    ins.append((int(r[si] or 0), r[1].strip(), int(r[ei] or 0), det))
tot = sum(x[0] for x in ins)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
order = sorted(range(len(ins)), key=lambda i: -ins[i][0])[:n]
print("total samples", tot, "instructions", len(ins))
for i in order:
    s, src, ex, det = ins[i]
    top = sorted(det.items(), key=lambda x: -x[1])[:3]
    print(f"{i:5d} {s:5d} {100*s/tot:4.1f}% ex={ex:8d} {src[:60]:60s} {top}")
