"""Per source line executed warp-instructions and stall samples from an
`ncu --page source --csv --print-source cuda,sass` export (all files).
usage: python tools/ncu_srclines.py export.csv [top-n]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, h, out = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        h = r
        continue
    if h is None or not r[0].isdigit():
        continue
    try:
        ex = int(r[h.index("Instructions Executed")] or 0)
        st = int(r[h.index("Warp Stall Sampling (All Samples)")] or 0)
    except (ValueError, IndexError):
        continue
    if ex or st:
        out.append((ex, st, fname, int(r[0]), r[1].strip()[:80]))
tex = sum(o[0] for o in out)
tst = sum(o[1] for o in out)
print(f"total warp-instructions {tex}  stall samples {tst}")
for ex, st, f, ln, src in sorted(out, key=lambda o: -o[0])[:n]:
    print(f"{ex:10d} {100 * ex / tex:5.1f}% {st:6d} {f}:{ln:<5d} {src}")
