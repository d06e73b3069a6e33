"""tcgen05 / TMEM / memory-op instruction counts per kernel of libromap.so
(cuobjdump -sass), the static evidence that the mixed kernels issue UTCHMMA
(tcgen05.mma) and LDTM (tcgen05.ld).  Usage: python tools/sass_summary.py [out.md]"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTCATOMSWS", "LDG", "REDG", "STG", "LDS", "STS", "SYNCS", "HMMA"]


def main(out=None):
    lib = os.path.join(ROOT, "paper_2304_05735_b200", "libromap.so")
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    pat = re.compile(r"\b(" + "|".join(OPS) + r")\b")
    cur, counts = None, collections.OrderedDict()
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        if cur:
            counts[cur].update(pat.findall(line))
    md = ["# SASS instruction counts (static, cuobjdump -sass libromap.so)", "",
          "| kernel | " + " | ".join(OPS) + " |", "|---|" + "---|" * len(OPS)]
    for fn, c in counts.items():
        name = subprocess.run(["c++filt", fn], capture_output=True, text=True).stdout.strip().split("(")[0] or fn[:60]
        if not any(c.values()):
            continue
        md.append(f"| `{name}` | " + " | ".join(str(c.get(o, 0)) for o in OPS) + " |")
    text = "\n".join(md) + "\n"
    if out:
        open(out, "w").write(text)
    print(text)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
