"""Opcode histogram (executed warp instructions, stall samples) from an
ncu source-page CSV export (--page source --csv --print-source sass)."""
import csv, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
h = [r for r in rows if r and r[0] == "Address"][0]
data = [r for r in rows if r and r[0].startswith("0x")]
iS, iE, iSrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
num = lambda v: int(float(v)) if v not in ("", "-") else 0
tot = sum(num(r[iS]) for r in data) or 1
ti = sum(num(r[iE]) for r in data) or 1
print("stall samples", tot, "warp instructions", ti, "static instructions", len(data))
c, cs = Counter(), Counter()
for r in data:
    toks = r[iSrc].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    c[op] += num(r[iE])
    cs[op] += num(r[iS])
for op, n in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{op:10s} {n:12d} {100 * n / ti:5.1f}%  stall-samples {100 * cs[op] / tot:5.1f}%")
