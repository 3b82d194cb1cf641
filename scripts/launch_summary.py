"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) per
kernel: launches, total time, share (cold-cache serialised launch times --
compare SHARES with bench.py's CUDA-event profile, not absolutes)."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
h = rows[0]
iK, iM, iV, iU = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
acc = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if len(r) <= iV or r[iM] != "gpu__time_duration.sum":
        continue
    v = float(r[iV].replace(",", ""))
    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[iU], 1.0)
    name = r[iK].split("(")[0].replace("(anonymous namespace)::", "")[-70:]
    acc[name][0] += 1
    acc[name][1] += v
tot = sum(v[1] for v in acc.values())
print(f"launches {sum(v[0] for v in acc.values())}, total {tot / 1e3:.2f} ms")
for name, (n, us) in sorted(acc.items(), key=lambda kv: -kv[1][1]):
    print(f"{name:72s} {n:5d} {us:11.1f} us {100 * us / tot:5.1f}%")
