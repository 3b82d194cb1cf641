"""Per-instruction table of one kernel from an ncu report (source page, SASS):
instructions executed, stall samples; prints the hottest instructions and
the total executed warp instructions."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
i = next(k for k, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[i]
data = [dict(zip(hdr, r)) for r in rows[i + 1:] if len(r) == len(hdr) and r[0].startswith("0x")]
ie = lambda d: int(d["Instructions Executed"] or 0)
tot = sum(ie(d) for d in data)
samp = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
print(f"instructions executed (warp): {tot}, stall samples: {samp}")
for d in data:
    pass
# group by opcode
from collections import Counter
c = Counter()
for d in data:
    op = d["Source"].split()[0] if not d["Source"].strip().startswith("@") else d["Source"].split()[1]
    c[op.split(".")[0]] += ie(d)
print("by opcode:", ", ".join(f"{k}={v/tot:.1%}" for k, v in c.most_common(18)))
for d in sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:top]:
    print(f'{d["Address"][-5:]} {ie(d):9d} {d["Warp Stall Sampling (All Samples)"]:>6} {d["Source"].strip()[:70]}')

# stall reasons summed over the kernel, and the top instructions per reason
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot_r = {h: sum(int(d[h] or 0) for d in data) for h in reasons}
print("stalls:", ", ".join(f"{h[6:]}={v}" for h, v in sorted(tot_r.items(), key=lambda kv: -kv[1]) if v))
for h, v in sorted(tot_r.items(), key=lambda kv: -kv[1])[:3]:
    print(f"-- {h}")
    for d in sorted(data, key=lambda d: -int(d[h] or 0))[:6]:
        print(f'   {d["Address"][-5:]} {int(d[h] or 0):5d} {d["Source"].strip()[:70]}')
