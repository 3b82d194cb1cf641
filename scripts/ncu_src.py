"""Per-SASS-line view of one kernel of an ncu report exported with
`ncu -i rep --page source --csv --kernel-id :::N > file.csv`: hottest lines by
stall samples, shared-memory lines with excess wavefronts, instruction mix."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[h]
ix = {name: i for i, name in enumerate(hdr)}
print(rows[0][1][:120] if rows[0] else "")


def num(v):
    try:
        return float(v)
    except ValueError:
        return 0.0


out, tot = [], 0
for r in rows[h + 1:]:
    if len(r) < len(hdr):
        continue
    samp = int(num(r[ix["# Samples"]]))
    tot += samp
    out.append(dict(samp=samp, src=r[ix["Source"]], wf=num(r[ix["L1 Wavefronts Shared"]]),
                    ideal=num(r[ix["L1 Wavefronts Shared Ideal"]]), exc=num(r[ix["L1 Wavefronts Shared Excessive"]]),
                    n=int(num(r[ix["Instructions Executed"]])), lsb=r[ix["stall_long_sb"]], ssb=r[ix["stall_short_sb"]],
                    loc=num(r[ix["L2 Theoretical Sectors Local"]]) if "L2 Theoretical Sectors Local" in ix else 0.0))
print("total samples", tot)
print("== top lines by samples")
for o in sorted(out, key=lambda o: -o["samp"])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{o['samp']:7d} n={o['n']:9d} lsb={o['lsb']:>6} ssb={o['ssb']:>6} wf={o['wf']:.0f}/{o['ideal']:.0f}  {o['src'][:90]}")
print("== shared-memory lines with excess wavefronts")
for o in out:
    if o["exc"] > 0:
        print(f"   exc={o['exc']:.0f} wf={o['wf']:.0f} ideal={o['ideal']:.0f} n={o['n']}  {o['src'][:90]}")
print("== local-memory lines")
for o in out:
    if o["loc"] > 0:
        print(f"   sectors={o['loc']:.0f} n={o['n']}  {o['src'][:90]}")
mix = collections.Counter()
for o in out:
    parts = o["src"].split()
    if not parts:
        continue
    op = parts[1] if parts[0].startswith("@") and len(parts) > 1 else parts[0]
    mix[op.split(".")[0]] += o["n"]
print("== warp-instruction mix", mix.most_common(24), "total", sum(mix.values()))
