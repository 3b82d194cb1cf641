"""Per-kernel DRAM traffic (dram__bytes_read + dram__bytes_write, per launch)
from an `ncu --set full` report, keyed by the library's profile names, written
to profiles/ncu_traffic.json for bench.py's roofline `traffic` field.

  python scripts/ncu_traffic.py gpurun_out/full.ncu-rep [out.json]
"""
import csv, json, re, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else "profiles/ncu_traffic.json"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def name_of(k):
    if "update8_kernel" in k:
        return "multi_update_lo_c128" if ", float>" in k else "multi_update_c128"
    if "gram8_kernel" in k:
        return "multi_gram_c128"
    if "apply_lo_kernel" in k:
        return "apply_fine_c128"
    if "fused_pre_kernel<float" in k:
        return "fused_pre_fine_c64"
    if "fused_post_kernel<float" in k:
        return "fused_post_fine_c64"
    if "update_kernel" in k:
        return "multi_update_c128"
    if "gram_kernel" in k:
        return "multi_gram_c128"
    m = re.search(r"fine_v4_kernel<float, (\d), (\d), (\w+)>", k)
    if m:
        mode, out_t = int(m.group(2)), m.group(3)
        if mode == 2:
            return "jacobi_out64_fine_c64" if out_t == "double2" else "jacobi_fine_c64"
        return {0: "apply_fine_c64", 1: "residual_fine_c64"}[mode]
    m = re.search(r"level_kernel<double, \d, 0, 0>", k)
    if m:
        return "apply_fine_c128"
    return None


acc = defaultdict(lambda: {"n": 0, "bytes": 0.0, "us": 0.0})
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    nm = name_of(d["Kernel Name"])
    if not nm:
        continue
    b = sum(float(d[m]) * scale[u[m]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    acc[nm]["n"] += 1
    acc[nm]["bytes"] += b
    acc[nm]["us"] += float(d["gpu__time_duration.sum"]) * (1e-3 if u["gpu__time_duration.sum"] == "nsecond" else 1)
res = {k: {"dram_bytes_per_launch": v["bytes"] / v["n"], "launches_captured": v["n"],
           "ncu_us_per_launch": round(v["us"] / v["n"], 2),
           "note": f"mean over {v['n']} consecutive launches of one ncu --set full capture ({rep.split('/')[-1]})"}
       for k, v in acc.items()}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
