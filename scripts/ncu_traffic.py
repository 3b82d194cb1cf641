"""Per-kernel DRAM traffic (dram__bytes_read + dram__bytes_write, per launch)
from an `ncu --set full` report, keyed by the library's profile names, written
to profiles/ncu_traffic.json for bench.py's roofline `traffic` field.

  python scripts/ncu_traffic.py gpurun_out/full.ncu-rep [out.json]
"""
import csv, json, re, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else "profiles/ncu_traffic.json"
# bench workload geometry (config 2, 8-column blocks): fine nodes, coarse
# (level-1) nodes, block width -- for the per-launch algorithmic bytes
N, NC, K = 1025 * 513, 513 * 257, 8


def algorithmic(k):
    """Algorithmic bytes of one captured launch (SURVEY 8d formulas, as the
    library's profiler counts them), or None when the name does not fix them."""
    m = re.search(r"gram8_kernel<(\d+)>", k)
    if m:  # Arnoldi Gram: Y = W is the last of the nb X blocks
        return int(m.group(1)) * N * K * 16
    m = re.search(r"update8_kernel<(\d+), (double|float)>", k)
    if m:  # the Arnoldi update writes Q from nb blocks (Yin = null); the
        # restart update X += Z Y reads nb c64 blocks and X
        nb = int(m.group(1))
        return (nb + 1) * N * K * 16 if m.group(2) == "double" else nb * N * K * 8 + 2 * N * K * 16
    if "fused_pre_k8_kernel<" in k:
        return N * (K * (16 + 8) + 16) + NC * K * 8
    if "fused_post_k8_kernel<" in k:
        return N * (K * (8 + 16 + 8) + 16) + NC * K * 8
    m = re.search(r"stencil9_k8_kernel<(\d)", k)
    if m:  # level-1 Galerkin sweep (2) / residual (1) / apply (0)
        mode = int(m.group(1))
        return NC * ((2 if mode == 0 else 3) * K * 8 + (9 + (1 if mode == 2 else 0)) * 8)
    if "fused_pre_kernel<float" in k:
        return N * (K * (16 + 8) + 16) + NC * K * 8
    if "fused_post_kernel<float" in k:
        return N * (K * (8 + 16 + 8) + 16) + NC * K * 8
    if "apply_lo_kernel" in k:
        return N * (K * (8 + 16) + 16)
    return None
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
    if "fused_pre_k8_kernel<" in k:
        return "fused_pre_fine_c64"
    if "fused_post_k8_kernel<" in k:
        return "fused_post_fine_c64"
    m = re.search(r"stencil9_k8_kernel<(\d)", k)
    if m:
        return {0: "apply_stencil_c64_L1", 1: "residual_stencil_c64_L1", 2: "jacobi_stencil_c64_L1"}[int(m.group(1))]
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


acc = defaultdict(lambda: {"n": 0, "bytes": 0.0, "us": 0.0, "alg": 0.0, "nalg": 0, "bytes_alg": 0.0})
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    nm = name_of(d["Kernel Name"])
    if not nm:
        continue
    b = sum(float(d[m]) * scale[u[m]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    acc[nm]["n"] += 1
    acc[nm]["bytes"] += b
    a = algorithmic(d["Kernel Name"])
    if a:
        acc[nm]["alg"] += a
        acc[nm]["bytes_alg"] += b
        acc[nm]["nalg"] += 1
    acc[nm]["us"] += float(d["gpu__time_duration.sum"]) * (1e-3 if u["gpu__time_duration.sum"] == "nsecond" else 1)
res = {k: {"dram_bytes_per_launch": v["bytes"] / v["n"], "launches_captured": v["n"],
           "dram_over_algorithmic": round(v["bytes_alg"] / v["alg"], 4) if v["nalg"] else None,
           "ncu_us_per_launch": round(v["us"] / v["n"], 2),
           "note": f"mean over {v['n']} consecutive launches of one ncu --set full capture ({rep.split('/')[-1]})"}
       for k, v in acc.items()}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
