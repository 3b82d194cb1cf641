"""Per-launch timeline of the bench workload (4 concurrent 8-column groups)
from CUDA events (hz_profile_trace): writes the raw trace and prints the
busy fraction, concurrency histogram and per-kernel time shares.

  python scripts/timeline.py [cycles] [out.json]
"""
import sys, json
sys.path.insert(0, ".")
import torch
import paper_1607_00968_b200 as hz
import bench

cycles = int(sys.argv[1]) if len(sys.argv) > 1 else 60
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/trace.json"
cfg = bench.build_workload(0, 1, 32)
cfg.max_cycles = cycles
S = hz.HelmholtzSolver(hz.HelmholtzProblem.from_config(cfg), hz.HelmholtzSolveOptions.from_config(cfg))
B = torch.from_numpy(cfg.rhs_block()).cuda()
S.solve_block(B)
with hz.kernel_profile(trace=True) as p:
    S.solve_block(B)
tr = p.trace
json.dump(tr, open(out, "w"))
ev = []
for name, sid, t0, d, b in tr:
    ev.append((t0, 1, name, b / max(d, 1e-6)))
    ev.append((t0 + d, -1, name, b / max(d, 1e-6)))
ev.sort(key=lambda e: (e[0], e[1]))
t_lo, t_hi = min(e[0] for e in ev), max(e[0] for e in ev)
wall = t_hi - t_lo
hist, active, last, rate, bytes_t = {}, 0, t_lo, 0.0, 0.0
for t, kind, name, r in ev:
    dt = t - last
    hist[active] = hist.get(active, 0.0) + dt
    last = t
    active += kind
    rate += kind * r
tot_b = sum(x[4] for x in tr)
tot_d = sum(x[3] for x in tr)
print(f"launches {len(tr)}  wall {wall:.2f} ms  kernel-sum {tot_d:.2f} ms  mean concurrency {tot_d / wall:.2f}")
print(f"algorithmic bytes {tot_b / 1e9:.2f} GB -> {tot_b / 1e6 / wall:.0f} GB/s over the wall")
print("time share by number of active kernels:", {k: round(v / wall, 3) for k, v in sorted(hist.items())})
agg = {}
for name, sid, t0, d, b in tr:
    a = agg.setdefault(name, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += d
    a[2] += b
for name, (n, d, b) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:20]:
    print(f"{name:28s} n={n:6d} sum_ms={d:8.2f} ({100 * d / tot_d:5.1f}%) avg_us={1e3 * d / n:7.1f} GB/s={b / 1e6 / d:7.0f}")
