"""Per-kernel CUDA-event profile of one config-2 block solve (GPU)."""
import sys, json, time
sys.path.insert(0, ".")
import torch
import paper_1607_00968_b200 as hz
import bench

k = int(sys.argv[1]) if len(sys.argv) > 1 else 32
cfg = bench.build_workload(0, 1, k)
if len(sys.argv) > 2:
    cfg.precond_precision = sys.argv[2]
P = hz.HelmholtzProblem.from_config(cfg)
S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg, max_cycles=int(sys.argv[3]) if len(sys.argv) > 3 else 30))
B = torch.from_numpy(cfg.rhs_block()).cuda()
X, rep = S.solve_block(B)
torch.cuda.synchronize()
t = time.time()
X, rep = S.solve_block(B)
dt = time.time() - t
print("cycles", rep.cycles, "s", dt, "ms/cycle", 1e3 * dt / rep.cycles)
with hz.kernel_profile() as p:
    S.solve_block(B)
tot = sum(r["ms"] for r in p.result.values())
for name, r in sorted(p.result.items(), key=lambda kv: -kv[1]["ms"]):
    gbs = r["bytes"] / (r["ms"] / 1e3) / 1e9 if r["ms"] else 0
    tf = r["flops"] / (r["ms"] / 1e3) / 1e12 if r["ms"] else 0
    print(f"{name:24s} n={r['count']:6d} ms={r['ms']:9.2f} ({100*r['ms']/tot:5.1f}%) avg_us={1e3*r['ms']/r['count']:9.1f} GB/s={gbs:8.1f} TF/s={tf:6.2f}")
print("kernel total ms", tot, "wall ms", 1e3 * dt)
