"""DMMA vs FFMA tiles for the c128 Gram / update on the config-2 solve."""
import os, sys, time, json
sys.path.insert(0, ".")
import subprocess
for dm in ("1", "0"):
    code = r'''
import sys, time, json
sys.path.insert(0, ".")
import torch, paper_1607_00968_b200 as hz, bench
cfg = bench.build_workload(0, 1, 32)
P = hz.HelmholtzProblem.from_config(cfg)
S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg))
B = torch.from_numpy(cfg.rhs_block()).cuda()
X, rep = S.solve_block(B)
torch.cuda.synchronize(); t = time.time()
X, rep = S.solve_block(B)
torch.cuda.synchronize(); dt = time.time() - t
with hz.kernel_profile() as p:
    S.solve_block(B)
r = {k: round(v["ms"] / v["count"] * 1e3, 1) for k, v in p.result.items() if k.startswith(("multi_", "coarse", "pip", "jacobi_fine"))}
tf = {k: round(v["flops"] / (v["ms"] / 1e3) / 1e12, 2) for k, v in p.result.items() if k.startswith("multi_")}
print(json.dumps(dict(dmma=sys.argv[1], cycles=rep.cycles, s=round(dt, 3), rhs_per_s=round(32 / dt, 2), ms_per_cycle=round(1e3 * dt / rep.cycles, 3), avg_us=r, tf=tf)))
'''
    env = dict(os.environ, HZ_DMMA=dm)
    out = subprocess.run([sys.executable, "-c", code, dm], env=env, capture_output=True, text=True)
    print(out.stdout.strip() or out.stderr[-2000:], flush=True)
