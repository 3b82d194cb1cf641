"""Multi-frequency batching throughput on the bench workload
(config 2, k = 32, c64 preconditioner): nf frequencies omega * (0.6, 0.8, 1.0)
solved sequentially vs as one concurrent batch (hz_solve_blocks_multi)."""
import sys, time, json
sys.path.insert(0, ".")
import torch, paper_1607_00968_b200 as hz, bench

base = bench.build_workload(0, 1, 32)
scales = [float(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ("0.6", "0.8", "1.0"))]
opts = hz.HelmholtzSolveOptions.from_config(base)
M = hz.MultiFrequencySolver(base.ndim, base.n, base.h, base.m, [base.omega * s for s in scales],
                            hz.AttenuationField(base.gamma_base, base.ramp), opts)
B = torch.from_numpy(base.rhs_block()).cuda()
Bs = [B] * len(M)
Xs, reps = M.solve_blocks(Bs)  # warm-up
for S in M.solvers:
    S.solve_block(B)
torch.cuda.synchronize()
t = time.perf_counter()
seq = [S.solve_block(B)[1] for S in M.solvers]
torch.cuda.synchronize()
t_seq = time.perf_counter() - t
t = time.perf_counter()
Xs, reps = M.solve_blocks(Bs)
torch.cuda.synchronize()
t_con = time.perf_counter() - t
nrhs = 32 * len(M)
print(json.dumps({"frequencies": scales, "cycles": [r.cycles for r in reps], "converged": all(r.all_converged() for r in reps),
                  "sequential_s": round(t_seq, 3), "concurrent_s": round(t_con, 3),
                  "rhs_freq_per_s_sequential": round(nrhs / t_seq, 2), "rhs_freq_per_s_concurrent": round(nrhs / t_con, 2),
                  "speedup": round(t_seq / t_con, 3)}))
