"""Preconditioner (c64 V-cycle of a c128 block) throughput: one k = 32 cycle
vs 4 concurrent k = 8 cycles (4 solvers, one host thread each) vs one k = 8
cycle alone -- does a lockstep k = 32 V-cycle beat the concurrent groups?
(hz_cycle_device synchronises per call: a few us of host latency each.)"""
import sys, time, threading
sys.path.insert(0, ".")
import torch
import paper_1607_00968_b200 as hz
import bench

N = 60
cfg = bench.build_workload(0, 1, 32)
cfg.krylov_block = 0
P = hz.HelmholtzProblem.from_config(cfg)
opts = hz.HelmholtzSolveOptions.from_config(cfg)
B = torch.from_numpy(cfg.rhs_block()).cuda()
S32 = hz.HelmholtzSolver(P, opts)
S8 = [hz.HelmholtzSolver(P, opts) for _ in range(4)]
B8 = [B[:, 8 * i:8 * i + 8].contiguous() for i in range(4)]


def run(S, b, n):
    for _ in range(n):
        S.cycle(b)


for S, b in [(S32, B)] + list(zip(S8, B8)):
    run(S, b, 3)
torch.cuda.synchronize()
t = time.perf_counter(); run(S32, B, N); torch.cuda.synchronize()
print(f"k=32 one cycle: {1e3 * (time.perf_counter() - t) / N:.3f} ms")
t = time.perf_counter(); run(S8[0], B8[0], N); torch.cuda.synchronize()
print(f"k=8 one cycle alone: {1e3 * (time.perf_counter() - t) / N:.3f} ms")
th = [threading.Thread(target=run, args=(S8[i], B8[i], N)) for i in range(4)]
t = time.perf_counter()
for x in th: x.start()
for x in th: x.join()
torch.cuda.synchronize()
print(f"4 x k=8 concurrent: {1e3 * (time.perf_counter() - t) / N:.3f} ms per round of 4 cycles")
