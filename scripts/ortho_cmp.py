"""Compare orthogonalisation variants (PIP one-pass vs CGS2) on config 2."""
import os, sys, time, json
sys.path.insert(0, ".")
import torch
import paper_1607_00968_b200 as hz
import bench
k = 32
for restart in (5, 10):
    for ortho in ("pip", "cgs2"):
        os.environ["HZ_ORTHO"] = ortho
        cfg = bench.build_workload(0, 1, k)
        cfg.restart = restart
        P = hz.HelmholtzProblem.from_config(cfg)
        S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg))
        B = torch.from_numpy(cfg.rhs_block()).cuda()
        X, rep = S.solve_block(B)
        torch.cuda.synchronize(); t = time.time()
        X, rep = S.solve_block(B)
        torch.cuda.synchronize(); dt = time.time() - t
        print(json.dumps(dict(restart=restart, ortho=ortho, cycles=rep.cycles, conv=rep.all_converged(),
                              worst=float(rep.rel_residual.max()), s=round(dt, 3), ms_per_cycle=round(1e3*dt/rep.cycles, 3),
                              rhs_per_s=round(k/dt, 2), qr=rep.qr_factorizations, grams=rep.block_gram_products)), flush=True)
        if ortho == "pip" and restart == 5:
            with hz.kernel_profile() as p:
                S.solve_block(B)
            tot = sum(r["ms"] for r in p.result.values())
            for name, r in sorted(p.result.items(), key=lambda kv: -kv[1]["ms"])[:8]:
                print(f"   {name:24s} n={r['count']:6d} ms={r['ms']:9.2f} ({100*r['ms']/tot:5.1f}%)", flush=True)
