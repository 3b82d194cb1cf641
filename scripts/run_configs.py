"""Run BASELINE configs 1-5 (one GPU) through the public API: setup time,
cycles, RHS/s, residuals. Solver settings per config are the converging
variants recorded in DESIGN.md §5."""
import sys, time, json, os
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1607_00968_b200 as hz
from paper_1607_00968_b200 import configs


def make(c):
    if c == 1:
        cfg = configs.config1(nlevels=3)                   # converging 3-level variant
        cfg.restart = 10
    elif c == 2:
        import bench
        cfg = bench.build_workload(0, 1, 32)
    elif c == 3:
        cfg = configs.config3(nlevels=3)                   # coarsest 33x33x17: plane block-tridiagonal
        cfg.precond_precision, cfg.krylov_block, cfg.restart = "c64", 8, 5  # 2 concurrent 8-column blocks
    elif c == 4:
        cfg = configs.config4(nlevels=3)                   # coarsest 65x65x33
        cfg.source_nodes = cfg.source_nodes[:8]            # k = 8 per GPU (64 RHS sharded 8 per GPU)
        cfg.precond_precision = "c64"
    elif c == 5:
        cfg = configs.config5(nlevels=6)                   # the literal 6 levels, coarsest 17x17x9
        # V(2,2), shift 1.2, w_J 0.5, FGMRES(5): 433 cycles, 20.3 s (profiles/r02_cfg5_sweep.jsonl; 4 levels / shift 1.0:
        # 397 cycles, 20.1 s; w_J 0.8 needed 4 levels + W at shift 1.5: 1,286 cycles, 84.8 s)
        cfg.shift, cfg.restart, cfg.jacobi_weight = 1.2, 5, 0.5
    for key in ("nlevels", "shift", "restart", "max_cycles", "precond_precision", "krylov_block", "jacobi_weight",
                "cycle", "stencil"):
        v = os.environ.get(f"HZ_CFG{c}_{key.upper()}")
        if v is not None:
            setattr(cfg, key, type(getattr(cfg, key))(v))
    return cfg


if __name__ == "__main__":
    which = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 2, 3, 4, 5]
    prof = os.environ.get("HZ_PROFILE") == "1"
    for c in which:
        cfg = make(c)
        t = time.time()
        P = hz.HelmholtzProblem.from_config(cfg)
        S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg))
        torch.cuda.synchronize()
        setup = time.time() - t
        B = torch.from_numpy(cfg.rhs_block()).cuda()
        # HZ_SLABS="1,8": solve once per slab count (parts as streams on this GPU)
        for slabs in [int(x) for x in os.environ.get("HZ_SLABS", "1").split(",")]:
            X = None
            torch.cuda.empty_cache()
            S.set_slabs(slabs)
            if os.environ.get("HZ_WARM", "1") == "1" and cfg.num_nodes * cfg.k < 2 ** 27:
                S.solve_block(B)  # warm-up solve (first-launch costs), not timed
            torch.cuda.synchronize(); t = time.time()
            X, rep = S.solve_block(B)
            torch.cuda.synchronize(); dt = time.time() - t
            out = dict(config=c, name=cfg.name, n=cfg.n, k=cfg.k, stencil=cfg.stencil, nlevels=cfg.nlevels, shift=cfg.shift,
                       restart=cfg.restart, prec=cfg.precond_precision, rhs_block=cfg.krylov_block, slabs=slabs,
                       setup_s=round(setup, 2),
                       solve_s=round(dt, 3), cycles=rep.cycles, converged=rep.all_converged(),
                       worst_res=float(rep.rel_residual.max()), rhs_per_s=round(cfg.k / dt, 3),
                       ms_per_cycle=round(1e3 * dt / max(rep.cycles, 1), 3))
            print(json.dumps(out), flush=True)
            if slabs > 1:
                S.set_slabs(1)
        if prof:
            with hz.kernel_profile() as p:
                S.solve_block(B)
            tot = sum(r["ms"] for r in p.result.values())
            for name, r in sorted(p.result.items(), key=lambda kv: -kv[1]["ms"])[:10]:
                print(f"   {name:24s} n={r['count']:6d} ms={r['ms']:9.2f} ({100*r['ms']/tot:5.1f}%) "
                      f"avg_us={1e3*r['ms']/r['count']:9.1f}", flush=True)
        del S, P, X, B
        torch.cuda.empty_cache()
