#!/usr/bin/env python
"""Run the REFERENCE solver to convergence on the bench workload's first RHS
block and commit the result as a golden fixture (TEST INFRASTRUCTURE).

The reference's own block_fgmres (oracle/_ref, the unmodified reference
sources compiled by oracle/Makefile; /root/reference/proj/core/src/krylov.cpp:178-280)
driven through the SURVEY §3.3 composition -- build_hierarchy +
MgHierarchy::cycle (V) + block_fgmres -- with exactly bench.py's WORKLOAD
settings (6 levels, shift 0.9, w_J 0.6, FGMRES(5), tol 1e-6) on block 0
(columns 0..7) of bench.build_workload(0, 1, 32). The reference has only a
complex128 preconditioner; our bench runs a complex64 one, so the fixture pins
(a) the reference's cycle count for the block (bench.py REF_CYCLES) and
(b) the converged solution, sampled on the receiver (surface) row and on a
strided node subset, against which tests/test_gpu_fullsize.py checks the GPU
bench solve (c64 and c128 preconditioner) at 1e-5.

  python scripts/ref_full_solve.py [--threads N] [--out tests/golden/cfg2_bench_block0.npz]
"""
from __future__ import annotations

import argparse
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from oracle import ref  # noqa: E402

SAMPLE_STRIDE = 997


def sample_nodes(cfg) -> np.ndarray:
    """Receiver row (the free surface z = 0: nodes 0..nx-1) + every
    SAMPLE_STRIDE-th node of the grid."""
    nx = int(cfg.n[0])
    return np.unique(np.concatenate([np.arange(nx), np.arange(0, cfg.num_nodes, SAMPLE_STRIDE)])).astype(np.int64)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def literal_config3():
    """BASELINE configs[2] as stated: 129x129x65, 7-point, k = 16, block FGMRES(10) + shifted-Laplacian MG with 4
    levels, V(2,2), tol 1e-6; the shift (1.0) and Jacobi weight (0.5) are not stated by BASELINE. 8-column blocks and
    the c64 cycle on the GPU side as in the other config-3 runs."""
    from paper_1607_00968_b200 import configs
    cfg = configs.config3(nlevels=4)
    cfg.shift, cfg.jacobi_weight, cfg.restart, cfg.cycle = 1.0, 0.5, 10, "V"
    cfg.precond_precision, cfg.krylov_block, cfg.max_cycles = "c64", 8, 600
    return cfg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--block", type=int, default=0)
    ap.add_argument("--blocks", default=None, help="comma-separated blocks solved in one run (one setup)")
    ap.add_argument("--config", type=int, default=2, help="2: the bench workload; 3: BASELINE config 3 at full size "
                    "(129x129x65, the converging 3-level variant of scripts/run_configs.py, 8-column blocks)")
    ap.add_argument("--bench", action="store_true", help="config 3 with bench.py --workload cfg3's solver settings "
                    "(-> cfg3_bench_block<b>.npz) instead of scripts/run_configs.py's recipe")
    ap.add_argument("--out", default=None)
    ap.add_argument("--literal", action="store_true", help="config 3 as BASELINE states it: 4 levels, V(2,2), FGMRES(10) "
                    "(with shift 1.0 and Jacobi weight 0.5, which BASELINE leaves open and at which the 4-level hierarchy "
                    "converges) -> cfg3_literal_block<b>.npz")
    args = ap.parse_args()
    blocks = [int(x) for x in args.blocks.split(",")] if args.blocks else [args.block]

    if args.config == 2:
        cfg = bench.build_workload(0, 1, bench.WORKLOAD["k"])
        settings = dict(bench.WORKLOAD)
        stem = "cfg2_bench_block"
    elif args.bench:
        bench.WORKLOAD = bench.WORKLOADS[f"cfg{args.config}"]
        cfg = bench.build_workload(0, 1, bench.WORKLOAD["k"])
        settings = dict(bench.WORKLOAD)
        stem = f"cfg{args.config}_bench_block"
    else:
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        import run_configs
        cfg = run_configs.make(args.config)
        if args.literal:
            cfg = literal_config3()
        settings = dict(config=args.config, n=list(map(int, cfg.n)), nlevels=cfg.nlevels, shift=cfg.shift,
                        restart=cfg.restart, cycle=cfg.cycle, pre=cfg.pre, post=cfg.post, wj=cfg.jacobi_weight,
                        tol=cfg.tol, krylov_block=cfg.krylov_block)
        stem = f"cfg{args.config}_literal_block" if args.literal else f"cfg{args.config}_full_block"
    b = cfg.krylov_block
    ref.set_num_threads(args.threads)
    t0 = time.perf_counter()
    R = ref.RefProblem.from_config(cfg)
    H = ref.RefHierarchy(R, cfg.nlevels, cfg.shift)
    setup_s = time.perf_counter() - t0
    nodes = sample_nodes(cfg)
    for block in blocks:
        out = args.out if (args.out and len(blocks) == 1) else os.path.join(ROOT, "tests", "golden", f"{stem}{block}.npz")
        cols = slice(block * b, (block + 1) * b)
        B = cfg.rhs_block(cols)
        t0 = time.perf_counter()
        X, rep = ref.krylov_solve(R, H, B, method="fgmres", kind=cfg.cycle, pre=cfg.pre, post=cfg.post,
                                  wj=cfg.jacobi_weight, restart=cfg.restart, tol=cfg.tol,
                                  max_cycles=cfg.max_cycles)
        solve_s = time.perf_counter() - t0
        np.savez_compressed(
            out, cycles=rep.cycles, col_cycles=np.asarray(rep.col_cycles), rel_residual=np.asarray(rep.rel_residual),
            converged=np.asarray(rep.converged), history=np.asarray(rep.history), nodes=nodes, x_sample=X[nodes],
            x_norm=np.linalg.norm(X, axis=0), source_nodes=np.asarray(cfg.source_nodes[cols]),
            setup_s=setup_s, solve_s=solve_s, threads=args.threads, cpu=cpu_model(),
            settings=str(dict(settings, block=block)))
        print(f"reference block {block}: cycles {rep.cycles}, col_cycles {list(map(int, rep.col_cycles))}, "
              f"max rel residual {np.max(rep.rel_residual):.3e}, converged {rep.all_converged()}, "
              f"setup {setup_s:.1f} s, solve {solve_s:.1f} s ({solve_s / max(rep.cycles, 1):.3f} s/cycle) "
              f"on {args.threads} threads ({cpu_model()}) -> {out}", flush=True)


if __name__ == "__main__":
    main()
