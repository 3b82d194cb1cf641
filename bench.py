#!/usr/bin/env python
"""Benchmark: Helmholtz right-hand sides solved per second to 1e-6 relative
residual (BASELINE.json metric) on BASELINE config 2 -- 2D 1025x513 layered
model, k = 32 surface sources per GPU, complex128 block FGMRES with a
complex64 shifted-Laplacian V(2,2) multigrid preconditioner; the 32 sources
are solved as 4 concurrent independent blocks of 8 (hz_options.rhs_block).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one block solve of the rank's k right-hand sides from zero to the
tolerance (setup excluded). N > 1 runs one process per GPU
under torchrun (started by the driver, or by this script re-executing itself
through torch.distributed.run when --gpus N > 1 and WORLD_SIZE is unset);
each rank owns its own block of k sources (weak scaling, no data-path
collective); the rank count must equal --gpus. `value` = all ranks' RHS / max-over-ranks device time.

The JSON line also carries: `e2e` (same metric through the C ABI with host
buffers, H2D/D2H inside the timed region), `roofline` (dominant kernel's
algorithmic GB/s from CUDA events in a profiled pass: one RHS block solved
alone, so concurrent kernels do not share each other's event windows),
`kernels` (all kernels), `cpu_baseline` (the reference C++ solver timed on
this host on a bounded sample, rank 0, N = 1), `clocks`, `gpu_launches`.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Helmholtz RHS solved/sec to 1e-6 residual"
UNIT = "RHS/s"

# The BASELINE config-2 solver (config 2 leaves levels / shift / cycle /
# Krylov / RHS blocking unstated): c128 block FGMRES(5) + c64
# shifted-Laplacian V(2,2), 6 levels to a 33x17 coarse grid, shift 0.9,
# damped-Jacobi weight 0.6, the 32 sources solved as 4 independent blocks of
# 8 columns running concurrently (hz_options.rhs_block = 8) -- the fastest
# converging setting of the GPU sweeps (DESIGN.md §5,
# profiles/r01_sweep_rhs_block.jsonl). Cycle counts barely depend on the
# block width here (390-430 for blocks of 1-32) while the block Krylov cost
# grows with it (8k^2 flops per row), so 8-column blocks turn the FP64-bound
# Gram/update of a 32-column block into HBM-bound ones. At shift 0.5 /
# w_J 0.8 the V-cycle stalls in the reference oracle and on the GPU alike.
WORKLOADS = {
    "cfg2": dict(cfg=2, k=32, nlevels=6, shift=0.9, jacobi_weight=0.6, cycle="V", restart=5, tol=1e-6,
                 max_cycles=2000, precond="c64", krylov_block=8, stencil=7),
    # BASELINE config 4's per-GPU shard (--workload cfg4): 3D 257x257x129 with
    # the compact 27-point fine operator, 8 of the 64 surface sources per GPU,
    # c128 FGMRES(5) + c64 W(2,2), 3 levels (4 and 5 levels stall below
    # 1e-2 in 500 cycles with either stencil: profiles/r02_cfg4_levels.txt);
    # W-cycle, shift 0.3, w_J 0.9 from profiles/r02_sweep_cfg4.txt (110 cycles;
    # V(2,2) at shift 0.5 / w_J 0.8 with FGMRES(10): 179-201 cycles)
    "cfg4": dict(cfg=4, k=8, nlevels=3, shift=0.3, jacobi_weight=0.9, cycle="W", restart=5, tol=1e-6,
                 max_cycles=600, precond="c64", krylov_block=0, stencil=27),
    # config 4's shard with the level count SURVEY §8d assigns it (--workload cfg4_literal): 5 levels, V(2,2); shift
    # 1.0 and Jacobi weight 0.5 (at 0.6-0.8 this hierarchy stalls): 400 cycles, 0.41 of the 3-level W-cycle line
    "cfg4_literal": dict(cfg=4, k=8, nlevels=5, shift=1.0, jacobi_weight=0.5, cycle="V", restart=5, tol=1e-6,
                         max_cycles=900, precond="c64", krylov_block=0, stencil=27),
    # BASELINE config 3 (--workload cfg3): 3D 129x129x65, 7-point operator, the
    # 16 surface sources as 2 concurrent blocks of 8, c128 FGMRES(5) + c64
    # W(2,2), 3 levels (the literal 4 levels stall): the paper's own
    # grid (BASELINE.md Table 1). W-cycle, shift 0.25, w_J 0.9 from the sweeps of
    # profiles/r02_sweep_cfg3.txt (80 cycles, 80.3 RHS/s; V at the same shift
    # 130 cycles, 65.8; V at shift 0.5 / w_J 0.8 155 cycles, 54.8; the
    # reference's own defaults are the W-cycle and shift 0.2). Its reference
    # numbers come from the committed full reference solves at these settings
    # (tests/golden/cfg3_bench_block*.npz, scripts/ref_full_solve.py --bench): the
    # reference's banded-LU setup of the 33x33x17 coarsest grid alone takes
    # minutes on host cores, too long for a bench step.
    "cfg3": dict(cfg=3, k=16, nlevels=3, shift=0.25, jacobi_weight=0.9, cycle="W", restart=5, tol=1e-6,
                 max_cycles=600, precond="c64", krylov_block=8, stencil=7, fixture="cfg3_bench_block"),
    # BASELINE config 3 exactly as stated (--workload cfg3_literal): 4 levels, V(2,2), block FGMRES(10); the shift
    # (1.0) and the Jacobi weight (0.5) are left open by BASELINE -- at w_J 0.6-0.8 this hierarchy stalls
    # (profiles/r02_sweep_literal_levels.txt). 243 cycles: 0.44 of the 3-level W-cycle line's throughput.
    "cfg3_literal": dict(cfg=3, k=16, nlevels=4, shift=1.0, jacobi_weight=0.5, cycle="V", restart=10, tol=1e-6,
                         max_cycles=600, precond="c64", krylov_block=8, stencil=7, fixture="cfg3_literal_block"),
}
WORKLOAD = WORKLOADS["cfg2"]


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        return False

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def rank_sources(cfg, rank, world, k):
    """Weak scaling. Config 2: world*k evenly spaced surface sources, rank r
    owns r, r+world, ... Config 4: the config's 64 sources (8x8 surface grid),
    8 per GPU: rank r owns sources r, r+8, ... (BASELINE configs[3])."""
    import numpy as np
    from paper_1607_00968_b200 import configs
    if WORKLOAD["cfg"] == 4:
        return np.asarray(cfg.source_nodes[rank % 8::8][:k], dtype=np.int64)
    if WORKLOAD["cfg"] == 3:  # every rank solves the config's own 16 sources (replicas: fixed per-GPU work)
        return np.asarray(cfg.source_nodes[:k], dtype=np.int64)
    full = configs.config2(nlevels=WORKLOAD["nlevels"], k=k * world)
    return np.asarray(full.source_nodes[rank::world], dtype=np.int64)


def build_workload(rank, world, k):
    from paper_1607_00968_b200 import configs
    if WORKLOAD["cfg"] == 4:
        cfg = configs.config4(nlevels=WORKLOAD["nlevels"])
    elif WORKLOAD["cfg"] == 3:
        cfg = configs.config3(nlevels=WORKLOAD["nlevels"])
    else:
        cfg = configs.config2(nlevels=WORKLOAD["nlevels"], k=k)
    cfg.source_nodes = rank_sources(cfg, rank, world, k)
    cfg.stencil = WORKLOAD["stencil"]
    cfg.shift = WORKLOAD["shift"]
    cfg.jacobi_weight = WORKLOAD["jacobi_weight"]
    cfg.cycle = WORKLOAD["cycle"]
    cfg.restart = WORKLOAD["restart"]
    cfg.tol = WORKLOAD["tol"]
    cfg.max_cycles = WORKLOAD["max_cycles"]
    cfg.precond_precision = WORKLOAD["precond"]
    cfg.krylov_block = WORKLOAD["krylov_block"]
    return cfg


def config_json(cfg, world, l2_note):
    if WORKLOAD["cfg"] == 4:
        wl = (f"BASELINE config 4 (per-GPU shard): 3D {cfg.n[0]}x{cfg.n[1]}x{cfg.n[2]} thrust-faulted layered model, "
              f"compact {cfg.stencil}-point fine stencil, k={cfg.k} RHS/GPU")
        grid = list(cfg.n)
    elif WORKLOAD["cfg"] == 3:
        wl = (f"BASELINE config 3: 3D {cfg.n[0]}x{cfg.n[1]}x{cfg.n[2]} layered model, 7-point stencil, "
              f"k={cfg.k} RHS/GPU")
        grid = list(cfg.n)
    else:
        wl = f"BASELINE config 2: 2D {cfg.n[0]}x{cfg.n[1]} layered model, k={cfg.k} RHS/GPU"
        grid = list(cfg.n[:2])
    return {"workload": wl, "grid": grid, "rhs_per_gpu": cfg.k, "global_rhs": cfg.k * world,
            "solver": f"block FGMRES({cfg.restart}) + {cfg.cycle}({cfg.pre},{cfg.post}) MG, "
                      f"{cfg.nlevels} levels, shift {cfg.shift}, w_J {cfg.jacobi_weight}",
            "rhs_blocking": (f"{-(-cfg.k // cfg.krylov_block)} independent block solves of {cfg.krylov_block} columns"
                             if 0 < cfg.krylov_block < cfg.k else f"one block of {cfg.k} columns"),
            "precision": "c128 Krylov / c64 preconditioner", "tol": cfg.tol,
            "parallelism": f"rhs-sharded x{world}", "l2": l2_note}


# ---------------------------------------------------------------- reference arm
def ref_cycles_measured():
    """Cycles the REFERENCE solver itself needs to reach 1e-6 on each RHS
    block of this workload: its own block_fgmres run to convergence
    (scripts/ref_full_solve.py -> tests/golden/cfg2_bench_block<b>.npz,
    complex128 preconditioner, the blocking of our arm). Returns
    ({block: cycles}, cpu model of the run)."""
    import numpy as np
    out, cpu = {}, None
    stem = WORKLOAD.get("fixture", "cfg2_bench_block")
    for b in range(8):
        f = os.path.join(ROOT, "tests", "golden", f"{stem}{b}.npz")
        if os.path.exists(f):
            g = np.load(f)
            out[b] = int(g["cycles"])
            cpu = str(g["cpu"])
    return out, cpu


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# GPU cycle count of this workload per 8-column block (mean over the 4
# blocks), the fallback when no reference count was measured for a block
DEFAULT_CYCLES = 391


class ReferenceRunner:
    """The reference C++ solver (oracle/_ref, stock-contraction build) driven
    through its public API -- build_hierarchy + MgHierarchy::cycle +
    block_fgmres -- with all host threads. Setup is done once
    (excluded). The workload's k sources are solved the way
    our arm blocks them: ceil(k/b) independent block_fgmres solves of b
    columns (b = krylov_block; one k-column block when 0). A step is a bounded
    sample of `sample_cycles` FGMRES iterations of one such block (c128
    preconditioner: the reference has no c64 path), extrapolated to full
    solves of all blocks: RHS/s = k / (blocks x s_per_cycle x cycles)."""

    def __init__(self, cfg, threads=None):
        os.environ["HZ_REF_VARIANT"] = "fast"
        from oracle import ref
        self.ref = ref
        self.cfg = cfg
        self.threads = threads or os.cpu_count() or 1
        ref.set_num_threads(self.threads)
        b = cfg.krylov_block if 0 < cfg.krylov_block < cfg.k else cfg.k
        self.block, self.nblocks = b, -(-cfg.k // b)
        self.B = cfg.rhs_block()[:, :b].copy()
        t0 = time.perf_counter()
        self.R = ref.RefProblem.from_config(cfg)
        self.H = ref.RefHierarchy(self.R, cfg.nlevels, cfg.shift)
        self.setup_s = time.perf_counter() - t0

    def step(self, sample_cycles):
        cfg = self.cfg
        t0 = time.perf_counter()
        _, rep = self.ref.krylov_solve(self.R, self.H, self.B, method="fgmres", kind=cfg.cycle,
                                       pre=cfg.pre, post=cfg.post, wj=cfg.jacobi_weight,
                                       restart=cfg.restart, tol=cfg.tol, max_cycles=sample_cycles)
        return (time.perf_counter() - t0) / max(rep.cycles, 1), rep.cycles

    def rhs_per_s(self, per_cycle, total_cycles):
        """total_cycles: preconditioner cycles summed over all blocks"""
        return self.cfg.k / (per_cycle * total_cycles)

    def describe(self, sample_cycles, total_cycles, source):
        cfg = self.cfg
        return (f"{sample_cycles} FGMRES({cfg.restart}) iterations (V-cycle + Arnoldi + LS) per step of one "
                f"{self.block}-column block of the workload ({self.nblocks} blocks) on the reference C++ solver "
                f"(oracle/_ref, {self.threads} threads of {cpu_model()}, c128 preconditioner -- the reference has "
                f"no c64 path), setup excluded; RHS/s = k / (s_per_cycle x {total_cycles:.0f} cycles summed over "
                f"the blocks, {source})")


def ref_total_cycles(nblocks, fallback_per_block):
    """Cycles of a full reference solve of the workload: the measured
    per-block counts, the fallback for blocks never measured."""
    meas, cpu = ref_cycles_measured()
    total = sum(meas.get(b, fallback_per_block) for b in range(nblocks))
    n_meas = sum(1 for b in range(nblocks) if b in meas)
    src = (f"reference-measured cycles for {n_meas}/{nblocks} blocks "
           f"({', '.join(str(meas[b]) for b in range(nblocks) if b in meas)}; "
           f"tests/golden/cfg2_bench_block*.npz, scripts/ref_full_solve.py on {cpu})")
    if n_meas < nblocks:
        src += f", {fallback_per_block:.0f} (GPU count) for the rest"
    return total, src


def reference_sample(cfg, gpu_cycles_per_block, sample_cycles, threads=None):
    run = ReferenceRunner(cfg, threads)
    per_cycle, _ = run.step(sample_cycles)
    total, src = ref_total_cycles(run.nblocks, gpu_cycles_per_block)
    return run.rhs_per_s(per_cycle, total), {"cores": run.threads, "s_per_cycle": per_cycle,
                                             "sample": run.describe(sample_cycles, total, src)}


def fixture_baseline():
    """Config 3: the reference's full solves of the workload's blocks as
    measured when the fixtures were made (scripts/ref_full_solve.py --config 3):
    (RHS/s over the measured blocks, cores, description) or None."""
    import numpy as np
    cfg = build_workload(0, 1, WORKLOAD["k"])
    b = cfg.krylov_block if 0 < cfg.krylov_block < cfg.k else cfg.k
    secs, cyc, cols, cpu, thr = 0.0, [], 0, None, None
    for blk in range(-(-cfg.k // b)):
        f = os.path.join(ROOT, "tests", "golden", f"{WORKLOAD['fixture']}{blk}.npz")
        if not os.path.exists(f):
            continue
        g = np.load(f)
        secs += float(g["solve_s"])
        cyc.append(int(g["cycles"]))
        cols += b
        cpu, thr = str(g["cpu"]), int(g["threads"])
    if not cols:
        return None
    return cols / secs, thr, (f"full reference solves (block_fgmres to 1e-6, c128 preconditioner, {cfg.nlevels} levels with the "
                              f"banded LU of the coarsest grid; setup excluded) of {cols} of the workload's "
                              f"{cfg.k} sources in {b}-column blocks: {', '.join(map(str, cyc))} cycles, {secs:.0f} s "
                              f"on {thr} threads of {cpu}, measured when tests/golden/{WORKLOAD['fixture']}*.npz were "
                              f"generated (scripts/ref_full_solve.py --config 3 --bench / --literal), not re-run here")


def reference_line_from_fixtures(args):
    fb = fixture_baseline()
    if fb is None:
        return {"impl": "reference", "unavailable": "no committed reference solve of this workload"}
    value, cores, sample = fb
    cfg = build_workload(0, 1, WORKLOAD["k"])
    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * cfg.k / value, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "c128", "data": "synthetic (seeded, SURVEY §8d)",
            "config": dict(config_json(cfg, 1, "n/a (CPU)"), precision="c128 Krylov / c128 preconditioner"),
            "impl": "reference", "measured": "recorded (fixture), not re-run",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def run_reference(args):
    ws, rank, local = dist_env()
    if ws > 1 and rank != 0:
        return 0
    if WORKLOAD["cfg"] == 3:
        print(json.dumps(reference_line_from_fixtures(args)), flush=True)
        return 0
    if WORKLOAD["cfg"] != 2:
        print(json.dumps({"impl": "reference", "unavailable": "the reference has no compact 27-point operator "
                          "(src/helmholtz.cpp:45-100 is 5/7-point only)"}), flush=True)
        return 0
    cfg = build_workload(0, 1, WORKLOAD["k"])
    run = ReferenceRunner(cfg)
    if args.ref_cycles:
        total, src = args.ref_cycles * run.nblocks, f"{args.ref_cycles:.0f} cycles per block (--ref-cycles)"
    else:
        total, src = ref_total_cycles(run.nblocks, DEFAULT_CYCLES)
    vals, walls = [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        per_cycle, _ = run.step(args.ref_sample_cycles)
        if i >= args.warmup:
            walls.append(1e3 * (time.perf_counter() - t0))
            vals.append(run.rhs_per_s(per_cycle, total))
    info = {"cores": run.threads, "sample": run.describe(args.ref_sample_cycles, total, src)}
    value = statistics.mean(vals)
    # a step is the bounded sample (ms_per_step = its measured wall time);
    # the full-solve time the value extrapolates to is reported beside it
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": statistics.mean(walls),
            "ms_full_solve_extrapolated": 1e3 * cfg.k / value, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded, SURVEY §8d)",
            "config": dict(config_json(cfg, 1, "n/a (CPU)"), precision="c128 Krylov / c128 preconditioner",
                           cpu=cpu_model()),
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": info["cores"], "kind": "reference",
                             "sample": info["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our arm
def block_cycles(rep, cfg):
    """Mean over the RHS blocks of each block solve's cycle count (the
    slowest column of the block); the cycle count of the solve when unblocked."""
    import numpy as np
    b = cfg.krylov_block
    if not 0 < b < cfg.k:
        return float(rep.cycles)
    cc = np.asarray(rep.col_cycles)
    return float(np.mean([cc[i:i + b].max() for i in range(0, cfg.k, b)]))


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_1607_00968_b200 as hz
    from paper_1607_00968_b200 import parallel

    ws, rank, local = dist_env()
    if ws != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={ws}")
    torch.cuda.set_device(local)
    if torch.cuda.device_count() < 1:
        raise SystemExit("bench: no CUDA device")
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = build_workload(rank, ws, WORKLOAD["k"])
    n, k = cfg.num_nodes, cfg.k
    t0 = time.perf_counter()
    P = hz.HelmholtzProblem.from_config(cfg, device=local)
    S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg))
    setup_s = time.perf_counter() - t0
    B_host = cfg.rhs_block()
    Bd = torch.from_numpy(B_host).to(f"cuda:{local}")
    Xd = torch.empty_like(Bd)

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up (also fixes the cycle count of the workload)
    rep = None
    for _ in range(args.warmup):
        _, rep = S.solve_block(Bd, out=Xd)
    assert rep is not None and rep.all_converged(), f"warm-up solve did not converge: {rep}"
    # ---- timed region: device-resident inputs (inputs > L2: 269 MB block)
    cycles = []
    launches0 = hz.kernel_launch_count()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    def step(_i):
        _, r = S.solve_block(Bd, out=Xd)  # library stream, ordered after `stream`; synchronised on return
        cycles.append(block_cycles(r, cfg))
        if not r.all_converged():
            raise RuntimeError(f"solve did not converge: {r.rel_residual}")

    def ev_stop():
        ev1.record(stream)
        ev1.synchronize()
        return ev0.elapsed_time(ev1)

    with ClockSampler(local) as clk:
        t_local = parallel.time_steps(step, args.steps, barrier, lambda: ev0.record(stream), ev_stop)
    launches = hz.kernel_launch_count() - launches0
    value, t_ms = parallel.whole_job_rate(k, args.steps, t_local, device=f"cuda:{local}")
    # ---- e2e: the public C ABI with pinned host buffers (H2D + D2H per step)
    Bp = torch.from_numpy(B_host).pin_memory()
    Xp = torch.empty_like(Bp).pin_memory()
    Bn, Xn = Bp.numpy(), Xp.numpy()
    wall = {}

    def e2e_step(_i):
        S.solve_block(Bn, out=Xn)

    def wall_stop():
        return 1e3 * (time.perf_counter() - wall["t0"])

    e2e_ms_local = parallel.time_steps(e2e_step, args.steps, barrier,
                                       lambda: wall.__setitem__("t0", time.perf_counter()), wall_stop)
    e2e, _ = parallel.whole_job_rate(k, args.steps, e2e_ms_local, device=f"cuda:{local}")
    # ---- profiled pass (same steps) for the per-kernel roofline
    # (blocked workload: one block solved alone -- the concurrent blocks run
    # the same kernels at the same shapes, but overlapping kernels would
    # share HBM inside each other's event windows)
    b = cfg.krylov_block if 0 < cfg.krylov_block < k else k
    Sp = S if b == k else hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg, rhs_block=0))
    Bp1 = Bd[:, :b].contiguous()
    Sp.solve_block(Bp1)
    with hz.kernel_profile() as prof:
        for _ in range(max(1, min(args.steps, 3))):
            Sp.solve_block(Bp1)
    kern = prof.result
    peak, peak_kind = peaks()
    table = {}
    for name, r in kern.items():
        avg_ms = r["ms"] / max(r["count"], 1)
        gbs = r["bytes"] / (r["ms"] / 1e3) / 1e9 if r["ms"] > 0 else 0.0
        table[name] = {"launches": r["count"], "avg_us": round(1e3 * avg_ms, 3),
                       "share": 0.0, "gbs": round(gbs, 1), "frac": round(gbs / peak, 3)}
    total_ms = sum(r["ms"] for r in kern.values()) or 1.0
    for name, r in kern.items():
        table[name]["share"] = round(r["ms"] / total_ms, 4)
    # roofline of the dominant kernel (largest share of the step): the FP64
    # tall-skinny Gram / block update at k = 32 are bound by the FP64 tensor
    # pipe (DMMA; 8 flop/B > the FP64 ridge), the grid kernels by HBM
    traffic_tab = {}
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        try:
            traffic_tab = json.load(open(tfile))
        except Exception:
            traffic_tab = {}
    try:
        fp64_peak, fp64_src = hz.measure_fp64_peak(), "measured live (hz_measure_fp64_peak, DMMA m8n8k4)"
    except Exception:
        fp64_peak, fp64_src = 37.1, "fallback: scripts/micro/fp64_peak.cu measurement on this pool"

    def roof(name):
        r = kern[name]
        secs = r["ms"] / 1e3
        gbs = r["bytes"] / secs / 1e9
        per = {"kernel": name, "launches": r["count"],
               "algorithmic_bytes_per_launch": r["bytes"] / r["count"],
               "hbm_gbs": round(gbs, 1), "hbm_frac": round(gbs / peak, 4),
               "traffic": None, "traffic_note": None}
        tt = traffic_tab.get(name) or {}
        if tt.get("dram_over_algorithmic"):
            # ncu DRAM bytes / algorithmic bytes of the captured launches,
            # applied to this kernel's mean algorithmic bytes per launch
            per["traffic"] = round(tt["dram_over_algorithmic"] * r["bytes"] / r["count"])
            per["traffic_note"] = (f"ncu dram__bytes_read+write = {tt['dram_over_algorithmic']:.3f} x algorithmic "
                                   f"over {tt.get('launches_captured')} captured launches ({tt.get('note', '')})")
        # the binding roofline: FP64 tensor pipe when the kernel's flops at
        # the DMMA peak take longer than its bytes at the HBM peak (the
        # 32-column Gram / update), else HBM (8-column blocks, stencils)
        # (only the complex128 Gram / update kernels run on the DMMA pipe; the coarse solves are FP32 / FP64 FMA
        # kernels whose flops are reported beside their HBM fraction)
        flops_bound = (name.startswith("multi_") and r.get("flops", 0) > 0 and
                       0.75 * r["flops"] / (fp64_peak * 1e12) > r["bytes"] / (peak * 1e9))
        if flops_bound:
            tf = r["flops"] / secs / 1e12
            per.update({"bound": "tensor", "achieved": round(tf, 2), "peak": round(fp64_peak, 2),
                        "unit": "TFLOP/s", "frac": round(tf / fp64_peak, 4), "peak_source": fp64_src,
                        "flops_note": "algorithmic complex flops 8nk^2 per block; issued real flops are 3/4 of "
                                      "that (3-multiplication complex product)",
                        "issued_frac": round(0.75 * tf / fp64_peak, 4)})
        else:
            per.update({"bound": "hbm", "achieved": round(gbs, 1), "peak": peak, "unit": "GB/s",
                        "frac": round(gbs / peak, 4), "peak_source": peak_kind})
            if r.get("flops", 0) > 0:
                per["fp64_tflops" if name.endswith("c128") else "fp32_tflops"] = round(r["flops"] / secs / 1e12, 2)
        return per

    dom = max(kern, key=lambda n_: kern[n_]["ms"])
    roofline = roof(dom)
    roofline["share"] = table[dom]["share"]
    if dom.startswith("coarse_bt"):
        roofline["note"] = ("the event profile times the two-sided plane-solver chain (~130 dependent launches) on its own; inside "
                            "the graph-replayed W-cycle a solve takes 1.83 ms on config 4 (4.7 GB of factors, 2.6 TB/s; timing-only "
                            "cut in profiles/r02_bt_res_ab.txt, DESIGN.md section 3)")
    stencil = [n_ for n_ in kern if n_.startswith(("jacobi", "residual", "apply", "restrict", "prolong", "fused"))]
    roof_st = None
    if stencil:
        dst = max(stencil, key=lambda n_: kern[n_]["ms"])
        roof_st = roof(dst)
        roof_st["share"] = table[dst]["share"]
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic (seeded, SURVEY §8d; random-free point sources)",
            "config": config_json(cfg, ws, f"inputs larger than L2 ({B_host.nbytes / 1e6:.0f} MB block, Krylov bases "
                                           f"{(2 * cfg.restart + 1) * B_host.nbytes / 1e9:.1f} GB)"),
            "cycles_per_solve": statistics.mean(cycles), "setup_s": round(setup_s, 3),
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": int(B_host.nbytes),
                    "d2h_bytes_per_step": int(B_host.nbytes)},
            "roofline": roofline, "roofline_stencil": roof_st, "kernels": table, "gpu_launches": int(launches),
            "clocks": clk.summary()}
    if rank == 0 and ws == 1 and WORKLOAD["cfg"] == 3:
        fb = fixture_baseline()
        line["cpu_baseline"] = ({"value": fb[0], "unit": UNIT, "cores": fb[1], "kind": "reference", "sample": fb[2]}
                                if fb else {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                                            "sample": "unavailable: no committed reference solve"})
    elif rank == 0 and ws == 1 and WORKLOAD["cfg"] != 2:
        line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                                "sample": "unavailable: the reference has no compact 27-point operator"}
    elif rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            v, info = reference_sample(cfg, statistics.mean(cycles), sample_cycles=args.cpu_sample_cycles)
            info["sample"] += f"; host {cpu_model()}"
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": info["cores"], "kind": "reference",
                                    "sample": info["sample"]}
        except Exception as e:  # the baseline is reported, never required
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg2",
                    help="cfg2 (default, the BASELINE metric's config), cfg3 (config 3, the paper's grid) or cfg4 (config 4's per-GPU shard)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-sample-cycles", type=int, default=2,
                    help="FGMRES iterations per reference step (bounded CPU sample)")
    ap.add_argument("--cpu-sample-cycles", type=int, default=5,
                    help="FGMRES iterations of the cpu_baseline sample in our arm (one restart)")
    ap.add_argument("--ref-cycles", type=float, default=None,
                    help="per-block cycle count to extrapolate the reference sample to (default: the reference's "
                         "own measured counts, tests/golden/cfg2_bench_block*.npz)")
    args = ap.parse_args()
    global WORKLOAD
    WORKLOAD = WORKLOADS[args.workload]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # launched directly with --gpus N: become the torchrun launch the
        # driver uses (one process per GPU, 127.0.0.1 rendezvous)
        from paper_1607_00968_b200 import parallel
        argv = parallel.torchrun_argv(args.gpus, os.path.abspath(__file__), sys.argv[1:])
        os.execv(argv[0], argv)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
