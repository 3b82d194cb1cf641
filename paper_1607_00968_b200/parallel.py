"""Multi-GPU execution of the multi-RHS solve.

One process per GPU (torch.distributed; NCCL on the GPU box, gloo in the CPU
tests). Sources shard naturally: every rank owns a disjoint set of sources
and runs its own independent block solve -- the data path has no collective.
The only exchange is the FWI gradient / misfit sum over sources, which the
reference leaves to its (absent) inversion layer: each rank
accumulates Re(-w^2 (1 - i gamma/w) u_s lambda_s) over its sources
(fwi_sensitivity_output, src/helmholtz_solver.cpp:103-111) and one
all_reduce(SUM) combines the ranks.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, Optional, Sequence

import numpy as np


def shard_sources(nsrc: int, rank: int, world: int) -> np.ndarray:
    """Strided ownership: rank r solves sources r, r + world, ... (balanced to
    within one source; identical blocks per rank when world divides nsrc)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    return np.arange(rank, nsrc, world, dtype=np.int64)


def block_of(sources: Sequence[int], rank: int, world: int) -> np.ndarray:
    return np.asarray(sources, dtype=np.int64)[shard_sources(len(sources), rank, world)]


def allreduce_sum(t, group=None):
    """In-place SUM over ranks of a torch tensor (NCCL or gloo); identity
    without an initialised process group."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def allreduce_max(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def torchrun_argv(nproc: int, script: str, args: Sequence[str], port: Optional[int] = None) -> list:
    """The single-node launch the driver uses for N > 1 (one process per GPU,
    rendezvous on 127.0.0.1): python -m torch.distributed.run ... script args."""
    import sys
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={int(nproc)}",
            "--master-addr", "127.0.0.1", "--master-port", str(port or free_port()), script, *args]


def time_steps(step: Callable[[int], None], steps: int, barrier: Callable[[], None],
               start: Callable[[], None], stop: Callable[[], float]) -> float:
    """Time exactly `steps` calls of step(i), bracketed by barrier() on both
    sides (barrier = process-group barrier + device synchronize). start() /
    stop() are the rank-local clock (CUDA events on the launching stream in
    bench.py); stop() runs after the closing barrier and returns the
    elapsed milliseconds of this rank."""
    barrier()
    start()
    for i in range(steps):
        step(i)
    barrier()
    return float(stop())


def whole_job_rate(units_per_rank_step: float, steps: int, t_ms_local: float, device=None):
    """Whole-job throughput over all ranks: the max over ranks of the timed
    region (the slowest rank ends the job) and value = units all ranks
    processed / that time. Returns (value per second, max ms). Identity
    reduction without an initialised process group."""
    import torch.distributed as dist
    world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    t_ms = allreduce_max(t_ms_local, device=device)
    return world * units_per_rank_step * steps / (t_ms / 1e3), t_ms


@dataclasses.dataclass
class GradientResult:
    gradient: object        # [n] float64 (torch tensor on the rank's device)
    misfit: float           # 0.5 * sum_s ||P^T u_s - d_s||^2 over ALL ranks
    local_sources: np.ndarray
    forward_cycles: int
    adjoint_cycles: int


def fwi_gradient(problem, solver, source_nodes: Sequence[int], receivers,
                 d_obs_fn: Callable[[np.ndarray], np.ndarray], rank: int = 0, world: int = 1,
                 device: Optional[str] = None) -> GradientResult:
    """Sharded FWI gradient for one frequency.

    Rank `rank` solves the forward block U = A^{-1} Q for its sources, samples
    the receivers (SamplingOperator::sample, inc/acquisition.hpp:40-51), forms
    the residuals r_s = P^T u_s - d_s and accumulates sum_s J_s^T r_s with ONE
    adjoint block solve (fwi_jacobian_transpose_vec,
    src/helmholtz_solver.cpp:127-139: lambda = A^{-1} P conj(r),
    g += Re(-w^2 (1 - i gamma/w) u lambda)), then all-reduces gradient and
    misfit. `receivers` is a SamplingOperator or an array of receiver grid
    nodes (unit weights). d_obs_fn(local_source_ids) -> [n_rec, k_local]
    complex observed data.
    """
    import torch
    from . import SamplingOperator, fwi_jacobian_transpose_vec

    dev = device or f"cuda:{problem.device}"
    if isinstance(receivers, SamplingOperator):
        Ps = receivers
    else:
        nodes = np.asarray(receivers, dtype=np.int64)
        n0, n1 = problem.n[0], problem.n[1]
        xyz = np.stack([(nodes % n0) * problem.h[0], ((nodes // n0) % n1) * problem.h[1],
                        (nodes // (n0 * n1)) * problem.h[2]], axis=1).astype(np.float64)
        Ps = SamplingOperator(problem, xyz)
    mine = shard_sources(len(source_nodes), rank, world)
    src = np.asarray(source_nodes, dtype=np.int64)[mine]
    n = problem.num_nodes
    k = len(src)
    g = torch.zeros(n, dtype=torch.float64, device=dev)
    misfit = torch.zeros(1, dtype=torch.float64, device=dev)
    fcyc = acyc = 0
    if k > 0:
        Q = torch.zeros((n, k), dtype=torch.complex128, device=dev)
        Q[torch.as_tensor(src, device=dev), torch.arange(k, device=dev)] = 1.0
        U, rep_f = solver.solve_block(Q)
        d = torch.as_tensor(d_obs_fn(mine), dtype=torch.complex128, device=dev).reshape(Ps.num_receivers, k)
        r = Ps.sample(U) - d
        misfit += 0.5 * torch.sum(torch.abs(r) ** 2)
        reps = []
        fwi_jacobian_transpose_vec(solver, U, Ps, r, g=g, report=reps)
        fcyc, acyc = rep_f.cycles, reps[0].cycles
    allreduce_sum(g)
    allreduce_sum(misfit)
    return GradientResult(g, float(misfit.item()), mine, fcyc, acyc)


@dataclasses.dataclass
class MultiGradientResult:
    gradient: object              # [n] float64: sum over frequencies (and ranks)
    misfit: float                 # sum over frequencies of the per-frequency misfits
    per_frequency: list           # [GradientResult-like (gradient, misfit, cycles)] per frequency
    local_sources: np.ndarray


def fwi_gradient_multi(problems, solvers, source_nodes: Sequence[int], receivers,
                       d_obs_fn: Callable[[int, np.ndarray], np.ndarray], rank: int = 0, world: int = 1,
                       device: Optional[str] = None) -> MultiGradientResult:
    """Multi-frequency FWI gradient: the misfit of one
    frequency-continuation stage is the sum over its frequencies (PAPER.md
    Algorithm 1 uses the data of omega_1..omega_k), so its gradient is the sum
    of the per-frequency gradients of fwi_gradient. All frequencies' forward
    block solves run as ONE concurrent batch (hz_solve_blocks_multi: one
    hierarchy / stream per frequency on this GPU), then their adjoint solves
    run concurrently the same way; per-frequency gradients are summed in
    frequency order and all-reduced once. d_obs_fn(f, local_source_ids) ->
    [n_rec, k_local] observed data of frequency f."""
    import torch
    from concurrent.futures import ThreadPoolExecutor
    from . import SamplingOperator, fwi_jacobian_transpose_vec, solve_blocks_multi

    nf = len(solvers)
    if len(problems) != nf or nf == 0:
        raise ValueError("fwi_gradient_multi: one problem per solver, at least one frequency")
    P0 = problems[0]
    dev = device or f"cuda:{P0.device}"
    samplers = []
    for P in problems:
        if isinstance(receivers, SamplingOperator):
            samplers.append(receivers)
            continue
        nodes = np.asarray(receivers, dtype=np.int64)
        n0, n1 = P.n[0], P.n[1]
        xyz = np.stack([(nodes % n0) * P.h[0], ((nodes // n0) % n1) * P.h[1],
                        (nodes // (n0 * n1)) * P.h[2]], axis=1).astype(np.float64)
        samplers.append(SamplingOperator(P, xyz))
    mine = shard_sources(len(source_nodes), rank, world)
    src = np.asarray(source_nodes, dtype=np.int64)[mine]
    n = P0.num_nodes
    k = len(src)
    g_f = [torch.zeros(n, dtype=torch.float64, device=dev) for _ in range(nf)]
    mis_f = [0.0] * nf
    cyc = [(0, 0)] * nf
    if k > 0:
        Q = torch.zeros((n, k), dtype=torch.complex128, device=dev)
        Q[torch.as_tensor(src, device=dev), torch.arange(k, device=dev)] = 1.0
        Us, reps_f = solve_blocks_multi(solvers, [Q] * nf)
        Rs = []
        for f in range(nf):
            d = torch.as_tensor(d_obs_fn(f, mine), dtype=torch.complex128, device=dev)
            r = samplers[f].sample(Us[f]) - d.reshape(samplers[f].num_receivers, k)
            mis_f[f] = float(0.5 * torch.sum(torch.abs(r) ** 2).item())
            Rs.append(r)
        torch.cuda.synchronize()

        def adjoint(f):
            reps = []
            fwi_jacobian_transpose_vec(solvers[f], Us[f], samplers[f], Rs[f], g=g_f[f], report=reps)
            return reps[0].cycles

        with ThreadPoolExecutor(max_workers=nf) as ex:  # ctypes releases the GIL: solves overlap
            acyc = list(ex.map(adjoint, range(nf)))
        cyc = [(reps_f[f].cycles, acyc[f]) for f in range(nf)]
    g = torch.zeros(n, dtype=torch.float64, device=dev)
    for f in range(nf):  # fixed frequency order
        g += g_f[f]
    misfit = torch.tensor([sum(mis_f)], dtype=torch.float64, device=dev)
    allreduce_sum(g)
    allreduce_sum(misfit)
    per = [{"misfit_local": mis_f[f], "forward_cycles": cyc[f][0], "adjoint_cycles": cyc[f][1]} for f in range(nf)]
    return MultiGradientResult(g, float(misfit.item()), per, mine)


def frequency_continuation(m0, omegas: Sequence[float], stage_solve: Callable, start: int = 1):
    """Frequency continuation, PAPER.md:96-107 (Algorithm 1): with
    omega_1 < ... < omega_nf, stage k solves the inversion with the data of
    omega_1..omega_k starting from the previous stage's model:
        m_k = stage_solve(m_{k-1}, omegas[:k]).
    stage_solve is the caller's inner inversion (e.g. gradient / Gauss-Newton
    steps built on MultiFrequencySolver and fwi_gradient_multi; the
    reference's inversion layer itself is absent). Returns
    the list of stage models [m_start, ..., m_nf]."""
    om = [float(w) for w in omegas]
    if any(b <= a for a, b in zip(om, om[1:])):
        raise ValueError("frequency_continuation: frequencies must be increasing")
    models = [m0]
    m = m0
    for kk in range(start, len(om) + 1):
        m = stage_solve(m, om[:kk])
        models.append(m)
    return models
