"""CPU tier, world_size 2 over gloo: the source sharding and the gradient /
misfit all-reduce of paper_1607_00968_b200.parallel (the N > 1 path of
SURVEY §8e). Per-rank partial gradients come from the numpy restatement of
the reference (oracle/port.py, dense direct solves on a small grid), so the
test exercises exactly the host-side exchange the GPU ranks perform."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1607_00968_b200 import configs, parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    from oracle import port
    cfg = configs.small_problem(2, (17, 17, 1), seed=3, layer=3)
    P = port.Problem.from_config(cfg)
    A = P.to_csr(0.0).toarray()
    nsrc = 6
    src = np.array([2 + 2 * s for s in range(nsrc)]) + 17 * 1
    rec = np.arange(17) + 17 * 2
    return cfg, P, A, src, rec


def _local_partials(rank, world):
    cfg, P, A, src, rec = _problem()
    mine = parallel.shard_sources(len(src), rank, world)
    n = P.num_nodes
    g = np.zeros(n)
    misfit = 0.0
    for s in mine:
        q = np.zeros(n, complex)
        q[src[s]] = 1.0
        u = np.linalg.solve(A, q)
        d = 0.9 * u[rec]  # synthetic "observed" data
        r = u[rec] - d
        misfit += 0.5 * np.sum(np.abs(r) ** 2)
        rhs = np.zeros(n, complex)
        rhs[rec] = np.conj(r)
        lam = np.linalg.solve(A, rhs)
        g += P.sensitivity_output(u, lam)
    return g, misfit


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g, m = _local_partials(rank, world)
    gt = torch.from_numpy(g)
    mt = torch.tensor([m], dtype=torch.float64)
    parallel.allreduce_sum(gt)
    parallel.allreduce_sum(mt)
    mx = parallel.allreduce_max(float(rank + 1))
    out[rank] = (gt.numpy().copy(), float(mt.item()), mx)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_sources_partition():
    for nsrc in (1, 5, 8, 64):
        for world in (1, 2, 3, 8):
            parts = [parallel.shard_sources(nsrc, r, world) for r in range(world)]
            allp = np.sort(np.concatenate(parts))
            assert np.array_equal(allp, np.arange(nsrc))
            sizes = [len(p) for p in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        parallel.shard_sources(4, 2, 2)


def test_gradient_allreduce_world2_matches_serial_sum():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    g_serial, m_serial = _local_partials(0, 1)
    for r in range(world):
        g, m, mx = out[r]
        assert np.allclose(g, g_serial, rtol=1e-12, atol=1e-14 * np.abs(g_serial).max())
        assert abs(m - m_serial) <= 1e-12 * abs(m_serial)
        assert mx == world
    # every rank holds the identical reduced gradient
    assert np.array_equal(out[0][0], out[1][0])


def test_allreduce_identity_without_process_group():
    t = torch.arange(4, dtype=torch.float64)
    assert torch.equal(parallel.allreduce_sum(t.clone()), t)
    assert parallel.allreduce_max(3.0) == 3.0


def _timing_worker(rank, world, port, out):
    """Each rank times 3 steps whose length depends on the rank; the job
    time must be the slowest rank's and the rate count every rank's units."""
    import time as _t
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    calls = []
    clock = {}

    def step(i):
        calls.append(i)
        _t.sleep(0.02 * (rank + 1))

    def start():
        clock["t0"] = _t.perf_counter()

    def stop():
        return 1e3 * (_t.perf_counter() - clock["t0"])

    t_local = parallel.time_steps(step, 3, dist.barrier, start, stop)
    value, t_max = parallel.whole_job_rate(8, 3, t_local)
    out[rank] = (calls, t_local, value, t_max)
    dist.barrier()
    dist.destroy_process_group()


def test_bench_timing_world2_max_over_ranks():
    """bench.py's timed region (parallel.time_steps + whole_job_rate): exactly
    K steps per rank between barriers, max over ranks, whole-job value."""
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_timing_worker, args=(world, port, out), nprocs=world, join=True)
    t_max = max(out[r][1] for r in range(world))
    for r in range(world):
        calls, t_local, value, tm = out[r]
        assert calls == [0, 1, 2]
        assert tm == t_max  # every rank sees the same reduced time
        assert value == pytest.approx(world * 8 * 3 / (t_max / 1e3))
    # the closing barrier makes the fast rank wait for the slow one
    assert out[0][1] >= 0.9 * 3 * 0.02 * world


def test_torchrun_argv_single_node_loopback():
    argv = parallel.torchrun_argv(4, "bench.py", ["--gpus", "4", "--steps", "2"], port=29555)
    assert argv[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in argv
    assert argv[argv.index("--master-addr") + 1] == "127.0.0.1"
    assert argv[-5:] == ["bench.py", "--gpus", "4", "--steps", "2"]
