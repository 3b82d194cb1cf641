"""GPU tier: slab decomposition along the slow axis.

Parts are cut on the slow axis; every part computes its own planes and reads
the neighbour faces through the global layout (on several GPUs, peer memory
over NVLink). On this one-GPU tier the parts are separate streams on one GPU,
ordered only by the slab events, which exercises the same partitioning and
synchronisation. A cycle does the same arithmetic per element whatever the
partition, so slab cycles must equal the single-stream cycle BITWISE; a slab
FGMRES solve differs only in the grouping of its Gram partial sums."""
import numpy as np
import pytest

from hzt_util import rel_err
from paper_1607_00968_b200 import configs

pytestmark = pytest.mark.gpu
hz = pytest.importorskip("paper_1607_00968_b200")


def _cfg3d():
    return configs.config3(nlevels=3, n=(65, 65, 33), sgrid=2, layer=8)


def _solver(cfg, precision="c128", kind="V", nlevels=None):
    P = hz.HelmholtzProblem.from_config(cfg)
    o = hz.HelmholtzSolveOptions.from_config(cfg)
    o.method = "MgFgmres"
    o.cycle = hz.CycleSpec(kind)
    o.precond_precision = precision
    if nlevels:
        o.nlevels = nlevels
    return hz.HelmholtzSolver(P, o)


@pytest.mark.parametrize("precision", ["c128", "c64"])
@pytest.mark.parametrize("kind", ["V", "W"])
def test_slab_cycle_3d_bitwise_equals_single_domain(precision, kind):
    cfg = _cfg3d()
    S = _solver(cfg, precision, kind)
    b = configs.random_block(cfg.num_nodes, 8, seed=11)
    x1 = S.cycle(b)
    for parts in (2, 4, 8):
        S.set_slabs(parts)
        xs = S.cycle(b)
        assert np.array_equal(xs, x1), f"{parts} parts"
    S.set_slabs(1)
    assert np.array_equal(S.cycle(b), x1)


def test_slab_cycle_2d_bitwise_equals_single_domain():
    cfg = configs.config1(nlevels=4, nx=129, k=4)
    S = _solver(cfg, "c128", "W", nlevels=4)
    b = configs.random_block(cfg.num_nodes, 4, seed=3)
    x1 = S.cycle(b)
    # the single-domain 2D cycle runs the fused fine-level visit (fused.cu),
    # slab mode the unfused kernels: c128 agrees to the last bits (nvcc's FMA
    # contraction differs between the two kernels), the slab runs bitwise
    xs = []
    for parts in (2, 3, 4):
        S.set_slabs(parts)
        xs.append(S.cycle(b))
        assert rel_err(xs[-1], x1) <= 1e-13, f"{parts} parts"
        assert np.array_equal(xs[-1], xs[0]), f"{parts} parts"


def test_slab_info_cuts_follow_coarsening():
    cfg = _cfg3d()
    S = _solver(cfg)
    S.set_slabs(4)
    P, agg, planes = S.slab_info()
    assert P == 4
    assert planes.shape == (3, 5)
    assert list(planes[0]) == [0, 8, 16, 24, 33]
    assert list(planes[1]) == [0, 4, 8, 12, 17]
    assert list(planes[2]) == [0, 2, 4, 6, 9]
    assert agg == 2  # the coarsest level is solved on part 0
    S.set_slabs(8)
    P, agg, planes = S.slab_info()
    assert list(planes[0]) == [0, 4, 8, 12, 16, 20, 24, 28, 33]
    assert agg == 2


@pytest.mark.parametrize("precision", ["c128", "c64"])
def test_slab_fgmres_solve_matches_single_domain_and_reference(ref, precision):
    cfg = _cfg3d()
    S = _solver(cfg, precision)
    B = cfg.rhs_block()
    X1, r1 = S.solve_block(B)
    S.set_slabs(4)
    X4, r4 = S.solve_block(B)
    assert r1.all_converged() and r4.all_converged()
    assert abs(r4.cycles - r1.cycles) <= 1
    assert np.all(r4.rel_residual <= 1e-6)
    for j in range(B.shape[1]):
        assert rel_err(X4[:, j], X1[:, j]) <= 1e-6
    R = ref.RefProblem.from_config(cfg)
    H = ref.RefHierarchy(R, 3, cfg.shift)
    Xr, rr = ref.krylov_solve(R, H, B, method="fgmres", kind="V", restart=cfg.restart, tol=1e-6,
                              max_cycles=cfg.max_cycles)
    for j in range(B.shape[1]):
        assert rel_err(X4[:, j], Xr[:, j]) <= 1e-5


def test_slab_device_tensor_solve():
    import torch
    cfg = _cfg3d()
    S = _solver(cfg, "c64")
    S.set_slabs(2)
    B = cfg.rhs_block()
    Xh, rh = S.solve_block(B)
    Xd, rd = S.solve_block(torch.from_numpy(B).cuda())
    assert rh.cycles == rd.cycles
    assert np.array_equal(Xh, Xd.cpu().numpy())


def test_slab_mode_validation():
    cfg = _cfg3d()
    P = hz.HelmholtzProblem.from_config(cfg)
    bic = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions(method="MgBicgstab", nlevels=3))
    with pytest.raises(hz.ValidationError):
        bic.set_slabs(2)
    kc = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions(method="MgFgmresK", nlevels=3))
    with pytest.raises(hz.ValidationError):
        kc.set_slabs(2)
    S = _solver(cfg)
    with pytest.raises(hz.ValidationError):
        S.set_slabs(17)  # fewer than 2 fine planes per part
    with pytest.raises(hz.ValidationError):
        S.set_slabs(2, devices=[0, 99])


VMM_CYCLE = (
    "import sys; sys.path.insert(0, '.'); import numpy as np\n"
    "sys.path.insert(0, 'tests'); from test_gpu_slabs import _cfg3d, _solver\n"
    "import paper_1607_00968_b200 as hz; from paper_1607_00968_b200 import configs, _native\n"
    "cfg = _cfg3d(); S = _solver(cfg, sys.argv[2], 'V')\n"
    "b = configs.random_block(cfg.num_nodes, 8, seed=11)\n"
    "x1 = S.cycle(b); n0 = _native.lib().hz_slab_vmm_chunks()\n"
    "S.set_slabs(int(sys.argv[3])); xs = S.cycle(b)\n"
    "X, rep = S.solve_block(cfg.rhs_block())\n"
    "np.savez(sys.argv[1], x1=x1, xs=xs, chunks=_native.lib().hz_slab_vmm_chunks() - n0, conv=rep.all_converged())\n")


@pytest.mark.parametrize("precision,parts", [("c128", 2), ("c64", 4)])
def test_slab_vmm_spanning_vectors_on_one_device(tmp_path, precision, parts):
    """HZ_SLAB_VMM=1: the spanning level vectors are built the multi-GPU way
    (one cuMemCreate chunk per part, cut at the page granularity and mapped
    into one reservation, cuMemSetAccess) with every part on this GPU; the
    slab cycle still equals the single-domain cycle bitwise and the slab
    solve converges. Only the cross-GPU peer reads stay unexercised."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "v.npz")
    env = dict(os.environ, HZ_SLAB_VMM="1")
    r = subprocess.run([sys.executable, "-c", VMM_CYCLE, out, precision, str(parts)], cwd=root, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = np.load(out)
    assert int(d["chunks"]) >= parts  # the VMM path ran (one chunk per part and spanning vector)
    assert np.array_equal(d["xs"], d["x1"])
    assert bool(d["conv"])
