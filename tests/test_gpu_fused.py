"""GPU tier: the fused finest-level V(2,2) visit (csrc/fused.cu: pre-smoothing
+ residual + restriction in one streaming kernel, prolongation + both
post-smoothing sweeps in another) against the unfused kernel sequence
(HZ_FUSED_VCYCLE=0) -- bitwise -- and, through the c128 cycle, against the
reference oracle's MgHierarchy::cycle (src/multigrid.cpp:162-199)."""
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

from hzt_util import rel_err
from paper_1607_00968_b200 import configs

pytestmark = pytest.mark.gpu
hz = pytest.importorskip("paper_1607_00968_b200")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CYCLE = (
    "import sys; sys.path.insert(0, '.'); import numpy as np\n"
    "import paper_1607_00968_b200 as hz; from paper_1607_00968_b200 import configs\n"
    "nx, nz, k, nl, prec, kind = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), sys.argv[6], sys.argv[7]\n"
    "cfg = configs.config2(nlevels=nl, k=k, nx=nx, nz=nz); cfg.precond_precision = prec; cfg.cycle = kind\n"
    "S = hz.HelmholtzSolver(hz.HelmholtzProblem.from_config(cfg), hz.HelmholtzSolveOptions.from_config(cfg))\n"
    "b = configs.random_block(cfg.num_nodes, k, seed=11)\n"
    "x1 = S.cycle(b); x2 = S.cycle(b)\n"
    "assert np.array_equal(x1, x2), 'cycle not deterministic'\n"
    "np.save(sys.argv[1], x1)\n")


def _run(code, path, flag, *args, **extra_env):
    env = dict(os.environ, HZ_FUSED_VCYCLE=flag, **extra_env)
    r = subprocess.run([sys.executable, "-c", code, path, *map(str, args)], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(path)


# (nx, nz, k, levels, precision, cycle): odd sizes that are not multiples of
# the strip width (122 / 124 fine nodes) or the row chunks (32), grids
# narrower than one strip, and the full config-2 geometry (9 strips x 17 chunks)
CASES = [
    (257, 129, 8, 4, "c64", "V"),
    (297, 161, 4, 3, "c64", "W"),
    (49, 41, 8, 3, "c64", "V"),
    (1025, 513, 8, 5, "c64", "V"),
    (129, 65, 32, 3, "c64", "V"),
    (257, 129, 4, 4, "c128", "V"),
    (297, 161, 2, 3, "c128", "W"),
    (65, 41, 6, 3, "c128", "V"),
    # k = 8 bulk-copy kernels: odd widths / heights against strips of 56 / 60
    # owned nodes and the row chunks, a grid narrower than one strip
    (301, 97, 8, 3, "c64", "W"),
    (65, 49, 8, 3, "c64", "V"),
    (121, 233, 8, 4, "c64", "V"),
]


@pytest.mark.parametrize("nx,nz,k,nl,prec,kind", CASES)
def test_fused_vcycle_bitwise_equals_unfused(nx, nz, k, nl, prec, kind):
    with tempfile.TemporaryDirectory() as d:
        fused = _run(CYCLE, os.path.join(d, "f.npy"), "1", nx, nz, k, nl, prec, kind)
        plain = _run(CYCLE, os.path.join(d, "p.npy"), "0", nx, nz, k, nl, prec, kind)
    assert np.all(np.isfinite(fused))
    if prec == "c64":
        assert np.array_equal(fused, plain), f"max rel diff {rel_err(fused, plain):.3e}"
        if k % 8 == 0:  # the opt-in two-vector thread units (HZ_FUSED_WIDE=1)
            with tempfile.TemporaryDirectory() as d:
                wide = _run(CYCLE, os.path.join(d, "w.npy"), "1", nx, nz, k, nl, prec, kind, HZ_FUSED_WIDE="1")
            assert np.array_equal(wide, plain)
    else:
        # complex128: same expressions, but nvcc may contract a complex
        # product into FMAs differently in the two kernels (last-bit
        # differences; the reference parity bar is 1e-12)
        assert rel_err(fused, plain) <= 1e-14


@pytest.mark.parametrize("nx,nz,nl,chunk", [(257, 129, 4, "0"), (1025, 513, 5, "0"), (301, 97, 3, "5"), (121, 233, 4, "3")])
def test_k8_bulk_copy_kernels_equal_streaming_kernels(nx, nz, nl, chunk):
    """k = 8: the bulk-copy (TMA) fused kernels against the cp.async
    streaming kernels they replace (HZ_FUSED_K8=0), bitwise, including
    forced short row chunks (HZ_K8_PRE_ROWS / HZ_K8_POST_CROWS)."""
    extra = {} if chunk == "0" else {"HZ_K8_PRE_ROWS": chunk, "HZ_K8_POST_CROWS": chunk}
    with tempfile.TemporaryDirectory() as d:
        new = _run(CYCLE, os.path.join(d, "n.npy"), "1", nx, nz, 8, nl, "c64", "V", **extra)
        old = _run(CYCLE, os.path.join(d, "o.npy"), "1", nx, nz, 8, nl, "c64", "V", HZ_FUSED_K8="0")
    assert np.array_equal(new, old), f"max rel diff {rel_err(new, old):.3e}"


@pytest.mark.parametrize("nx,nz,nl,kind", [(257, 129, 4, "V"), (1025, 513, 5, "V"), (301, 97, 3, "W"),
                                          (121, 233, 4, "K")])
def test_bulk_copy_galerkin_level_kernel_equals_plain(nx, nz, nl, kind):
    """complex64 2D Galerkin levels at k = 8: the bulk-copy row-staged
    kernel (stencil9_k8, all levels via HZ_S9_MIN_NODES=0) against the plain
    stencil kernels (HZ_S9=0), bitwise, through whole V / W / K cycles."""
    with tempfile.TemporaryDirectory() as d:
        new = _run(CYCLE, os.path.join(d, "n.npy"), "1", nx, nz, 8, nl, "c64", kind, HZ_S9_MIN_NODES="0")
        old = _run(CYCLE, os.path.join(d, "o.npy"), "1", nx, nz, 8, nl, "c64", kind, HZ_S9="0")
        odd = _run(CYCLE, os.path.join(d, "r.npy"), "1", nx, nz, 8, nl, "c64", kind, HZ_S9_ROWS="3")
    assert np.array_equal(new, old), f"max rel diff {rel_err(new, old):.3e}"
    assert np.array_equal(odd, old)


@pytest.mark.parametrize("nx,nz,nl,kind,rows", [(257, 129, 4, "V", "0"), (1025, 513, 5, "V", "0"), (301, 97, 3, "W", "5"),
                                               (121, 233, 4, "K", "9"), (65, 49, 3, "V", "4"), (1025, 513, 6, "W", "13")])
def test_two_sweep_galerkin_level_kernel_equals_single_sweeps(nx, nz, nl, kind, rows):
    """complex64 2D Galerkin levels at k = 8: both Jacobi sweeps of a visit in
    one launch (stencil9_pair_k8, zero-start and general; every level via
    HZ_S9_PAIR_MIN_NODES=0, odd row chunks via HZ_S9P_ROWS) against one launch
    per sweep (HZ_S9_PAIR=0), bitwise, through whole V / W / K cycles; the
    default (levels of >= 100k nodes only) likewise."""
    extra = {} if rows == "0" else {"HZ_S9P_ROWS": rows}
    with tempfile.TemporaryDirectory() as d:
        new = _run(CYCLE, os.path.join(d, "n.npy"), "1", nx, nz, 8, nl, "c64", kind, HZ_S9_PAIR_MIN_NODES="0", **extra)
        old = _run(CYCLE, os.path.join(d, "o.npy"), "1", nx, nz, 8, nl, "c64", kind, HZ_S9_PAIR="0")
        dfl = _run(CYCLE, os.path.join(d, "d.npy"), "1", nx, nz, 8, nl, "c64", kind)
    assert np.array_equal(new, old), f"max rel diff {rel_err(new, old):.3e}"
    assert np.array_equal(dfl, old)


@pytest.mark.parametrize("nx,nz,nl,kind,rows", [(257, 129, 4, "V", "0"), (1025, 513, 5, "V", "0"), (301, 97, 3, "W", "5"),
                                               (121, 233, 4, "K", "3"), (65, 49, 3, "V", "2"), (1025, 513, 6, "W", "7")])
def test_fused_galerkin_level_pre_visit_equals_unfused(nx, nz, nl, kind, rows):
    """complex64 2D Galerkin levels at k = 8 visited from x = 0: both
    pre-sweeps, the residual and its restriction in one launch
    (stencil9_pre_k8, opt-in with HZ_S9_PRE=1; every level via
    HZ_S9_PRE_MIN_NODES=0, odd coarse-row chunks via HZ_S9PRE_ROWS) against the
    unfused kernels (HZ_S9_PRE=0 and HZ_S9_PAIR=0), bitwise, through whole
    V / W / K cycles."""
    extra = {} if rows == "0" else {"HZ_S9PRE_ROWS": rows}
    with tempfile.TemporaryDirectory() as d:
        new = _run(CYCLE, os.path.join(d, "n.npy"), "1", nx, nz, 8, nl, "c64", kind, HZ_S9_PRE="1",
                   HZ_S9_PRE_MIN_NODES="0", HZ_S9_PAIR_MIN_NODES="0", **extra)
        old = _run(CYCLE, os.path.join(d, "o.npy"), "1", nx, nz, 8, nl, "c64", kind, HZ_S9_PRE="0", HZ_S9_PAIR="0")
        dfl = _run(CYCLE, os.path.join(d, "d.npy"), "1", nx, nz, 8, nl, "c64", kind)
    assert np.array_equal(new, old), f"max rel diff {rel_err(new, old):.3e}"
    assert np.array_equal(dfl, old)


def test_fused_c128_cycle_matches_reference():
    """c128 V(2,2) cycle through the fused fine level vs the compiled
    reference's MgHierarchy::cycle at the 1e-12 parity bar."""
    from oracle import ref
    cfg = configs.config2(nlevels=3, k=4, nx=129, nz=65)
    cfg.precond_precision = "c128"
    P = hz.HelmholtzProblem.from_config(cfg)
    S = hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg))
    b = configs.random_block(cfg.num_nodes, 4, seed=5)
    x = S.cycle(b)
    R = ref.RefProblem.from_config(cfg)
    H = ref.RefHierarchy(R, cfg.nlevels, cfg.shift)
    xr = H.cycle(b, kind="V", pre=cfg.pre, post=cfg.post, wj=cfg.jacobi_weight)
    assert rel_err(x, xr) <= 1e-12


SOLVE = (
    "import sys; sys.path.insert(0, '.'); import numpy as np\n"
    "import paper_1607_00968_b200 as hz; from paper_1607_00968_b200 import configs\n"
    "cfg = configs.config2(nlevels=4, k=8, nx=257, nz=129); cfg.restart = 3; cfg.max_cycles = 60\n"
    "S = hz.HelmholtzSolver(hz.HelmholtzProblem.from_config(cfg), hz.HelmholtzSolveOptions.from_config(cfg))\n"
    "X, rep = S.solve_block(cfg.rhs_block())\n"
    "assert np.all(np.isfinite(X)) and rep.cycles > 0\n"
    "np.save(sys.argv[1], X); print(rep.cycles)\n")


def test_fused_solve_bitwise_equals_unfused():
    """60 FGMRES(3) cycles with the c64 preconditioner (fused vs unfused fine
    level): the iterates are bitwise equal (convergence is not the point)."""
    with tempfile.TemporaryDirectory() as d:
        a = _run(SOLVE, os.path.join(d, "a.npy"), "1")
        b = _run(SOLVE, os.path.join(d, "b.npy"), "0")
    assert np.array_equal(a, b)

