"""CPU tier: pin the numpy restatement (oracle/port.py) against the golden
vectors the REFERENCE produced (tests/golden/*.npz, from oracle/_ref via
tests/golden/make_golden.py), and -- where the compiled reference is present
-- check the golden vectors are still what the reference computes."""
import os

import numpy as np
import pytest

from hzt_util import rel_err
from oracle import port

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(tag):
    return dict(np.load(os.path.join(GOLD, f"{tag}.npz")))


def problem(d):
    return port.Problem(int(d["ndim"]), tuple(int(x) for x in d["n"]), tuple(float(x) for x in d["h"]),
                        d["m"], float(d["omega"]), float(d["gamma_base"]), d["ramp"])


@pytest.mark.parametrize("tag", ["apply2d", "apply3d"])
def test_apply_block(tag):
    d = load(tag)
    P = problem(d)
    assert rel_err(P.apply_block(d["u"]), d["v"]) <= 1e-13
    assert np.allclose(P.mass, d["mass"], rtol=1e-15, atol=0)
    assert abs(P.points_per_wavelength() - float(d["ppw"])) <= 1e-12


def test_attenuation_ramp():
    d = load("ramp")
    assert np.array_equal(port.attenuation_ramp(2, (33, 17), (4, 0), (4, 5)), d["r2"])
    assert np.array_equal(port.attenuation_ramp(3, (9, 11, 7), (2, 3, 0), (1, 2, 3)), d["r3"])


def test_config_ramp_matches_reference_restatement():
    from paper_1607_00968_b200 import configs
    r = configs.quadratic_ramp(2, (33, 17, 1), (4, 0, 0), (4, 5, 0))
    assert np.array_equal(r, load("ramp")["r2"])


@pytest.mark.parametrize("tag", ["hier2d", "hier3d"])
def test_hierarchy_galerkin_and_cycles(tag):
    d = load(tag)
    P = problem(d)
    nl = int(d["nlevels"])
    H = port.Hierarchy(P, nl, float(d["shift"]))
    for l in range(nl):
        assert tuple(H.dims[l]) == tuple(int(x) for x in d[f"dims{l}"])
        A = H.A[l].tocsr()
        A.sort_indices()
        ref_A = __import__("scipy.sparse", fromlist=["csr_matrix"]).csr_matrix(
            (d[f"v{l}"], d[f"ci{l}"], d[f"rp{l}"]), shape=A.shape)
        diff = A - ref_A
        assert (abs(diff).max() if diff.nnz else 0.0) <= 1e-13 * abs(ref_A).max()
    b = d["b"]
    assert rel_err(H.cycle(b, kind="V"), d["xV"]) <= 1e-12
    assert rel_err(H.cycle(b, kind="W"), d["xW"]) <= 1e-12
    if "xK" in d:
        assert rel_err(H.cycle(b, kind="K"), d["xK"]) <= 1e-10
    assert rel_err(H.coarse @ d["bc"], d["xc"]) <= 1e-12


def test_fgmres_v_solve():
    d = load("fgmres")
    P = problem(d)
    X, rep = port.mg_krylov_solve(P, d["B"], int(d["nlevels"]), float(d["shift"]), method="fgmres",
                                  kind="V", restart=10, tol=1e-6, max_cycles=200)
    assert rep.all_converged()
    assert rep.cycles == int(d["cycles"])
    assert np.array_equal(rep.col_cycles, d["col_cycles"])
    for j in range(d["B"].shape[1]):
        assert rel_err(X[:, j], d["X"][:, j]) <= 1e-8
    assert np.allclose(rep.history, d["history"], rtol=1e-6)


def test_bicgstab_w_solve():
    d = load("bicgstab")
    P = problem(d)
    X, rep = port.mg_krylov_solve(P, d["B"], int(d["nlevels"]), float(d["shift"]), method="bicgstab",
                                  kind="W", tol=1e-6, max_cycles=200)
    assert rep.all_converged()
    assert abs(rep.cycles - int(d["cycles"])) <= 2
    for j in range(d["B"].shape[1]):
        assert rel_err(X[:, j], d["X"][:, j]) <= 1e-6


def test_dense_kernels():
    d = load("dense")
    Q, R, rd = port.thin_qr(d["W"])
    assert not rd and not bool(d["rd"])
    assert rel_err(Q, d["Q"]) <= 1e-13 and rel_err(R, d["R"]) <= 1e-13
    Y, res = port.least_squares(d["A"], d["Bl"])
    assert rel_err(Y, d["Y"]) <= 1e-12 and rel_err(res, d["res"]) <= 1e-12
    assert rel_err(d["Xg"].conj().T @ d["Yg"], d["G"]) <= 1e-14


def test_thin_qr_rank_deficiency():
    """thin_qr zeroes a collapsed column and flags it (inc/block.hpp:126-131)."""
    rng = np.random.default_rng(0)
    W = rng.standard_normal((40, 3)) + 0j
    W[:, 2] = 2 * W[:, 0] - W[:, 1]
    Q, R, rd = port.thin_qr(W)
    assert rd and not np.any(Q[:, 2]) and R[2, 2] == 0


def test_sensitivity():
    d = load("sens")
    P = problem(d)
    assert rel_err(P.sensitivity_output(d["u"], d["lam"]), d["g"]) <= 1e-14


def test_block_krylov_identity_kats():
    """A = I converges in one iteration; 2x2 SPD dense oracle."""
    B = np.array([[1.0 + 0j, 2.0], [3.0, -1.0]])
    op = port.BlockOperator(n=2, apply=lambda v: v)
    X, rep = port.block_fgmres(op, B, 5, 1e-10, 10)
    assert rep.cycles == 1 and np.allclose(X, B)
    A = np.array([[4.0, 1.0], [1.0, 3.0]], dtype=np.complex128)
    op = port.BlockOperator(n=2, apply=lambda v: A @ v)
    X, rep = port.block_fgmres(op, B, 5, 1e-12, 10)
    assert np.allclose(X, np.linalg.solve(A, B), rtol=1e-10)
    X, rep = port.block_bicgstab(op, B, 1e-12, 10)
    assert np.allclose(X, np.linalg.solve(A, B), rtol=1e-10)


def test_golden_vectors_are_the_references_answers(ref):
    """Where the compiled reference is present (this container / the GPU box),
    the committed fixtures must equal what it computes now (bitwise)."""
    d = load("apply2d")
    R = ref.RefProblem(int(d["ndim"]), d["n"], d["h"], d["m"], float(d["omega"]), float(d["gamma_base"]),
                       d["ramp"])
    assert np.array_equal(R.apply_block(d["u"]), d["v"])
    d = load("hier2d")
    R = ref.RefProblem(int(d["ndim"]), d["n"], d["h"], d["m"], float(d["omega"]), float(d["gamma_base"]),
                       d["ramp"])
    H = ref.RefHierarchy(R, int(d["nlevels"]), float(d["shift"]))
    assert np.array_equal(H.level_csr(1)[2], d["v1"])
    assert np.array_equal(H.cycle(d["b"], kind="V"), d["xV"])
