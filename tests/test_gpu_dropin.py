"""GPU tier: the drop-in's problem-level pieces through the C ABI against
the compiled reference: point_source / nearest_node (origin, exact
half-spacing ties toward the lower index, outside-grid rejection), the
batched device point-source block, mass, and to_csr(shift) vs the
reference's shifted CSR (bitwise)."""
import numpy as np
import pytest

from paper_1607_00968_b200 import configs

pytestmark = pytest.mark.gpu
hz = pytest.importorskip("paper_1607_00968_b200")


def _pair(origin=(0.0, 0.0, 0.0), ndim=2, n=(33, 17, 1)):
    from oracle import ref
    cfg = configs.small_problem(ndim, n, seed=5, layer=3)
    P = hz.HelmholtzProblem(cfg.ndim, cfg.n, cfg.h, cfg.m, cfg.omega, hz.AttenuationField(cfg.gamma_base, cfg.ramp),
                            device=0, origin=origin)
    return cfg, P, ref.RefProblem.from_config(cfg)


POINTS_2D = [(4.0, 3.0), (4.5, 3.0), (4.5, 3.5), (0.0, 0.0), (32.0, 16.0), (31.5, 15.5), (7.25, 8.75),
             (-1e-10, 2.0), (32.0 + 1e-10, 16.0)]


def test_point_source_matches_reference_with_ties():
    cfg, P, R = _pair()
    for x in POINTS_2D:
        q, qr = P.point_source(x, 2.0 - 0.5j), R.point_source(x, 2.0 - 0.5j)
        assert np.array_equal(q, qr), x
        assert P.nearest_node(x) == int(np.flatnonzero(qr)[0])
    # ties go low: 4.5 -> 4, 31.5 -> 31
    assert P.nearest_node((4.5, 3.5)) == 4 + 33 * 3
    assert P.nearest_node((31.5, 15.5)) == 31 + 33 * 15


def test_point_source_outside_grid_raises_like_reference():
    cfg, P, R = _pair()
    for x in [(-0.01, 1.0), (1.0, 16.01), (33.0, 1.0)]:
        with pytest.raises(hz.ValidationError):
            P.point_source(x)
        with pytest.raises(Exception):
            R.point_source(x)


def test_point_source_honours_grid_origin():
    o = (100.0, -7.0, 0.0)
    cfg, Po, R = _pair(origin=o)
    for x in POINTS_2D[:7]:
        shifted = (x[0] + o[0], x[1] + o[1])
        assert np.array_equal(Po.point_source(shifted), R.point_source(x)), x
    with pytest.raises(hz.ValidationError):
        Po.point_source((0.0, 0.0))  # inside the un-shifted box, outside this grid


def test_point_source_3d_matches_reference():
    cfg, P, R = _pair(ndim=3, n=(9, 9, 9))
    for x in [(4.5, 4.5, 4.5), (0.5, 8.0, 2.5), (8.0, 0.0, 0.0), (3.3, 2.5, 7.5)]:
        assert np.array_equal(P.point_source(x, 1j), R.point_source(x, 1j)), x


def test_device_point_source_block_equals_columns():
    import torch
    cfg, P, R = _pair()
    xs = [(4.5, 3.0), (10.0, 0.0), (31.5, 15.5), (16.25, 8.5)]
    amps = [1.0, 2.0 - 1j, 0.5j, -3.0]
    B = P.point_sources(xs, amps).cpu().numpy()
    for j, (x, a) in enumerate(zip(xs, amps)):
        assert np.array_equal(B[:, j], R.point_source(x, a))
    B1 = P.point_sources(xs).cpu().numpy()
    assert np.array_equal(B1[:, 2], R.point_source(xs[2], 1.0))


def test_mass_gamma_factor_and_to_csr_bitwise():
    from oracle import ref
    cfg, P, R = _pair()
    assert np.array_equal(P.mass(), R.mass())
    H = ref.RefHierarchy(R, 2, 0.5)
    rp, ci, v = P.to_csr(0.5)
    rr, cr, vr = H.level_csr(0)
    assert np.array_equal(rp, rr) and np.array_equal(ci, cr) and np.array_equal(v, vr)
    gf = P.gamma_factor()
    assert np.array_equal(gf, 1.0 - 1j * ((cfg.gamma_base + cfg.omega * cfg.ramp) / cfg.omega))
