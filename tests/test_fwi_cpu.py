"""CPU tier: the numpy restatement of the receiver sampling and Compact16
quantisation (oracle/port.py) pinned against the compiled reference, and the
JSWF1 writer / reader of the Python mirror (host file-format code) byte for
byte against the reference's files. No GPU."""
import os
import tempfile

import numpy as np
import pytest

from oracle import port


def _fields(n, nsrc, seed):
    rng = np.random.default_rng(seed)
    F = (rng.standard_normal((nsrc, n)) + 1j * rng.standard_normal((nsrc, n))) * np.array(
        [1e-3, 1.0, 7.5e4, 3.0][:nsrc])[:, None]
    F[0, :5] = 0.0
    F[1, 7] = 1e-12
    F[-1] = 0.0
    return F


@pytest.mark.parametrize("ndim,n", [(2, (65, 33, 1)), (3, (17, 17, 9))])
def test_sampling_port_matches_reference(ref, ndim, n):
    rng = np.random.default_rng(4)
    xyz = np.zeros((25, 3))
    for a in range(ndim):
        xyz[:, a] = rng.uniform(0, n[a] - 1, 25)
    xyz[:4, :ndim] = np.floor(xyz[:4, :ndim])  # on nodes: zero weights dropped
    xyz[5] = xyz[6]
    R = ref.RefSampling(ndim, n, (1.0, 1.0, 1.0), xyz)
    op = port.sampling_operator(ndim, n, (1.0, 1.0, 1.0), (0.0, 0.0, 0.0), xyz)
    for r in range(25):
        nodes, w = R.receiver(r)
        assert np.array_equal(op[r][0], nodes) and np.array_equal(op[r][1], w)
    nn = int(np.prod(n))
    u = rng.standard_normal(nn) + 1j * rng.standard_normal(nn)
    assert np.array_equal(port.sample(op, u), R.sample(u))
    d = rng.standard_normal(25) + 1j * rng.standard_normal(25)
    assert np.array_equal(port.sample_adjoint(op, d, nn), R.sample_adjoint(d))


def test_compact16_port_matches_reference(ref):
    dims = (33, 17)
    F = _fields(dims[0] * dims[1], 4, seed=3)
    expect = ref.wavefield_roundtrip(F, dims, compact=True)
    for s in range(4):
        q, scale = port.compact16(F[s])
        assert np.array_equal(port.compact16_field(q, scale), expect[s])
        peak = max(np.abs(F[s].real).max(), np.abs(F[s].imag).max())
        err = np.abs(port.compact16_field(q, scale) - F[s]).max()
        assert err <= 2.0 ** -10 * max(peak, 1e-300) * 2  # documented round-trip bound


@pytest.mark.parametrize("precision", ["Full32", "Compact16"])
def test_jswf1_writer_matches_reference_bytes(ref, precision):
    """Host file format only: a Compact16 batch is filled from the port's
    quantisation (the product quantises on the GPU; tested in the GPU tier)."""
    from paper_1607_00968_b200 import fwi
    dims = (33, 17)
    n = dims[0] * dims[1]
    F = _fields(n, 3, seed=5)
    B = fwi.WavefieldBatch(n, precision)
    for s in range(3):
        if precision == "Full32":
            B._ids.append(s)
            B._full.append(F[s].copy())
        else:
            q, scale = port.compact16(F[s])
            B._ids.append(s)
            B._q.append(q)
            B._scale.append(scale)
    with tempfile.TemporaryDirectory() as d:
        pr, pm = os.path.join(d, "ref.jswf"), os.path.join(d, "ours.jswf")
        ref.wavefield_roundtrip(F, dims, compact=precision == "Compact16", path=pr)
        B.save(pm)
        assert open(pr, "rb").read() == open(pm, "rb").read()
        L = fwi.WavefieldBatch.load(pm, n)
        Lr = ref.wavefield_load(pr, dims, 3)
        assert len(L) == 3
        for s in range(3):
            assert np.array_equal(L.field(s), Lr[s])
