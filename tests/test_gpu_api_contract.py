"""GPU tier: the API contract fixes of round 2 -- caller-supplied
solution buffers are validated before the library writes n*k*16 bytes into
them; hz_solve_helmholtz reports HZ_CONVERGENCE whatever report pointers
the caller passes; device solves are ordered after the caller's stream."""
import ctypes as C

import numpy as np
import pytest

from paper_1607_00968_b200 import configs

pytestmark = pytest.mark.gpu
hz = pytest.importorskip("paper_1607_00968_b200")


def _solver(max_cycles=200, tol=1e-6):
    cfg = configs.config1(nlevels=3, nx=65)
    cfg.max_cycles, cfg.tol = max_cycles, tol
    P = hz.HelmholtzProblem.from_config(cfg)
    return cfg, P, hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(cfg))


def test_out_buffer_is_validated_host_and_device():
    import torch
    cfg, P, S = _solver()
    B = cfg.rhs_block()
    n, k = B.shape
    for bad in (np.empty((n, k + 1), np.complex128), np.empty((n, k), np.complex64),
                np.empty((k, n), np.complex128).T, torch.empty((n, k), dtype=torch.complex128)):
        with pytest.raises(hz.ValidationError):
            S.solve_block(B, out=bad)
    with pytest.raises(hz.ValidationError):  # out aliasing B: the solve zeroes X before reading B
        S.solve_block(B, out=B)
    Bd = torch.from_numpy(B).cuda()
    for bad in (torch.empty((n, k + 1), dtype=torch.complex128, device="cuda"),
                torch.empty((n, k), dtype=torch.complex64, device="cuda"),
                torch.empty((k, n), dtype=torch.complex128, device="cuda").t(), np.empty_like(B), Bd):
        with pytest.raises(hz.ValidationError):
            S.solve_block(Bd, out=bad)
    X = np.empty_like(B)
    Xr, rep = S.solve_block(B, out=X)
    assert Xr is X and rep.all_converged()
    Xd = torch.empty_like(Bd)
    Xdr, _ = S.solve_block(Bd, out=Xd)
    assert Xdr is Xd and np.array_equal(Xd.cpu().numpy(), X)


def test_solve_helmholtz_raises_convergence_without_report():
    from paper_1607_00968_b200 import _native
    cfg, P, S = _solver(max_cycles=3)
    B = cfg.rhs_block()
    X = np.empty_like(B)
    L = _native.lib()
    st = L.hz_solve_helmholtz(S._h, B.shape[0], B.shape[1], B.ctypes.data, X.ctypes.data, None)
    assert st == 2  # HZ_CONVERGENCE with a NULL report
    rep = _native.hz_report()  # a report without per-column buffers
    st = L.hz_solve_helmholtz(S._h, B.shape[0], B.shape[1], B.ctypes.data, X.ctypes.data, C.byref(rep))
    assert st == 2 and rep.cycles == 3
    cfg2, P2, S2 = _solver()
    st = L.hz_solve_helmholtz(S2._h, B.shape[0], B.shape[1], B.ctypes.data, X.ctypes.data, None)
    assert st == 0


def test_device_solve_ordered_after_callers_stream():
    """B written on a side stream right before the call: the solve waits for
    that stream (hz_solve_block_device_stream), not for the legacy stream."""
    import torch
    cfg, P, S = _solver()
    B = cfg.rhs_block()
    X_ref, _ = S.solve_block(B)
    side = torch.cuda.Stream()
    Bd = torch.empty((B.shape[0], B.shape[1]), dtype=torch.complex128, device="cuda")
    src = torch.from_numpy(B).pin_memory()
    with torch.cuda.stream(side):
        torch.cuda._sleep(5_000_000)  # keep the side stream busy before the copy lands
        Bd.copy_(src, non_blocking=True)
        Xd, rep = S.solve_block(Bd)  # current stream = side: the library waits on it
    assert rep.all_converged()
    assert np.array_equal(Xd.cpu().numpy(), X_ref)
