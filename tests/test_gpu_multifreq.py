"""GPU tier: multi-frequency batching -- several (m, omega)
hierarchies resident on one GPU, solved as one concurrent batch
(hz_solve_blocks_multi: one host thread / stream per frequency). Every
frequency's result must equal its own sequential solve bitwise and the
compiled reference within the solver tolerance; the multi-frequency FWI
gradient must equal the frequency-ordered sum of the single-frequency ones."""
import dataclasses

import numpy as np
import pytest

from hzt_util import rel_err
from paper_1607_00968_b200 import configs

pytestmark = pytest.mark.gpu
hz = pytest.importorskip("paper_1607_00968_b200")

SCALES = (0.6, 0.8, 1.0)  # omega_f / omega (increasing, as a continuation stage)


def _cfgs():
    base = configs.config1(nlevels=3, nx=65)
    return [dataclasses.replace(base, omega=base.omega * s) for s in SCALES]


def _solvers(cfgs):
    return [hz.HelmholtzSolver(hz.HelmholtzProblem.from_config(c), hz.HelmholtzSolveOptions.from_config(c))
            for c in cfgs]


def test_multi_frequency_batch_matches_sequential_and_reference(ref):
    cfgs = _cfgs()
    solvers = _solvers(cfgs)
    B = cfgs[0].rhs_block()
    Xs, reps = hz.solve_blocks_multi(solvers, [B] * len(cfgs))
    for c, S, X, rep in zip(cfgs, solvers, Xs, reps):
        Xq, rq = S.solve_block(B)
        assert np.array_equal(X, Xq) and rep.cycles == rq.cycles  # concurrency changes nothing
        assert rep.all_converged()
        R = ref.RefProblem.from_config(c)
        H = ref.RefHierarchy(R, c.nlevels, c.shift)
        Xr, rr = ref.krylov_solve(R, H, B, method="fgmres", kind="V", restart=c.restart, tol=c.tol,
                                  max_cycles=c.max_cycles)
        assert rr.all_converged()
        assert abs(rep.cycles - rr.cycles) <= 0.05 * rr.cycles + 2
        for j in range(B.shape[1]):
            assert rel_err(X[:, j], Xr[:, j]) <= 1e-5


def test_multi_frequency_solver_device_blocks():
    import torch
    base = configs.config1(nlevels=3, nx=65)
    M = hz.MultiFrequencySolver(base.ndim, base.n, base.h, base.m, [base.omega * s for s in SCALES],
                                hz.AttenuationField(base.gamma_base, base.ramp),
                                hz.HelmholtzSolveOptions.from_config(base))
    assert len(M) == len(SCALES)
    B = base.rhs_block()
    Bd = torch.from_numpy(B).cuda()
    Xd, rd = M.solve_blocks([Bd] * len(M))
    Xh, rh = M.solve_blocks([B] * len(M))
    for a, b, p, q in zip(Xd, Xh, rd, rh):
        assert np.array_equal(a.cpu().numpy(), b) and p.cycles == q.cycles and p.all_converged()


def test_multi_frequency_gradient_is_sum_of_single_frequency():
    import torch
    from paper_1607_00968_b200 import parallel
    cfgs = _cfgs()
    probs = [hz.HelmholtzProblem.from_config(c) for c in cfgs]
    solvers = [hz.HelmholtzSolver(P, hz.HelmholtzSolveOptions.from_config(c)) for P, c in zip(probs, cfgs)]
    n0 = cfgs[0].n[0]
    src = [int(s) for s in cfgs[0].source_nodes]
    rec = np.arange(8, n0 - 8, dtype=np.int64) + n0 * 2  # a receiver line below the surface
    rng = np.random.default_rng(3)
    dobs = [rng.standard_normal((len(rec), len(src))) * 1e-3 + 0j for _ in cfgs]
    res = parallel.fwi_gradient_multi(probs, solvers, src, rec, lambda f, mine: dobs[f][:, mine])
    g = torch.zeros_like(res.gradient)
    mis = 0.0
    for f, (P, S) in enumerate(zip(probs, solvers)):
        r1 = parallel.fwi_gradient(P, S, src, rec, lambda mine, f=f: dobs[f][:, mine])
        g += r1.gradient
        mis += r1.misfit
    assert torch.equal(res.gradient, g)
    assert abs(res.misfit - mis) <= 1e-12 * abs(mis)
    assert float(torch.linalg.norm(g)) > 0


def test_multi_frequency_rejects_shared_solver():
    base = configs.config1(nlevels=3, nx=65)
    S = _solvers([base])[0]
    B = base.rhs_block()
    with pytest.raises(hz.ValidationError):
        hz.solve_blocks_multi([S, S], [B, B])
