"""TEST INFRASTRUCTURE ONLY: ctypes driver for the compiled reference oracle.

Loads oracle/_ref/libseistomo_ref.so -- the UNMODIFIED reference C++ library
(/root/reference/proj/core, built by oracle/Makefile) plus our extern "C" shim
(oracle/ref_shim.cpp) -- and exposes the reference's public API with numpy
arrays. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference arm may import this module; the product path never does.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# libseistomo_ref.so: -ffp-contract=off build (the parity checker);
# libseistomo_ref_fast.so: stock contraction (the CPU baseline bench.py times).
# HZ_REF_VARIANT=fast selects the latter.
LIB_PATH = os.path.join(_HERE, "_ref", "libseistomo_ref.so")
LIB_PATH_FAST = os.path.join(_HERE, "_ref", "libseistomo_ref_fast.so")

_lib = None

_KIND = {"V": 0, "W": 1, "K": 2}
_METHOD = {"MgBicgstab": 0, "MgFgmresW": 1, "MgFgmresK": 2, "DenseLuSmall": 3}


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"reference status {code}: {msg}")
        self.code = code


class _Report(C.Structure):
    _fields_ = [("cycles", C.c_int), ("qr_factorizations", C.c_int),
                ("block_gram_products", C.c_longlong), ("wall_s", C.c_double),
                ("history_len", C.c_int)]


@dataclasses.dataclass
class RefReport:
    cycles: int
    col_cycles: np.ndarray
    rel_residual: np.ndarray
    converged: np.ndarray
    history: np.ndarray
    wall_s: float
    qr_factorizations: int
    block_gram_products: int

    def all_converged(self) -> bool:
        return bool(len(self.converged) and np.all(self.converged))


def _path() -> str:
    return LIB_PATH_FAST if os.environ.get("HZ_REF_VARIANT") == "fast" else LIB_PATH


def available() -> bool:
    return os.path.exists(_path())


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"reference oracle not built: {_path()} (run make -C oracle)")
        _lib = C.CDLL(_path())
        _lib.ref_last_error.restype = C.c_char_p
        _lib.ref_problem_ppw.restype = C.c_double
        _lib.ref_hier_coarse_lu_bytes.restype = C.c_longlong
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _check(code: int):
    if code != 0:
        raise RefError(code, lib().ref_last_error().decode())


def set_num_threads(n: int):
    lib().ref_set_num_threads(int(n))


def num_threads() -> int:
    return int(lib().ref_num_threads())


def _as_cblock(a: np.ndarray, n: int) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.complex128)
    if a.ndim == 1:
        a = a.reshape(n, 1)
    return a


class RefProblem:
    """seistomo::HelmholtzProblem (inc/helmholtz.hpp:19-57)."""

    def __init__(self, ndim, n, h, m, omega, gamma_base, ramp, allow_coarse=False):
        self.ndim = int(ndim)
        self.n = tuple(int(x) for x in n)
        self.num_nodes = self.n[0] * self.n[1] * self.n[2]
        nn = np.asarray(self.n, dtype=np.int64)
        hh = np.asarray(h, dtype=np.float64)
        self._m = np.ascontiguousarray(m, dtype=np.float64)
        self._ramp = np.ascontiguousarray(ramp, dtype=np.float64)
        out = C.c_void_p()
        _check(lib().ref_problem_create(C.c_int(self.ndim), _p(nn), _p(hh), _p(self._m),
                                        C.c_double(omega), C.c_double(gamma_base), _p(self._ramp),
                                        C.c_int(1 if allow_coarse else 0), C.byref(out)))
        self._h = out

    @classmethod
    def from_config(cls, cfg, allow_coarse=False):
        return cls(cfg.ndim, cfg.n, cfg.h, cfg.m, cfg.omega, cfg.gamma_base, cfg.ramp, allow_coarse)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ref_problem_destroy(self._h)
            self._h = None

    def ppw(self) -> float:
        return float(lib().ref_problem_ppw(self._h))

    def mass(self) -> np.ndarray:
        out = np.empty(self.num_nodes, dtype=np.complex128)
        lib().ref_problem_mass(self._h, _p(out))
        return out

    def apply_block(self, u: np.ndarray) -> np.ndarray:
        u = _as_cblock(u, self.num_nodes)
        out = np.empty_like(u)
        _check(lib().ref_apply_block(self._h, C.c_longlong(u.shape[0]), C.c_int(u.shape[1]),
                                     _p(u), _p(out)))
        return out

    def point_source(self, x, amp=1.0 + 0j) -> np.ndarray:
        xx = np.asarray(list(x) + [0.0] * (3 - len(x)), dtype=np.float64)
        out = np.empty(self.num_nodes, dtype=np.complex128)
        _check(lib().ref_point_source(self._h, _p(xx), C.c_double(amp.real), C.c_double(amp.imag),
                                      _p(out)))
        return out

    def sensitivity_output(self, u: np.ndarray, lam: np.ndarray) -> np.ndarray:
        u = np.ascontiguousarray(u, dtype=np.complex128)
        lam = np.ascontiguousarray(lam, dtype=np.complex128)
        g = np.empty(self.num_nodes, dtype=np.float64)
        _check(lib().ref_sensitivity_output(self._h, _p(u), _p(lam), _p(g)))
        return g


class RefHierarchy:
    """seistomo::MgHierarchy<cplx> built by build_hierarchy (src/multigrid.cpp:204-208)."""

    def __init__(self, problem: RefProblem, nlevels: int, shift: float):
        out = C.c_void_p()
        _check(lib().ref_hier_create(problem._h, C.c_int(nlevels), C.c_double(shift), C.byref(out)))
        self._h = out
        self.problem = problem

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ref_hier_destroy(self._h)
            self._h = None

    def num_levels(self) -> int:
        return int(lib().ref_hier_num_levels(self._h))

    def level_dims(self, l: int):
        dims = np.zeros(3, dtype=np.int64)
        nnz = C.c_longlong()
        lib().ref_hier_level_info(self._h, C.c_int(l), _p(dims), C.byref(nnz))
        return tuple(int(x) for x in dims), int(nnz.value)

    def level_csr(self, l: int):
        dims, nnz = self.level_dims(l)
        rows = dims[0] * dims[1] * dims[2]
        rp = np.empty(rows + 1, dtype=np.int64)
        ci = np.empty(nnz, dtype=np.int32)
        v = np.empty(nnz, dtype=np.complex128)
        lib().ref_hier_level_csr(self._h, C.c_int(l), _p(rp), _p(ci), _p(v))
        return rp, ci, v

    def coarse_lu_bytes(self) -> int:
        return int(lib().ref_hier_coarse_lu_bytes(self._h))

    def cycle(self, b: np.ndarray, x: Optional[np.ndarray] = None, kind="V", pre=2, post=2,
              wj=0.8, k_inner=2) -> np.ndarray:
        b = _as_cblock(b, b.shape[0])
        x = np.zeros_like(b) if x is None else np.array(_as_cblock(x, b.shape[0]), copy=True)
        _check(lib().ref_hier_cycle(self._h, C.c_int(_KIND[kind]), C.c_int(pre), C.c_int(post),
                                    C.c_double(wj), C.c_int(k_inner), C.c_longlong(b.shape[0]),
                                    C.c_int(b.shape[1]), _p(b), _p(x)))
        return x

    def coarse_solve(self, b: np.ndarray) -> np.ndarray:
        x = np.array(_as_cblock(b, b.shape[0]), copy=True)
        _check(lib().ref_hier_coarse_solve(self._h, C.c_longlong(x.shape[0]), C.c_int(x.shape[1]),
                                           _p(x)))
        return x


def _report_buffers(k, cap):
    return (_Report(), np.zeros(k, np.int32), np.zeros(k, np.float64), np.zeros(k, np.int32),
            np.zeros(cap, np.float64))


def _make_report(rep, cc, rr, cv, hist, cap) -> RefReport:
    hl = min(rep.history_len, cap)
    return RefReport(cycles=rep.cycles, col_cycles=cc.copy(), rel_residual=rr.copy(),
                     converged=cv.astype(bool), history=hist[:hl].copy(), wall_s=rep.wall_s,
                     qr_factorizations=rep.qr_factorizations,
                     block_gram_products=rep.block_gram_products)


def krylov_solve(problem: RefProblem, hier: Optional[RefHierarchy], B: np.ndarray, method="fgmres",
                 kind="V", pre=2, post=2, wj=0.8, k_inner=2, restart=10, tol=1e-6,
                 max_cycles=200):
    """SURVEY §3.3 composition: apply_block + (out:=0; MgHierarchy::cycle) as
    a BlockOperator into block_fgmres / block_bicgstab."""
    B = _as_cblock(B, problem.num_nodes)
    n, k = B.shape
    X = np.empty_like(B)
    cap = max_cycles + 8
    rep, cc, rr, cv, hist = _report_buffers(k, cap)
    _check(lib().ref_krylov_solve(
        problem._h, hier._h if hier is not None else None, C.c_int(1 if method == "bicgstab" else 0),
        C.c_int(_KIND[kind]), C.c_int(pre), C.c_int(post), C.c_double(wj), C.c_int(k_inner),
        C.c_int(restart), C.c_double(tol), C.c_int(max_cycles), C.c_longlong(n), C.c_int(k), _p(B),
        _p(X), C.byref(rep), _p(cc), _p(rr), _p(cv), _p(hist), C.c_int(cap)))
    return X, _make_report(rep, cc, rr, cv, hist, cap)


class RefSolver:
    """seistomo::HelmholtzSolver (inc/helmholtz_solver.hpp:30-79)."""

    def __init__(self, problem: RefProblem, method="MgBicgstab", tol=1e-6, max_cycles=200,
                 nlevels=3, shift=0.2, pre=2, post=2, wj=0.8, k_inner=2, restart=5,
                 dense_threshold=3000):
        out = C.c_void_p()
        _check(lib().ref_solver_create(problem._h, C.c_int(_METHOD[method]), C.c_double(tol),
                                       C.c_int(max_cycles), C.c_int(nlevels), C.c_double(shift),
                                       C.c_int(pre), C.c_int(post), C.c_double(wj),
                                       C.c_int(k_inner), C.c_int(restart),
                                       C.c_longlong(dense_threshold), C.byref(out)))
        self._h = out
        self.problem = problem
        self.max_cycles = max_cycles

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ref_solver_destroy(self._h)
            self._h = None

    def solve_block(self, B: np.ndarray):
        B = _as_cblock(B, self.problem.num_nodes)
        n, k = B.shape
        X = np.empty_like(B)
        cap = self.max_cycles + 8
        rep, cc, rr, cv, hist = _report_buffers(k, cap)
        _check(lib().ref_solver_solve_block(self._h, C.c_longlong(n), C.c_int(k), _p(B), _p(X),
                                            C.byref(rep), _p(cc), _p(rr), _p(cv), _p(hist),
                                            C.c_int(cap)))
        return X, _make_report(rep, cc, rr, cv, hist, cap)


def gram(X: np.ndarray, Y: np.ndarray) -> np.ndarray:
    X = np.ascontiguousarray(X, dtype=np.complex128)
    Y = np.ascontiguousarray(Y, dtype=np.complex128)
    G = np.empty((X.shape[1], Y.shape[1]), dtype=np.complex128)
    lib().ref_gram(C.c_longlong(X.shape[0]), C.c_int(X.shape[1]), C.c_int(Y.shape[1]), _p(X), _p(Y),
                   _p(G))
    return G


def thin_qr(W: np.ndarray):
    Q = np.array(np.ascontiguousarray(W, dtype=np.complex128), copy=True)
    R = np.empty((Q.shape[1], Q.shape[1]), dtype=np.complex128)
    rd = lib().ref_thin_qr(C.c_longlong(Q.shape[0]), C.c_int(Q.shape[1]), _p(Q), _p(R))
    return Q, R, bool(rd)


def least_squares(A: np.ndarray, B: np.ndarray):
    A = np.ascontiguousarray(A, dtype=np.complex128)
    B = np.ascontiguousarray(B, dtype=np.complex128)
    Y = np.empty((A.shape[1], B.shape[1]), dtype=np.complex128)
    res = np.empty(B.shape[1], dtype=np.float64)
    _check(lib().ref_least_squares(C.c_longlong(A.shape[0]), C.c_longlong(A.shape[1]),
                                   C.c_longlong(B.shape[1]), _p(A), _p(B), _p(Y), _p(res)))
    return Y, res


def attenuation_ramp(ndim, n, lo, hi) -> np.ndarray:
    nn = np.asarray(list(n) + [1] * (3 - len(n)), dtype=np.int64)
    lo_ = np.asarray(list(lo) + [0] * (3 - len(lo)), dtype=np.int32)
    hi_ = np.asarray(list(hi) + [0] * (3 - len(hi)), dtype=np.int32)
    out = np.empty(int(np.prod(nn)), dtype=np.float64)
    _check(lib().ref_attenuation_ramp(C.c_int(ndim), _p(nn), _p(lo_), _p(hi_), _p(out)))
    return out


# ---- FWI path either side of the solve
class RefSampling:
    """seistomo::SamplingOperator over receivers at physical points
    (inc/acquisition.hpp:30-62, src/acquisition.cpp:33-62)."""

    def __init__(self, ndim, n, h, receivers_xyz, origin=(0.0, 0.0, 0.0)):
        nn = np.asarray(list(n) + [1] * (3 - len(n)), dtype=np.int64)
        hh = np.asarray(list(h) + [1.0] * (3 - len(h)), dtype=np.float64)
        oo = np.asarray(list(origin) + [0.0] * (3 - len(origin)), dtype=np.float64)
        xyz = np.ascontiguousarray(receivers_xyz, dtype=np.float64).reshape(-1, 3)
        self.nrec = xyz.shape[0]
        self.n = int(nn.prod())
        out = C.c_void_p()
        _check(lib().ref_sampling_create(C.c_int(ndim), _p(nn), _p(hh), _p(oo), C.c_longlong(self.nrec),
                                         _p(xyz), C.byref(out)))
        self._h = out

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ref_sampling_destroy(self._h)
            self._h = None

    def receiver(self, r):
        nodes = np.zeros(8, np.int64)
        w = np.zeros(8, np.float64)
        c = lib().ref_sampling_receiver(self._h, C.c_longlong(r), _p(nodes), _p(w))
        return nodes[:c].copy(), w[:c].copy()

    def sample(self, u):
        u = np.ascontiguousarray(u, dtype=np.complex128).reshape(-1)
        d = np.empty(self.nrec, np.complex128)
        _check(lib().ref_sample(self._h, _p(u), _p(d)))
        return d

    def sample_adjoint(self, d):
        d = np.ascontiguousarray(d, dtype=np.complex128).reshape(-1)
        u = np.empty(self.n, np.complex128)
        _check(lib().ref_sample_adjoint(self._h, _p(d), _p(u)))
        return u


def fwi_sensitivity_rhs(problem: RefProblem, u, v):
    u = np.ascontiguousarray(u, dtype=np.complex128).reshape(-1)
    v = np.ascontiguousarray(v, dtype=np.float64).reshape(-1)
    out = np.empty_like(u)
    _check(lib().ref_fwi_sensitivity_rhs(problem._h, _p(u), _p(v), _p(out)))
    return out


def fwi_jacobian_vec(solver: RefSolver, u, sampling: RefSampling, v):
    u = np.ascontiguousarray(u, dtype=np.complex128).reshape(-1)
    v = np.ascontiguousarray(v, dtype=np.float64).reshape(-1)
    d = np.empty(sampling.nrec, np.complex128)
    _check(lib().ref_fwi_jacobian_vec(solver._h, sampling._h, _p(u), _p(v), _p(d)))
    return d


def fwi_jacobian_transpose_vec(solver: RefSolver, u, sampling: RefSampling, w):
    u = np.ascontiguousarray(u, dtype=np.complex128).reshape(-1)
    w = np.ascontiguousarray(w, dtype=np.complex128).reshape(-1)
    g = np.empty(u.size, np.float64)
    _check(lib().ref_fwi_jacobian_transpose_vec(solver._h, sampling._h, _p(u), _p(w), _p(g)))
    return g


# ---- wavefield output
def wavefield_roundtrip(fields, dims2d, compact: bool, path: str = ""):
    """WavefieldBatch append (Full32 / Compact16) -> field(s); optional JSWF1
    save (src/helmholtz.cpp:137-195). fields: [nsrc][n] complex."""
    F = np.ascontiguousarray(fields, dtype=np.complex128)
    nsrc, n = F.shape
    out = np.empty_like(F)
    _check(lib().ref_wavefield_roundtrip(C.c_longlong(dims2d[0]), C.c_longlong(dims2d[1]), C.c_int(nsrc), _p(F),
                                         C.c_int(1 if compact else 0), _p(out), path.encode()))
    return out


def wavefield_load(path: str, dims2d, max_src: int):
    n = dims2d[0] * dims2d[1]
    out = np.zeros((max_src, n), np.complex128)
    ns = C.c_int(0)
    _check(lib().ref_wavefield_load(path.encode(), C.c_longlong(dims2d[0]), C.c_longlong(dims2d[1]),
                                    C.c_int(max_src), _p(out), C.byref(ns)))
    return out[:ns.value]
