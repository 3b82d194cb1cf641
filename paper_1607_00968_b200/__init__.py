"""B200-native multi-RHS Helmholtz solver (shifted-Laplacian MG + block Krylov).

Python mirror of the reference's solver interface (seistomo,
/root/reference/proj/core/include/seistomo/{helmholtz,helmholtz_solver,
multigrid,krylov}.hpp) over the C ABI of include/hz_b200.h. Names, argument
meaning and error classes follow the reference so callers (and the parity
tests) read like the reference's own:

    prob = HelmholtzProblem(ndim, n, h, m, omega, AttenuationField(base, ramp))
    solver = HelmholtzSolver(prob, HelmholtzSolveOptions(method="MgFgmresW"))
    X, report = solver.solve_block(B)          # B: [n][k] complex128

Blocks are node-major [n][k] complex128 (BlockVec, inc/block.hpp:13-27), as
numpy arrays (host; copies are part of the call) or torch CUDA tensors
(device-resident; no copies). All compute runs in libhz_b200.so on the GPU.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _native
from ._native import hz_options, hz_report

__all__ = [
    "ValidationError", "ConvergenceError", "BreakdownError", "FactorizationError", "StateError",
    "IoError", "CudaError", "NcclError", "AttenuationField", "HelmholtzProblem",
    "HelmholtzSolveOptions", "CycleSpec", "HelmholtzSolver", "SolveReport", "solve_helmholtz",
    "fwi_sensitivity_output", "kernel_launch_count", "device_count", "SamplingOperator",
    "fwi_sensitivity_rhs", "fwi_jacobian_vec", "fwi_jacobian_transpose_vec", "WavefieldBatch", "Full32",
    "Compact16", "compact16",
]


# ---------------------------------------------------------------- errors
class HzError(RuntimeError):
    code = -1


class ValidationError(HzError, ValueError):  # seistomo::ValidationError
    code = 1


class ConvergenceError(HzError):  # seistomo::ConvergenceError{residual_history}
    code = 2

    def __init__(self, msg, residual_history=None):
        super().__init__(msg)
        self.residual_history = [] if residual_history is None else [float(x) for x in residual_history]


class BreakdownError(HzError):
    code = 3


class FactorizationError(HzError):
    code = 4


class StateError(HzError):
    code = 5


class IoError(HzError):
    code = 6


class CudaError(HzError):
    code = 7


class NcclError(HzError):
    code = 8


_ERRORS = {c.code: c for c in (ValidationError, ConvergenceError, BreakdownError,
                               FactorizationError, StateError, IoError, CudaError, NcclError)}


def _check(status: int):
    if status != 0:
        msg = _native.lib().hz_last_error_message().decode(errors="replace")
        raise _ERRORS.get(status, HzError)(msg)


def kernel_launch_count() -> int:
    return int(_native.lib().hz_kernel_launch_count())


def device_count() -> int:
    return int(_native.lib().hz_device_count())


def measure_fp64_peak() -> float:
    """FP64 tensor-pipe (DMMA) peak of the current device, TFLOP/s, measured
    live (the denominator of the FP64-bound Gram / block-update kernels)."""
    v = C.c_double()
    _check(_native.lib().hz_measure_fp64_peak(C.byref(v)))
    return float(v.value)


def solve_blocks_multi(solvers: Sequence["HelmholtzSolver"], Bs, outs=None):
    """Multi-frequency batching: solvers[i].solve_block(Bs[i])
    for every i, run concurrently (hz_solve_blocks_multi[_device]: one host
    thread per solve, kernels overlapping on the GPU). Each solver owns its
    (m, omega) hierarchy, stream and Krylov workspace -- typically one per
    frequency of a frequency-continuation stage. Results
    equal the sequential solves. Bs: all numpy (host) or all torch (device)."""
    cnt = len(solvers)
    if len(Bs) != cnt:
        raise ValidationError("solve_blocks_multi: one right-hand-side block per solver")
    if len({id(s) for s in solvers}) != cnt:
        raise ValidationError("solve_blocks_multi: solvers must be distinct")
    if cnt == 0:
        return [], []
    dev = _is_torch(Bs[0])
    Xs, reps, bufs, ptrB, ptrX, ns, ks = [], [], [], [], [], [], []
    for i, (S, B) in enumerate(zip(solvers, Bs)):
        n = S.problem.num_nodes
        if dev:
            B = _dev_block(B, n, S.problem.device)
            import torch
            X = _check_out(outs[i], B, dev=True) if outs is not None else torch.empty_like(B)
            ptrB.append(B.data_ptr())
            ptrX.append(X.data_ptr())
        else:
            B = _host_block(B, n)
            X = _check_out(outs[i], B, dev=False) if outs is not None else np.empty_like(B)
            ptrB.append(B.ctypes.data)
            ptrX.append(X.ctypes.data)
        r, b = S._report(B.shape[1], S.options.max_cycles + 8)
        Xs.append(X)
        reps.append(r)
        bufs.append((b, B))
        ns.append(n)
        ks.append(B.shape[1])
    if dev:
        import torch
        torch.cuda.synchronize()
    L = _native.lib()
    hs = (C.c_void_p * cnt)(*[S._h for S in solvers])
    rep_arr = (hz_report * cnt)(*reps)
    nn = (C.c_int64 * cnt)(*ns)
    kk = (C.c_int * cnt)(*ks)
    pb = (C.c_void_p * cnt)(*ptrB)
    px = (C.c_void_p * cnt)(*ptrX)
    fn = L.hz_solve_blocks_multi_device if dev else L.hz_solve_blocks_multi
    _check(fn(cnt, hs, nn, kk, pb, px, rep_arr))
    return Xs, [S._finish(rep_arr[i], bufs[i][0]) for i, S in enumerate(solvers)]


def _dev_blocks(Xs):
    import torch
    Xs = [x.contiguous() for x in Xs]
    if not Xs or any(x.dtype != torch.complex128 or not x.is_cuda or x.dim() != 2 for x in Xs):
        raise ValidationError("block algebra: complex128 [n][k] CUDA tensors expected")
    if any(x.shape != Xs[0].shape for x in Xs):
        raise ValidationError("block algebra: all blocks must have the same shape")
    return Xs


def block_gram(Xs, Y):
    """G_i = X_i^H Y for every block X_i (gram, inc/block.hpp:51-74, batched
    over the blocks as the Arnoldi step uses it): [nb, k, k] complex128 numpy."""
    import torch
    Xs = _dev_blocks(Xs)
    Y = _dev_blocks([Y])[0]
    n, k = Xs[0].shape
    nb = len(Xs)
    G = np.empty((nb, k, k), dtype=np.complex128)
    ptrs = (C.c_void_p * nb)(*[x.data_ptr() for x in Xs])
    torch.cuda.synchronize()
    with torch.cuda.device(Y.device):
        _check(_native.lib().hz_block_gram_device(n, k, nb, ptrs, Y.data_ptr(), G.ctypes.data))
    return G


def block_add_scaled(Y, Xs, Cs):
    """Y += sum_i X_i C_i in place (add_block_scaled, inc/block.hpp:76-88,
    batched); Y a contiguous complex128 CUDA tensor, Cs [nb, k, k]."""
    import torch
    Xs = _dev_blocks(Xs)
    if not Y.is_contiguous():
        raise ValidationError("block_add_scaled: Y must be contiguous")
    n, k = Xs[0].shape
    nb = len(Xs)
    Cs = np.ascontiguousarray(np.asarray(Cs, dtype=np.complex128).reshape(nb, k, k))
    ptrs = (C.c_void_p * nb)(*[x.data_ptr() for x in Xs])
    torch.cuda.synchronize()
    with torch.cuda.device(Y.device):
        _check(_native.lib().hz_block_add_scaled_device(n, k, nb, ptrs, Cs.ctypes.data, Y.data_ptr()))
    return Y


class MultiFrequencySolver:
    """Several (m, omega) hierarchies resident on one GPU: one
    HelmholtzProblem + HelmholtzSolver per frequency over the same slowness
    squared m and attenuation, solved as one concurrent batch. The caller is
    the frequency-continuation loop (Algorithm 1)."""

    def __init__(self, ndim, n, h, m, omegas: Sequence[float], gamma: "AttenuationField",
                 options: Optional["HelmholtzSolveOptions"] = None, allow_coarse_ppw: bool = False,
                 device: int = 0):
        self.omegas = [float(w) for w in omegas]
        self.problems = [HelmholtzProblem(ndim, n, h, m, w, gamma, allow_coarse_ppw=allow_coarse_ppw,
                                          device=device) for w in self.omegas]
        self.solvers = [HelmholtzSolver(P, options) for P in self.problems]

    def __len__(self):
        return len(self.solvers)

    def solve_blocks(self, Bs, outs=None):
        """X_f = A(m, omega_f)^{-1} B_f for every frequency f, concurrently."""
        return solve_blocks_multi(self.solvers, Bs, outs)


class kernel_profile:
    """Context manager: CUDA-event timing of every library kernel launched
    inside the block. `.result` maps kernel name -> {count, ms, bytes, flops}
    (summed event durations and algorithmic bytes / flops); with
    trace=True, `.trace` lists [name, stream, start_ms, dur_ms, bytes] per
    launch (hz_profile_trace)."""

    def __init__(self, trace: bool = False):
        self.want_trace = trace

    def __enter__(self):
        _check(_native.lib().hz_profile_begin())
        self.result = {}
        return self

    def __exit__(self, *exc):
        import json
        L = _native.lib()
        _check(L.hz_profile_end())
        need = L.hz_profile_report(None, 0)
        if need < 0:
            raise CudaError(L.hz_last_error_message().decode())
        buf = C.create_string_buffer(int(need))
        L.hz_profile_report(buf, need)
        self.result = json.loads(buf.value.decode())
        if getattr(self, "want_trace", False):
            need = L.hz_profile_trace(None, 0)
            buf = C.create_string_buffer(int(need))
            L.hz_profile_trace(buf, need)
            self.trace = json.loads(buf.value.decode())
        return False


# ---------------------------------------------------------------- data
def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _host_block(a, n: int) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.complex128)
    if a.ndim == 1:
        a = a.reshape(n, 1)
    if a.ndim != 2 or a.shape[0] != n:
        raise ValidationError(f"block must be [n={n}][k] complex, got shape {a.shape}")
    return a


def _dev_block(t, n: int, device: Optional[int] = None):
    import torch
    if t.dtype != torch.complex128 or not t.is_cuda:
        raise ValidationError("device blocks must be complex128 CUDA tensors")
    if device is not None and t.device.index != device:
        raise ValidationError(f"block is on cuda:{t.device.index}, the solver on cuda:{device}")
    if t.dim() == 1:
        t = t.reshape(n, 1)
    if t.dim() != 2 or t.shape[0] != n:
        raise ValidationError(f"block must be [n={n}][k], got {tuple(t.shape)}")
    return t.contiguous()


def _check_out(out, B, dev: bool):
    """A caller-supplied solution buffer must be exactly what the C library
    writes n*k*16 bytes into: complex128, B's [n][k] shape, C-contiguous, on
    B's side (host / the same device) and not overlapping B (the solve zeroes
    X before it reads B, src/krylov.cpp:178-200)."""
    if dev:
        import torch
        if not _is_torch(out) or out.dtype != torch.complex128 or not out.is_cuda:
            raise ValidationError("out must be a complex128 CUDA tensor for a device block")
        if out.device != B.device:
            raise ValidationError(f"out is on {out.device}, B on {B.device}")
        if tuple(out.shape) != tuple(B.shape) or not out.is_contiguous():
            raise ValidationError(f"out must be a contiguous [n][k] = {tuple(B.shape)} tensor")
        a0, a1 = out.data_ptr(), out.data_ptr() + out.numel() * 16
        b0, b1 = B.data_ptr(), B.data_ptr() + B.numel() * 16
        if a0 < b1 and b0 < a1:
            raise ValidationError("out must not share memory with B")
        return out
    if _is_torch(out) or not isinstance(out, np.ndarray):
        raise ValidationError("out must be a numpy complex128 array for a host block")
    if out.dtype != np.complex128 or out.shape != B.shape or not out.flags["C_CONTIGUOUS"] \
            or not out.flags["WRITEABLE"]:
        raise ValidationError(f"out must be a writeable C-contiguous complex128 [n][k] = {B.shape} array")
    if np.shares_memory(out, B):
        raise ValidationError("out must not share memory with B")
    return out


@dataclasses.dataclass
class AttenuationField:
    """AttenuationField (inc/attenuation.hpp:11-22): gamma(omega) = base + omega*ramp."""
    base: float
    ramp: np.ndarray


@dataclasses.dataclass
class SolveReport:
    """seistomo::SolveReport (inc/krylov.hpp:19-40)."""
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

    def mean_col_cycles(self) -> float:
        return float(np.mean(self.col_cycles)) if len(self.col_cycles) else 0.0


class HelmholtzProblem:
    """HelmholtzProblem (inc/helmholtz.hpp:19-57): A = Lap_h + w^2 (1 - i gamma/w) m,
    5-point (2D) / 7-point (3D), truncated (Dirichlet) boundary rows."""

    def __init__(self, ndim: int, n: Sequence[int], h: Sequence[float], m, omega: float,
                 gamma: AttenuationField, allow_coarse_ppw: bool = False, device: int = 0,
                 origin: Sequence[float] = (0.0, 0.0, 0.0), stencil: int = 7):
        n3 = list(n) + [1] * (3 - len(n))
        h3 = list(h) + [1.0] * (3 - len(h))
        self.ndim = int(ndim)
        self.n = tuple(int(x) for x in n3)
        if self.ndim == 2:
            self.n = (self.n[0], self.n[1], 1)
        self.h = tuple(float(x) for x in h3)
        self.omega = float(omega)
        self.num_nodes = self.n[0] * self.n[1] * self.n[2]
        self.device = int(device)
        self.origin = tuple(float(x) for x in (list(origin) + [0.0] * (3 - len(origin)))[:3])
        m = np.ascontiguousarray(m, dtype=np.float64).reshape(-1)
        ramp = np.ascontiguousarray(gamma.ramp, dtype=np.float64).reshape(-1)
        if m.size != self.num_nodes or ramp.size != self.num_nodes:
            raise ValidationError("model / attenuation size does not match grid")
        self.m = m
        self.gamma = AttenuationField(float(gamma.base), ramp)
        nn = np.asarray(self.n, dtype=np.int64)
        hh = np.asarray(self.h, dtype=np.float64)
        out = C.c_void_p()
        self.stencil = int(stencil)
        _check(_native.lib().hz_problem_create_ex(self.ndim, nn.ctypes.data, hh.ctypes.data, m.ctypes.data,
                                                  self.omega, self.gamma.base, ramp.ctypes.data,
                                                  1 if allow_coarse_ppw else 0, self.device, self.stencil,
                                                  C.byref(out)))
        self._h = out

    @classmethod
    def from_config(cls, cfg, device: int = 0, allow_coarse_ppw: bool = False):
        return cls(cfg.ndim, cfg.n, cfg.h, cfg.m, cfg.omega, AttenuationField(cfg.gamma_base, cfg.ramp),
                   allow_coarse_ppw=allow_coarse_ppw, device=device, stencil=getattr(cfg, "stencil", 7))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _native.lib().hz_problem_destroy(h)
            except Exception:
                pass
            self._h = None

    def points_per_wavelength(self) -> float:
        v = C.c_double()
        _check(_native.lib().hz_problem_ppw(self._h, C.byref(v)))
        return float(v.value)

    def gamma_factor(self) -> np.ndarray:
        """(1 - i gamma/omega) per node (HelmholtzProblem::gamma_factor)."""
        out = np.empty(self.num_nodes, np.complex128)
        _check(_native.lib().hz_problem_gamma_factor(self._h, out.ctypes.data))
        return out

    def apply_block(self, u):
        """v = A u (HelmholtzProblem::apply_block, src/helmholtz.cpp:71-100)."""
        if _is_torch(u):
            import torch
            u = _dev_block(u, self.num_nodes)
            out = torch.empty_like(u)
            stream = torch.cuda.current_stream(u.device).cuda_stream
            _check(_native.lib().hz_apply_block_device(self._h, self.num_nodes, u.shape[1], u.data_ptr(),
                                                       out.data_ptr(), stream))
            return out
        u = _host_block(u, self.num_nodes)
        out = np.empty_like(u)
        _check(_native.lib().hz_apply_block(self._h, self.num_nodes, u.shape[1], u.ctypes.data,
                                            out.ctypes.data))
        return out

    def _xyz(self, x) -> np.ndarray:
        xx = np.zeros(3, np.float64)
        xx[:len(x)] = np.asarray(x, dtype=np.float64)
        return xx

    def nearest_node(self, x: Sequence[float]) -> int:
        """RegularGrid::nearest_node (src/grid.cpp:46-55) on this grid at
        `origin`: exact half-spacing ties go to the lower index."""
        node = C.c_int64()
        o = np.ascontiguousarray(self.origin, np.float64)
        _check(_native.lib().hz_problem_nearest_node(self._h, o.ctypes.data, self._xyz(x).ctypes.data,
                                                     C.byref(node)))
        return int(node.value)

    def point_source(self, x: Sequence[float], amplitude: complex = 1.0) -> np.ndarray:
        """FV point source amp/prod(h) at the nearest node, ties to the lower
        index (HelmholtzProblem::point_source, src/helmholtz.cpp:124-132);
        ValidationError outside the grid (RegularGrid::contains)."""
        q = np.empty(self.num_nodes, dtype=np.complex128)
        o = np.ascontiguousarray(self.origin, np.float64)
        a = complex(amplitude)
        _check(_native.lib().hz_problem_point_source(self._h, o.ctypes.data, self._xyz(x).ctypes.data, a.real,
                                                     a.imag, q.ctypes.data))
        return q

    def point_sources(self, xs, amplitudes=None):
        """k point sources as one device block [n][k] (complex128 CUDA tensor,
        column j = point_source(xs[j], amplitudes[j])), zero-filled and
        scattered on the GPU (hz_point_sources_device)."""
        import torch
        xs = np.asarray(xs, dtype=np.float64)
        k = xs.shape[0]
        xyz = np.zeros((k, 3), np.float64)
        xyz[:, :xs.shape[1]] = xs
        amp = None
        if amplitudes is not None:
            amp = np.ascontiguousarray(np.asarray(amplitudes, dtype=np.complex128).reshape(k))
        B = torch.empty((self.num_nodes, k), dtype=torch.complex128, device=f"cuda:{self.device}")
        o = np.ascontiguousarray(self.origin, np.float64)
        stream = torch.cuda.current_stream(B.device).cuda_stream
        _check(_native.lib().hz_point_sources_device(self._h, o.ctypes.data, k, xyz.ctypes.data,
                                                     None if amp is None else amp.ctypes.data, B.data_ptr(),
                                                     stream))
        return B

    def mass(self) -> np.ndarray:
        """omega^2 (1 - i gamma/omega) m per node (HelmholtzProblem::mass)."""
        out = np.empty(self.num_nodes, np.complex128)
        _check(_native.lib().hz_problem_mass(self._h, out.ctypes.data))
        return out

    def to_csr(self, shift_factor: float = 0.0):
        """HelmholtzProblem::to_csr (src/helmholtz.cpp:102-122) as
        (row_ptr int64, col int32, values complex128)."""
        nnz = C.c_int64()
        L = _native.lib()
        _check(L.hz_problem_to_csr(self._h, float(shift_factor), None, None, None, 0, C.byref(nnz)))
        rp = np.empty(self.num_nodes + 1, np.int64)
        ci = np.empty(nnz.value, np.int32)
        v = np.empty(nnz.value, np.complex128)
        _check(L.hz_problem_to_csr(self._h, float(shift_factor), rp.ctypes.data, ci.ctypes.data, v.ctypes.data,
                                   nnz.value, C.byref(nnz)))
        return rp, ci, v


_METHODS = {"MgBicgstab": 0, "MgFgmresW": 1, "MgFgmresK": 2, "DenseLuSmall": 3, "MgFgmres": 4,
            "MgBicgstabCycle": 5}
_KINDS = {"V": 0, "W": 1, "K": 2}


@dataclasses.dataclass
class CycleSpec:
    """CycleSpec (inc/multigrid.hpp:17-23)."""
    kind: str = "W"
    pre: int = 2
    post: int = 2
    jacobi_weight: float = 0.8
    k_inner: int = 2


@dataclasses.dataclass
class HelmholtzSolveOptions:
    """HelmholtzSolveOptions (inc/helmholtz_solver.hpp:14-24). `method` adds
    "MgFgmres" / "MgBicgstabCycle" (cycle kind taken from cycle.kind, the
    SURVEY §3.3 composition) and `precond_precision` ("c128" | "c64")."""
    method: str = "MgBicgstab"
    tol: float = 1e-6
    max_cycles: int = 200
    nlevels: int = 3
    shift_factor: float = 0.2
    cycle: CycleSpec = dataclasses.field(default_factory=CycleSpec)
    fgmres_restart: int = 5
    dense_threshold: int = 3000
    allow_coarse_ppw: bool = False
    precond_precision: str = "c128"
    # 0: one block Krylov solve over all k columns (the reference's
    # solve_block); b > 0: ceil(k/b) independent block solves of <= b
    # contiguous columns, run concurrently on the GPU (hz_options.rhs_block)
    rhs_block: int = 0

    def to_c(self) -> hz_options:
        o = hz_options()
        if self.method not in _METHODS:
            raise ValidationError(f"unknown method {self.method}")
        if self.cycle.kind not in _KINDS:
            raise ValidationError(f"unknown cycle kind {self.cycle.kind}")
        if self.precond_precision not in ("c128", "c64"):
            raise ValidationError("precond_precision must be c128 or c64")
        o.method = _METHODS[self.method]
        o.tol = self.tol
        o.max_cycles = self.max_cycles
        o.nlevels = self.nlevels
        o.shift_factor = self.shift_factor
        o.cycle_kind = _KINDS[self.cycle.kind]
        o.pre = self.cycle.pre
        o.post = self.cycle.post
        o.jacobi_weight = self.cycle.jacobi_weight
        o.k_inner = self.cycle.k_inner
        o.fgmres_restart = self.fgmres_restart
        o.dense_threshold = self.dense_threshold
        o.precond_precision = 0 if self.precond_precision == "c128" else 1
        if self.rhs_block < 0:
            raise ValidationError("rhs_block must be >= 0")
        o.rhs_block = self.rhs_block
        return o

    @classmethod
    def from_config(cls, cfg, **over):
        kind = cfg.cycle
        method = "MgFgmres" if cfg.method == "fgmres" else "MgBicgstabCycle"
        o = cls(method=method, tol=cfg.tol, max_cycles=cfg.max_cycles, nlevels=cfg.nlevels,
                shift_factor=cfg.shift, cycle=CycleSpec(kind, cfg.pre, cfg.post, cfg.jacobi_weight),
                fgmres_restart=cfg.restart, precond_precision=cfg.precond_precision,
                rhs_block=cfg.krylov_block)
        for k, v in over.items():
            setattr(o, k, v)
        return o


class HelmholtzSolver:
    """HelmholtzSolver (inc/helmholtz_solver.hpp:30-55): the multigrid
    hierarchy is built once per (m, omega) on the GPU and reused for every
    block of right-hand sides."""

    def __init__(self, problem: HelmholtzProblem, options: Optional[HelmholtzSolveOptions] = None):
        self.problem = problem
        self.options = options or HelmholtzSolveOptions()
        self._opts = self.options.to_c()
        out = C.c_void_p()
        _check(_native.lib().hz_solver_create(problem._h, C.byref(self._opts), C.byref(out)))
        self._h = out

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _native.lib().hz_solver_destroy(h)
            except Exception:
                pass
            self._h = None

    def set_tolerance(self, tol: float):
        self.options.tol = tol
        _check(_native.lib().hz_solver_set_tolerance(self._h, tol))

    def set_slabs(self, nparts: int, devices=None):
        """Slab-decompose every following solve / cycle along the slow grid
        axis over `nparts` parts (config 5): part p runs on GPU
        devices[p] (default: all on the problem's GPU as separate streams).
        nparts=1 with devices=None returns to the single-stream solver."""
        if devices is None:
            arr = None
        else:
            devs = np.ascontiguousarray(devices, dtype=np.int32)
            if devs.size != nparts:
                raise ValidationError("set_slabs: one device per part")
            arr = devs
        _check(_native.lib().hz_solver_set_slabs(
            self._h, int(nparts), None if arr is None else arr.ctypes.data_as(C.c_void_p)))
        self._slab_devices = arr

    def slab_info(self):
        """(nparts, agg_level, planes) with planes[l][p] the first plane of
        part p on level l and planes[l][nparts] the level's plane count."""
        P = C.c_int(0)
        agg = C.c_int(0)
        _check(_native.lib().hz_solver_slab_info(self._h, C.byref(P), C.byref(agg), None, 0))
        nl = C.c_int(0)
        _check(_native.lib().hz_hierarchy_num_levels(self._h, C.byref(nl)))
        planes = np.zeros((max(nl.value, 1), P.value + 1), np.int64)
        _check(_native.lib().hz_solver_slab_info(self._h, C.byref(P), C.byref(agg),
                                                 planes.ctypes.data_as(C.c_void_p), planes.size))
        return P.value, agg.value, planes

    def _report(self, k: int, cap: int):
        cc = np.zeros(k, np.int32)
        rr = np.zeros(k, np.float64)
        cv = np.zeros(k, np.int32)
        hist = np.zeros(cap, np.float64)
        rep = hz_report()
        rep.col_cycles = cc.ctypes.data_as(C.POINTER(C.c_int))
        rep.rel_residual = rr.ctypes.data_as(C.POINTER(C.c_double))
        rep.converged = cv.ctypes.data_as(C.POINTER(C.c_int))
        rep.history = hist.ctypes.data_as(C.POINTER(C.c_double))
        rep.history_cap = cap
        return rep, (cc, rr, cv, hist)

    @staticmethod
    def _finish(rep, bufs) -> SolveReport:
        cc, rr, cv, hist = bufs
        return SolveReport(cycles=rep.cycles, col_cycles=cc.copy(), rel_residual=rr.copy(),
                           converged=cv.astype(bool), history=hist[:min(rep.history_len, len(hist))].copy(),
                           wall_s=rep.wall_s, qr_factorizations=rep.qr_factorizations,
                           block_gram_products=rep.block_gram_products)

    def solve_block(self, B, out=None) -> Tuple[object, SolveReport]:
        """HelmholtzSolver::solve_block (src/helmholtz_solver.cpp:35-72)."""
        n = self.problem.num_nodes
        cap = self.options.max_cycles + 8
        if _is_torch(B):
            import torch
            B = _dev_block(B, n, self.problem.device)
            X = _check_out(out, B, dev=True) if out is not None else torch.empty_like(B)
            rep, bufs = self._report(B.shape[1], cap)
            stream = torch.cuda.current_stream(B.device).cuda_stream
            _check(_native.lib().hz_solve_block_device_stream(self._h, n, B.shape[1], B.data_ptr(), X.data_ptr(),
                                                              C.byref(rep), stream))
            return X, self._finish(rep, bufs)
        B = _host_block(B, n)
        X = _check_out(out, B, dev=False) if out is not None else np.empty_like(B)
        rep, bufs = self._report(B.shape[1], cap)
        _check(_native.lib().hz_solve_block(self._h, n, B.shape[1], B.ctypes.data, X.ctypes.data,
                                            C.byref(rep)))
        return X, self._finish(rep, bufs)

    def solve(self, rhs):
        """HelmholtzSolver::solve (src/helmholtz_solver.cpp:74-79)."""
        X, rep = self.solve_block(np.asarray(rhs).reshape(-1, 1))
        return X[:, 0].copy(), rep

    def cycle(self, b):
        """One preconditioner application from x = 0 (out := 0;
        MgHierarchy::cycle, src/helmholtz_solver.cpp:65-68)."""
        n = self.problem.num_nodes
        if _is_torch(b):
            import torch
            b = _dev_block(b, n, self.problem.device)
            x = torch.empty_like(b)
            stream = torch.cuda.current_stream(b.device).cuda_stream
            _check(_native.lib().hz_cycle_device_stream(self._h, n, b.shape[1], b.data_ptr(), x.data_ptr(), stream))
            return x
        b = _host_block(b, n)
        x = np.empty_like(b)
        _check(_native.lib().hz_cycle(self._h, n, b.shape[1], b.ctypes.data, x.ctypes.data))
        return x

    def num_levels(self) -> int:
        v = C.c_int()
        _check(_native.lib().hz_hierarchy_num_levels(self._h, C.byref(v)))
        return int(v.value)

    def level_dims(self, level: int):
        d = np.zeros(3, np.int64)
        _check(_native.lib().hz_hierarchy_level_dims(self._h, level, d.ctypes.data))
        return tuple(int(x) for x in d)

    def level_coefficients(self, level: int) -> np.ndarray:
        """level 0: shifted centre [n]; level >= 1: Galerkin planes [3^ndim][n]."""
        d = self.level_dims(level)
        nn = d[0] * d[1] * d[2]
        count = nn if level == 0 else nn * (27 if self.problem.ndim == 3 else 9)
        out = np.empty(count, np.complex128)
        _check(_native.lib().hz_hierarchy_level_coefficients(self._h, level, out.ctypes.data, count))
        return out if level == 0 else out.reshape(-1, nn)

    def coarse_solve(self, b) -> np.ndarray:
        """MgHierarchy::coarse_solve (src/multigrid.cpp:114-117)."""
        b = np.ascontiguousarray(b, dtype=np.complex128)
        if b.ndim == 1:
            b = b.reshape(-1, 1)
        x = np.empty_like(b)
        _check(_native.lib().hz_coarse_solve(self._h, b.shape[0], b.shape[1], b.ctypes.data, x.ctypes.data))
        return x


def fwi_sensitivity_output(problem: HelmholtzProblem, U, L, g=None):
    """sum_s fwi_sensitivity_output(problem, u_s, lambda_s)
    (src/helmholtz_solver.cpp:103-111): g[i] = sum_s Re(-w^2 (1 - i gamma/w) u_s lambda_s).
    Host numpy or device torch blocks; g accumulates when given."""
    n = problem.num_nodes
    if _is_torch(U):
        import torch
        U = _dev_block(U, n)
        L = _dev_block(L, n)
        acc = g is not None
        if g is None:
            g = torch.empty(n, dtype=torch.float64, device=U.device)
        stream = torch.cuda.current_stream(U.device).cuda_stream
        _check(_native.lib().hz_sensitivity_accumulate_device(problem._h, n, U.shape[1], U.data_ptr(),
                                                              L.data_ptr(), g.data_ptr(), 1 if acc else 0,
                                                              stream))
        return g
    U = _host_block(U, n)
    L = _host_block(L, n)
    acc = g is not None
    if g is None:
        g = np.empty(n, np.float64)
    _check(_native.lib().hz_sensitivity_accumulate(problem._h, n, U.shape[1], U.ctypes.data, L.ctypes.data,
                                                   g.ctypes.data, 1 if acc else 0))
    return g


# FWI path either side of the solve and wavefield output
from .fwi import (Compact16, Full32, SamplingOperator, WavefieldBatch, compact16,  # noqa: E402
                  fwi_jacobian_transpose_vec, fwi_jacobian_vec, fwi_sensitivity_rhs, solve_helmholtz)
