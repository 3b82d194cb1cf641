"""The steps either side of the block solve in FWI and wavefield output
(SURVEY §8f.1 and §8f.3), mirroring the reference's API:

* SamplingOperator (inc/acquisition.hpp:30-62): receiver gather P^T u and
  scatter P d as GPU kernels (hz_sample*), bitwise the reference's sums;
* fwi_sensitivity_rhs / fwi_jacobian_vec / fwi_jacobian_transpose_vec
  (src/helmholtz_solver.cpp:95-139), batched over k sources as ONE block
  solve (k = 1 is the reference function exactly);
* WavefieldBatch with StoragePrecision Full32 / Compact16 and the JSWF1 file
  format (inc/helmholtz.hpp:59-91, src/helmholtz.cpp:137-233); Compact16
  quantisation runs on the GPU, so a Compact16 solve returns 4 bytes per
  entry to the host instead of 16;
* solve_helmholtz (src/helmholtz_solver.cpp:81-93).

The JSWF1 writer / reader are file-format code on the host (numpy binary16 is
IEEE round-to-nearest-even, the reference's float_to_half).
"""
import ctypes as C
from typing import List, Optional

import numpy as np

from . import (ConvergenceError, HelmholtzProblem, HelmholtzSolver, IoError, SolveReport, StateError,
               ValidationError, _check, _dev_block, _host_block, _is_torch, _native)

Full32 = "Full32"
Compact16 = "Compact16"


class SamplingOperator:
    """SamplingOperator(AcquisitionGeometry, grid): receivers at physical
    points xyz [nrec][3] (h-scaled, relative to `origin`), multilinear weights
    over the <= 2^ndim enclosing nodes (src/acquisition.cpp:33-62)."""

    def __init__(self, problem: HelmholtzProblem, receivers_xyz, origin=(0.0, 0.0, 0.0)):
        xyz = np.ascontiguousarray(receivers_xyz, dtype=np.float64).reshape(-1, 3)
        org = np.ascontiguousarray(list(origin) + [0.0] * (3 - len(origin)), dtype=np.float64)
        out = C.c_void_p()
        _check(_native.lib().hz_sampling_create(problem._h, org.ctypes.data, xyz.shape[0], xyz.ctypes.data,
                                                C.byref(out)))
        self._h = out
        self.problem = problem
        self.num_receivers = int(xyz.shape[0])

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _native.lib().hz_sampling_destroy(h)
            except Exception:
                pass
            self._h = None

    def receiver(self, r: int):
        """(nodes, weights) of receiver r (receiver_nodes / receiver_weights)."""
        nodes = np.zeros(8, np.int64)
        w = np.zeros(8, np.float64)
        c = C.c_int(0)
        _check(_native.lib().hz_sampling_receiver(self._h, int(r), nodes.ctypes.data, w.ctypes.data, C.byref(c)))
        return nodes[:c.value].copy(), w[:c.value].copy()

    def sample(self, U):
        """P^T U: [n] or [n][k] -> [nrec] or [nrec][k] (numpy or CUDA tensor)."""
        n = self.problem.num_nodes
        one = getattr(U, "ndim", 2) == 1
        if _is_torch(U):
            import torch
            U = _dev_block(U, n)
            D = torch.empty((self.num_receivers, U.shape[1]), dtype=torch.complex128, device=U.device)
            stream = torch.cuda.current_stream(U.device).cuda_stream
            _check(_native.lib().hz_sample_device(self._h, U.shape[1], U.data_ptr(), D.data_ptr(), stream))
            return D[:, 0] if one else D
        U = _host_block(U, n)
        D = np.empty((self.num_receivers, U.shape[1]), np.complex128)
        _check(_native.lib().hz_sample(self._h, U.shape[1], U.ctypes.data, D.ctypes.data))
        return D[:, 0].copy() if one else D

    def sample_adjoint(self, D, conj: bool = False):
        """P D (or P conj(D)): [nrec] or [nrec][k] -> [n] or [n][k]."""
        n = self.problem.num_nodes
        one = getattr(D, "ndim", 2) == 1
        if _is_torch(D):
            import torch
            D = D.reshape(self.num_receivers, -1).contiguous()
            U = torch.empty((n, D.shape[1]), dtype=torch.complex128, device=D.device)
            stream = torch.cuda.current_stream(D.device).cuda_stream
            _check(_native.lib().hz_sample_adjoint_device(self._h, D.shape[1], D.data_ptr(), U.data_ptr(),
                                                          1 if conj else 0, stream))
            return U[:, 0] if one else U
        D = np.ascontiguousarray(D, dtype=np.complex128).reshape(self.num_receivers, -1)
        U = np.empty((n, D.shape[1]), np.complex128)
        _check(_native.lib().hz_sample_adjoint(self._h, D.shape[1], D.ctypes.data, U.ctypes.data, 1 if conj else 0))
        return U[:, 0].copy() if one else U


def _report(solver: HelmholtzSolver, k: int):
    return solver._report(k, solver.options.max_cycles + 8)


def _finish_or_raise(solver, status, rep, bufs):
    r = HelmholtzSolver._finish(rep, bufs)
    if status == ConvergenceError.code:
        msg = _native.lib().hz_last_error_message().decode(errors="replace")
        raise ConvergenceError(msg, r.history)
    _check(status)
    return r


def fwi_sensitivity_rhs(problem: HelmholtzProblem, U, v):
    """-w^2 (1 - i gamma/w) U v (src/helmholtz_solver.cpp:95-101), U [n] or
    [n][k] (sources), v real [n]; on the GPU."""
    import torch
    n = problem.num_nodes
    host = not _is_torch(U)
    dev = f"cuda:{problem.device}"
    one = getattr(U, "ndim", 2) == 1
    Ut = torch.from_numpy(_host_block(U, n)).to(dev) if host else _dev_block(U, n)
    vt = torch.as_tensor(np.ascontiguousarray(v, np.float64) if not _is_torch(v) else v,
                         dtype=torch.float64, device=Ut.device).contiguous()
    R = torch.empty_like(Ut)
    stream = torch.cuda.current_stream(Ut.device).cuda_stream
    _check(_native.lib().hz_fwi_sensitivity_rhs_device(problem._h, n, Ut.shape[1], Ut.data_ptr(), vt.data_ptr(),
                                                       R.data_ptr(), stream))
    if host:
        R = R.cpu().numpy()
        return R[:, 0].copy() if one else R
    return R[:, 0] if one else R


def fwi_jacobian_vec(solver: HelmholtzSolver, U, P: SamplingOperator, v, report: Optional[list] = None):
    """fwi_jacobian_vec (src/helmholtz_solver.cpp:113-125): P^T A^{-1}
    (-w^2 gf u v) for the stored field(s) U ([n] or [n][k], one block solve).
    ConvergenceError (with the residual history) if the solve misses tol."""
    n = solver.problem.num_nodes
    one = getattr(U, "ndim", 2) == 1
    if _is_torch(U):
        import torch
        U = _dev_block(U, n)
        vt = torch.as_tensor(v, dtype=torch.float64, device=U.device).contiguous()
        D = torch.empty((P.num_receivers, U.shape[1]), dtype=torch.complex128, device=U.device)
        rep, bufs = _report(solver, U.shape[1])
        torch.cuda.current_stream(U.device).synchronize()
        st = _native.lib().hz_fwi_jacobian_vec_device(solver._h, P._h, n, U.shape[1], U.data_ptr(), vt.data_ptr(),
                                                      D.data_ptr(), C.byref(rep))
    else:
        if np.asarray(v).size != n:
            raise ValidationError("fwi_jacobian_vec: model vector size mismatch")
        U = _host_block(U, n)
        vv = np.ascontiguousarray(v, dtype=np.float64)
        D = np.empty((P.num_receivers, U.shape[1]), np.complex128)
        rep, bufs = _report(solver, U.shape[1])
        st = _native.lib().hz_fwi_jacobian_vec(solver._h, P._h, n, U.shape[1], U.ctypes.data, vv.ctypes.data,
                                               D.ctypes.data, C.byref(rep))
    r = _finish_or_raise(solver, st, rep, bufs)
    if report is not None:
        report.append(r)
    return D[:, 0] if one else D


def fwi_jacobian_transpose_vec(solver: HelmholtzSolver, U, P: SamplingOperator, W, g=None,
                               report: Optional[list] = None):
    """fwi_jacobian_transpose_vec (src/helmholtz_solver.cpp:127-139) summed
    over the k sources of U [n][k] / W [nrec][k]: g[n] (+)= sum_s
    Re(-w^2 gf u_s lambda_s), lambda_s = A^{-1} P conj(w_s)."""
    n = solver.problem.num_nodes
    if _is_torch(U):
        import torch
        U = _dev_block(U, n)
        W = W.reshape(P.num_receivers, -1).contiguous()
        acc = g is not None
        if g is None:
            g = torch.empty(n, dtype=torch.float64, device=U.device)
        rep, bufs = _report(solver, U.shape[1])
        torch.cuda.current_stream(U.device).synchronize()
        st = _native.lib().hz_fwi_jacobian_transpose_vec_device(solver._h, P._h, n, U.shape[1], U.data_ptr(),
                                                                W.data_ptr(), g.data_ptr(), 1 if acc else 0,
                                                                C.byref(rep))
    else:
        U = _host_block(U, n)
        W = np.ascontiguousarray(W, dtype=np.complex128).reshape(P.num_receivers, -1)
        if W.shape[1] != U.shape[1]:
            raise ValidationError("fwi_jacobian_transpose_vec: one receiver vector per field")
        acc = g is not None
        if g is None:
            g = np.empty(n, np.float64)
        rep, bufs = _report(solver, U.shape[1])
        st = _native.lib().hz_fwi_jacobian_transpose_vec(solver._h, P._h, n, U.shape[1], U.ctypes.data,
                                                         W.ctypes.data, g.ctypes.data, 1 if acc else 0,
                                                         C.byref(rep))
    r = _finish_or_raise(solver, st, rep, bufs)
    if report is not None:
        report.append(r)
    return g


# ---------------------------------------------------------------- wavefields
def compact16(X):
    """Compact16 quantisation (WavefieldBatch::append, src/helmholtz.cpp:143-151)
    of the columns of X [n][k] on the GPU: (Q uint16 [k][n][2], scales [k])."""
    if _is_torch(X):
        import torch
        X = X.reshape(X.shape[0], -1).contiguous()
        n, k = X.shape
        Q = torch.empty((k, n, 2), dtype=torch.int16, device=X.device)
        scales = np.empty(k, np.float64)
        stream = torch.cuda.current_stream(X.device).cuda_stream
        _check(_native.lib().hz_compact16_device(n, k, X.data_ptr(), Q.data_ptr(), scales.ctypes.data, stream))
        return Q.cpu().numpy().view(np.uint16), scales
    X = np.ascontiguousarray(X, dtype=np.complex128)
    if X.ndim == 1:
        X = X.reshape(-1, 1)
    n, k = X.shape
    Q = np.empty((k, n, 2), np.uint16)
    scales = np.empty(k, np.float64)
    _check(_native.lib().hz_compact16(n, k, X.ctypes.data, Q.ctypes.data, scales.ctypes.data))
    return Q, scales


class WavefieldBatch:
    """Solved wavefields of a batch of sources (inc/helmholtz.hpp:59-91):
    Full32 keeps complex128, Compact16 keeps binary16 (re, im) against a
    per-source power-of-two scale."""

    def __init__(self, num_nodes: int, precision: str = Full32):
        if precision not in (Full32, Compact16):
            raise ValidationError(f"unknown storage precision {precision}")
        self.num_nodes = int(num_nodes)
        self.precision = precision
        self._ids: List[int] = []
        self._full: List[np.ndarray] = []
        self._q: List[np.ndarray] = []
        self._scale: List[float] = []

    def append(self, source_id: int, u):
        self.append_block([source_id], np.asarray(u).reshape(-1, 1) if not _is_torch(u) else u.reshape(-1, 1))

    def append_block(self, source_ids, X):
        """Append the columns of X [n][k] (quantised on the GPU for Compact16)."""
        n = self.num_nodes
        if X.shape[0] != n:
            raise ValidationError("wavefield batch: field size mismatch")
        if self.precision == Full32:
            Xh = X.cpu().numpy() if _is_torch(X) else np.asarray(X, dtype=np.complex128)
            for c, s in enumerate(source_ids):
                self._ids.append(int(s))
                self._full.append(np.ascontiguousarray(Xh[:, c], dtype=np.complex128))
            return
        Q, scales = compact16(X)
        for c, s in enumerate(source_ids):
            self._ids.append(int(s))
            self._q.append(Q[c])
            self._scale.append(float(scales[c]))

    def __len__(self):
        return len(self._ids)

    def size(self) -> int:
        return len(self._ids)

    def source_id(self, idx: int) -> int:
        return self._ids[idx]

    def field(self, idx: int) -> np.ndarray:
        if idx < 0 or idx >= len(self._ids):
            raise StateError("wavefield batch: no stored field at index")
        if self.precision == Full32:
            return self._full[idx].copy()
        q = self._q[idx].view(np.float16).astype(np.float64) * self._scale[idx]
        return q[:, 0] + 1j * q[:, 1]

    def save(self, path: str):
        """JSWF1 file: "JSWF1 <nsrc> <nnodes> <f32|f16>\\n" then per source the
        interleaved little-endian (re, im) in that precision
        (WavefieldBatch::save, src/helmholtz.cpp:164-195)."""
        tok = "f32" if self.precision == Full32 else "f16"
        try:
            with open(path, "wb") as f:
                f.write(f"JSWF1 {len(self)} {self.num_nodes} {tok}\n".encode())
                for s in range(len(self)):
                    u = self.field(s)
                    buf = np.empty(2 * self.num_nodes, np.float32)
                    buf[0::2] = u.real.astype(np.float32)
                    buf[1::2] = u.imag.astype(np.float32)
                    if tok == "f16":
                        buf = buf.astype(np.float16)
                    f.write(buf.astype(buf.dtype.newbyteorder("<"), copy=False).tobytes())
        except OSError as e:
            raise IoError(f"cannot open for write: {path}") from e

    @staticmethod
    def load(path: str, num_nodes: int) -> "WavefieldBatch":
        """WavefieldBatch::load (src/helmholtz.cpp:197-233): a Full32 batch."""
        try:
            with open(path, "rb") as f:
                header = f.readline().decode(errors="replace").split()
                if len(header) != 4 or header[0] != "JSWF1":
                    raise IoError(f"bad JSWF1 header: {path}")
                nsrc, nn, tok = int(header[1]), int(header[2]), header[3]
                if nn != num_nodes:
                    raise IoError(f"JSWF1 node count does not match grid: {path}")
                if tok not in ("f16", "f32"):
                    raise IoError(f"bad JSWF1 precision token: {path}")
                dt = np.dtype("<f2") if tok == "f16" else np.dtype("<f4")
                b = WavefieldBatch(nn, Full32)
                for s in range(nsrc):
                    raw = f.read(2 * nn * dt.itemsize)
                    if len(raw) != 2 * nn * dt.itemsize:
                        raise IoError(f"truncated JSWF1 payload: {path}")
                    v = np.frombuffer(raw, dt).astype(np.float64)
                    b.append(s, v[0::2] + 1j * v[1::2])
                return b
        except OSError as e:
            raise IoError(f"cannot open: {path}") from e


def solve_helmholtz(solver: HelmholtzSolver, rhs, precision: str = Full32,
                    report: Optional[list] = None) -> WavefieldBatch:
    """solve_helmholtz (src/helmholtz_solver.cpp:81-93): one block solve of
    the right-hand sides, ConvergenceError (with the residual history) if any
    column misses tol, returned as a WavefieldBatch. Compact16 quantises on the
    GPU and brings back 4 bytes per entry."""
    n = solver.problem.num_nodes
    B = np.stack([np.asarray(q, dtype=np.complex128).reshape(-1) for q in rhs], axis=1)
    k = B.shape[1]
    batch = WavefieldBatch(n, precision)
    if precision == Full32:
        X, rep = solver.solve_block(B)
        if not rep.all_converged():
            raise ConvergenceError("helmholtz solve: tolerance not met within cycle cap", rep.history)
        batch.append_block(list(range(k)), X)
    else:
        Q = np.empty((k, n, 2), np.uint16)
        scales = np.empty(k, np.float64)
        r, bufs = _report(solver, k)
        B = _host_block(B, n)
        st = _native.lib().hz_solve_helmholtz_compact16(solver._h, n, k, B.ctypes.data, Q.ctypes.data,
                                                        scales.ctypes.data, C.byref(r))
        rep = _finish_or_raise(solver, st, r, bufs)
        for c in range(k):
            batch._ids.append(c)
            batch._q.append(Q[c])
            batch._scale.append(float(scales[c]))
    if report is not None:
        report.append(rep)
    return batch
