"""Preconditioned CG consumer of ``apply_inverse`` (src/krylov.py:48-77).

The factor is used as the preconditioner exactly as the reference's bench does
(src/bench.py:169-171).  The matvec with A runs on the host here: Krylov
solvers are a consumer of the hot path, not part of it.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple

import numpy as np


@dataclass
class SolveReport:
    x: np.ndarray
    n_i: int
    residual: float
    converged: bool


def pcg(a, b, precond=None, tol: float = 1e-12, max_iter: int = 1000) -> SolveReport:
    """CG on ||b - A x|| / ||b|| <= tol with an SPD preconditioner callable."""
    pc = precond if precond is not None else (lambda v: v)
    b = np.asarray(b, dtype=float)
    bn = float(np.linalg.norm(b))
    if bn == 0.0:
        return SolveReport(np.zeros_like(b), 0, 0.0, True)
    x = np.zeros_like(b)
    r = b.copy()
    z = pc(r)
    p = z.copy()
    rz = float(r @ z)
    res = 1.0
    for it in range(1, max_iter + 1):
        ap = a @ p
        alpha = rz / float(p @ ap)
        x += alpha * p
        r -= alpha * ap
        res = float(np.linalg.norm(r)) / bn
        if res <= tol:
            return SolveReport(x, it, res, True)
        z = pc(r)
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return SolveReport(x, max_iter, res, False)


def pcg_gpu(f, a, b, tol: float = 1e-12, max_iter: int = 1000) -> SolveReport:
    """The same PCG run on the device (hifde_pcg): SpMV, dot products and
    updates in CUDA kernels, ``f.apply_inverse`` as the preconditioner without
    host round trips (the host reads one residual per iteration)."""
    import ctypes as C
    import scipy.sparse as sp

    csr = sp.csr_matrix(a) if not sp.isspmatrix_csr(a) else a
    ip = np.ascontiguousarray(csr.indptr, dtype=np.int64)
    ix = np.ascontiguousarray(csr.indices, dtype=np.int32)
    va = np.ascontiguousarray(csr.data, dtype=np.float64)
    bb = np.ascontiguousarray(np.asarray(b, dtype=np.float64))
    if bb.ndim != 1 or bb.shape[0] != f.n:
        raise ValueError("pcg_gpu takes one right-hand side of length N")
    x = np.empty_like(bb)
    it, res, conv = C.c_int(), C.c_double(), C.c_int()
    code = f._lib.hifde_pcg(f._h, ip.ctypes.data, ix.ctypes.data, va.ctypes.data, bb.ctypes.data,
                            x.ctypes.data, f.n, float(tol), int(max_iter), 0, None,
                            C.byref(it), C.byref(res), C.byref(conv))
    if code:
        from .driver import _raise
        _raise(f._lib, code)
    return SolveReport(x, int(it.value), float(res.value), bool(conv.value))


class EstimateResult(NamedTuple):
    """Power-iteration norm estimate (src/krylov.py:140-149)."""
    value: float
    converged: bool
    iterations: int

    def __float__(self) -> float:
        return self.value


POWER_ITER_RTOL = 1e-2
POWER_ITER_CAP = 512


def _power_norm_gpu(f, a, kind: int, seed) -> EstimateResult:
    import ctypes as C
    import scipy.sparse as sp

    csr = sp.csr_matrix(a) if not sp.isspmatrix_csr(a) else a
    ip = np.ascontiguousarray(csr.indptr, dtype=np.int64)
    ix = np.ascontiguousarray(csr.indices, dtype=np.int32)
    va = np.ascontiguousarray(csr.data, dtype=np.float64)
    rng = np.random.default_rng(seed)  # the reference's start vector
    x = rng.random(f.n)
    x /= np.linalg.norm(x)
    val, conv, it = C.c_double(), C.c_int(), C.c_int()
    code = f._lib.hifde_power_norm(f._h, ip.ctypes.data, ix.ctypes.data, va.ctypes.data, f.n, kind,
                                   x.ctypes.data, POWER_ITER_RTOL, POWER_ITER_CAP, C.byref(val), C.byref(conv),
                                   C.byref(it))
    if code:
        from .driver import _raise
        _raise(f._lib, code)
    return EstimateResult(float(val.value), bool(conv.value), int(it.value))


def estimate_apply_error(a, f, seed: int = 0) -> EstimateResult:
    """||A - F|| / ||A|| by power iteration on the device (src/krylov.py:173-186)."""
    num = _power_norm_gpu(f, a, 0, (seed, 0xA))
    den = _power_norm_gpu(f, a, 1, (seed, 0xB))
    value = num.value / den.value if den.value else np.inf
    return EstimateResult(value, num.converged and den.converged, num.iterations + den.iterations)


def estimate_solve_error(a, f, seed: int = 0) -> EstimateResult:
    """||I - A F^-1|| by power iteration on the device (src/krylov.py:189-201)."""
    return _power_norm_gpu(f, a, 2, (seed, 0xC))


def gmres(a, b, precond=None, tol: float = 1e-12, max_iter: int = 1000, restart: int = 32) -> SolveReport:
    """Right-preconditioned restarted GMRES (src/krylov.py:80-137 semantics):
    modified Gram-Schmidt Arnoldi on A M, Givens rotations on the Hessenberg
    matrix; n_i counts operator applications; stops on ||b - A x|| / ||b||."""
    M = precond if precond is not None else (lambda v: v)
    A = a.__matmul__ if hasattr(a, "__matmul__") else a
    b = np.asarray(b, dtype=float)
    bn = float(np.linalg.norm(b))
    if bn == 0.0:
        return SolveReport(np.zeros_like(b), 0, 0.0, True)
    x = np.zeros_like(b)
    its = 0
    while True:
        r = b - A(x)
        res = float(np.linalg.norm(r)) / bn
        if res <= tol:
            return SolveReport(x, its, res, True)
        if its >= max_iter:
            return SolveReport(x, its, res, False)
        m = min(restart, max_iter - its)
        V = np.zeros((m + 1, b.size))
        Hm = np.zeros((m + 1, m))
        c, sn = np.zeros(m), np.zeros(m)
        rhs = np.zeros(m + 1)
        beta = res * bn
        V[0] = r / beta
        rhs[0] = beta
        used = 0
        for j in range(m):
            w = A(M(V[j]))
            its += 1
            for i in range(j + 1):          # modified Gram-Schmidt
                Hm[i, j] = float(w @ V[i])
                w = w - Hm[i, j] * V[i]
            hn = float(np.linalg.norm(w))
            Hm[j + 1, j] = hn
            if hn != 0.0:
                V[j + 1] = w / hn
            for i in range(j):              # earlier rotations
                hi, hi1 = Hm[i, j], Hm[i + 1, j]
                Hm[i, j] = c[i] * hi + sn[i] * hi1
                Hm[i + 1, j] = -sn[i] * hi + c[i] * hi1
            rho = float(np.hypot(Hm[j, j], Hm[j + 1, j]))
            c[j], sn[j] = (1.0, 0.0) if rho == 0.0 else (Hm[j, j] / rho, Hm[j + 1, j] / rho)
            Hm[j, j], Hm[j + 1, j] = rho, 0.0
            rhs[j + 1] = -sn[j] * rhs[j]
            rhs[j] = c[j] * rhs[j]
            used = j + 1
            if abs(rhs[j + 1]) / bn <= tol or hn == 0.0:
                break
        y = np.zeros(used)
        for i in range(used - 1, -1, -1):   # back substitution on the rotated H
            y[i] = (rhs[i] - Hm[i, i + 1:used] @ y[i + 1:]) / Hm[i, i]
        x = x + M(V[:used].T @ y)
