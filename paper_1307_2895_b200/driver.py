"""Reference-facing API of the B200 HIF-DE path.

Same names, signatures, options and error classes as the reference's hot-path
entry points (``src/driver.py:201-259``), backed by the sm_100a library
through its C ABI (``include/hifde_gpu.h``):

* ``factor_hifde(a, grid, eps, spd=True, skip_levels=0, verify=False)``
* ``factor_hifde3x(a, grid, eps, spd=True, skip_levels=1, verify=False)``
* ``factor_mf(a, grid, spd=True, verify=False)``
* ``GeneralizedLDL.apply_inverse(b)`` / ``apply_inverse(f, b)``

``a`` is anything the reference accepts that can produce a symmetric CSR
(the reference's ``SparseSymMatrix`` via ``to_scipy()``, a SciPy sparse matrix,
or a dense array); unlike the reference it is not consumed.  ``grid`` is any
object with ``dim, n, m, nlevels`` (the reference's ``GridConfig`` works).
There is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np
import scipy.sparse as sp

from . import _lib as L


class FactorizationError(Exception):
    """Base class for factorization failures (src/dense.py:41-42)."""


class IndefiniteBlockError(FactorizationError):
    """Cholesky requested on a block that is not positive definite."""


class SingularBlockError(FactorizationError):
    """A pivot fell below the singularity threshold."""


def _raise(lib, code: int):
    msg = lib.hifde_last_error().decode(errors="replace")
    if code == L.HIFDE_INDEFINITE:
        raise IndefiniteBlockError(msg)
    if code == L.HIFDE_SINGULAR:
        raise SingularBlockError(msg)
    if code == L.HIFDE_BADARG:
        raise ValueError(msg)
    if code == L.HIFDE_INTERNAL:
        raise AssertionError(msg)
    raise RuntimeError(msg)


def _as_csr(a) -> sp.csr_matrix:
    if hasattr(a, "to_scipy"):
        a = a.to_scipy()
    if sp.issparse(a) and a.format == "csr" and a.dtype == np.float64 and a.has_canonical_format:
        m = a  # read only: the factor never modifies A, so no copy
    else:
        m = sp.csr_matrix(a, dtype=np.float64)
        m.sum_duplicates()
        m.sort_indices()
    if m.shape[0] != m.shape[1]:
        raise ValueError("matrix must be square")
    return m


class GeneralizedLDL:
    """GPU-resident generalized LDL factor (src/driver.py:64-149).

    ``apply_inverse`` runs the up/down sweep on the device; ``metrics`` holds
    the reference's keys (``s_top``, ``active_trace``, ``level_seconds``,
    ``m_f_bytes``, ``t_f_seconds``) plus ``skeleton_counts`` and per-level
    algorithmic FLOP/byte counts.
    """

    def __init__(self, handle: int, lib, spd: bool, pending=None):
        self._h = C.c_void_p(handle)
        self._lib = lib
        self.spd = spd
        self._info = None
        # wait=False factorization still running on the library's thread:
        # (n, dim, eps, input arrays kept alive); everything else is read
        # from the finished factor on first use (wait())
        self._pending = pending
        if pending is None:
            self._load()
        else:
            self.n, self.dim, self.eps = int(pending[0]), int(pending[1]), float(pending[2])

    def wait(self) -> "GeneralizedLDL":
        """Blocks until a ``wait=False`` factorization is complete and raises
        what it raised (the reference's exceptions)."""
        if self._info is None:
            self._load()
        return self

    def _load(self):
        lib = self._lib
        code = lib.hifde_wait(self._h)
        self._pending = None
        if code:
            _raise(lib, code)
        info = L.Info()
        lib.hifde_get_info(self._h, C.byref(info))
        self.n = int(info.n)
        self.dim = int(info.dim)
        self.eps = float(info.eps)
        self._device_bytes = int(info.device_bytes)
        self._level_info = []
        for i in range(info.nlevels + 1):
            li = L.LevelInfo()
            lib.hifde_get_level(self._h, i, C.byref(li))
            self._level_info.append({k: getattr(li, k) for k, _ in L.LevelInfo._fields_})
        levels = self._level_info[:-1]
        trace = [(-1.0, self.n)] + [(d["tag"], int(d["active_after"])) for d in levels]
        self._metrics = {
            "s_top": int(info.s_top),
            "active_trace": trace,
            "level_seconds": [(d["tag"], d["seconds"]) for d in levels],
            "m_f_bytes": int(info.m_f_bytes),
            "t_f_seconds": float(info.t_f_seconds),
            "skeleton_counts": [(d["tag"], int(d["nskel"])) for d in levels if d["kind"] == 1],
            "factor_gflop": sum(d["gflop"] for d in self._level_info),
            "factor_gbytes": sum(d["gbytes"] for d in self._level_info),
            "launches": int(lib.hifde_last_launch_count()),
            "nranks": int(info.nranks),
            "xfer_bytes": int(info.xfer_bytes),
        }
        self._info = info

    @property
    def metrics(self) -> dict:
        return self.wait()._metrics

    @property
    def level_info(self) -> list:
        return self.wait()._level_info

    @property
    def device_bytes(self) -> int:
        return self.wait()._device_bytes

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def storage_bytes(self) -> int:
        return self.metrics["m_f_bytes"]

    def shard_info(self) -> dict:
        """Live state of a sharded factor: whether this rank's
        arena holds every record yet (real ranks hold their own until apply /
        export / power sum them) and the vector bytes its partitioned solves
        exchanged with the other ranks."""
        info = L.Info()
        self._lib.hifde_get_info(self._h, C.byref(info))
        return {"nranks": int(info.nranks), "factor_whole": bool(info.factor_whole),
                "solve_xfer_bytes": int(info.solve_xfer_bytes)}

    def _out(self, like: np.ndarray) -> np.ndarray:
        """Output array for a host solve/apply: large results live in a
        page-locked block of the library's caching pool (DMA'd straight into,
        recycled when the array is garbage-collected); small ones are plain."""
        if like.nbytes < _PINNED_MIN:
            return np.empty_like(like)
        blk = _PinnedBlock.get(self._lib, like.nbytes)
        if blk is None:
            return np.empty_like(like)
        blk.__array_interface__ = {"shape": like.shape, "typestr": "<f8", "data": (blk.ptr, False), "version": 3}
        return np.asarray(blk)

    def apply_inverse(self, b) -> np.ndarray:
        """x ~= A^{-1} b for b of shape (N,) or (N, nrhs); host arrays."""
        arr = np.ascontiguousarray(np.asarray(b, dtype=np.float64))
        vec = arr.ndim == 1
        if arr.shape[0] != self.n:
            raise ValueError("right-hand side has the wrong length")
        nrhs = 1 if vec else arr.shape[1]
        out = self._out(arr)
        if arr.size:
            code = self._lib.hifde_solve(self._h, arr.ctypes.data, out.ctypes.data, self.n, nrhs, 0, None)
            self._pending = None  # (the solve has waited for a wait=False factorization)
            if code:
                _raise(self._lib, code)
        return out

    def apply(self, x) -> np.ndarray:
        """y ~= A x through the factored operator (src/driver.py:95-111); host arrays."""
        arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
        if arr.shape[0] != self.n:
            raise ValueError("vector has the wrong length")
        nrhs = 1 if arr.ndim == 1 else arr.shape[1]
        out = self._out(arr)
        if arr.size:
            code = self._lib.hifde_apply(self._h, arr.ctypes.data, out.ctypes.data, self.n, nrhs, 0, None)
            if code:
                _raise(self._lib, code)
        return out

    def apply_device(self, x_ptr: int, y_ptr: int, nrhs: int, stream: Optional[int] = None):
        """Device-pointer variant of apply (row-major N x nrhs float64 buffers)."""
        code = self._lib.hifde_apply(self._h, C.c_void_p(x_ptr), C.c_void_p(y_ptr), self.n, nrhs, 1,
                                     C.c_void_p(stream) if stream else None)
        if code:
            _raise(self._lib, code)

    def apply_inverse_device(self, b_ptr: int, x_ptr: int, nrhs: int, stream: Optional[int] = None):
        """Device-pointer variant (row-major N x nrhs float64 buffers)."""
        code = self._lib.hifde_solve(self._h, C.c_void_p(b_ptr), C.c_void_p(x_ptr), self.n, nrhs, 1,
                                     C.c_void_p(stream) if stream else None)
        if code:
            _raise(self._lib, code)

    def kernel_stats(self, phase: int = 0) -> list:
        """Per (kernel, level): launches, CUDA-event seconds, algorithmic GB
        and GFLOP (factors created with ``kernel_log=True``; phase 0 the
        factorization, 1 the last solve)."""
        n = C.c_int64()
        code = self._lib.hifde_kernel_stats(self._h, phase, None, 0, C.byref(n))
        if code:
            _raise(self._lib, code)
        arr = (L.KernelStat * max(n.value, 1))()
        code = self._lib.hifde_kernel_stats(self._h, phase, arr, n.value, C.byref(n))
        if code:
            _raise(self._lib, code)
        return [{"name": a.name.decode(), "tag": a.tag, "phase": a.phase, "launches": a.launches,
                 "seconds": a.seconds, "gbytes": a.gbytes, "gflop": a.gflop} for a in arr[:n.value]]

    def close(self):
        if self._h is not None and self._h.value:
            self._lib.hifde_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_PINNED_MIN = 8 << 20


class _PinnedBlock:
    """Owner of one hifde_host_alloc block; the numpy array built on it keeps
    it alive (array base) and the block returns to the pool with it."""

    __slots__ = ("ptr", "lib", "__array_interface__", "__weakref__")

    @classmethod
    def get(cls, lib, nbytes: int):
        p = C.c_void_p()
        if lib.hifde_host_alloc(nbytes, C.byref(p)) or not p.value:
            return None
        blk = cls()
        blk.ptr, blk.lib = p.value, lib
        return blk

    def __del__(self):
        try:
            self.lib.hifde_host_free(C.c_void_p(self.ptr))
        except Exception:
            pass


def _pinned_array(lib, shape, dtype) -> np.ndarray:
    dtype = np.dtype(dtype)
    nbytes = int(np.prod(shape)) * dtype.itemsize
    blk = _PinnedBlock.get(lib, max(nbytes, 1))
    if blk is None:
        raise MemoryError("page-locked host allocation failed")
    blk.__array_interface__ = {"shape": tuple(shape), "typestr": dtype.str, "data": (blk.ptr, False),
                               "version": 3}
    return np.asarray(blk)


def pinned_empty(shape, dtype=np.float64) -> np.ndarray:
    """Uninitialized host array in a page-locked block of the library's
    caching pool (returned to the pool when the array is collected).
    Right-hand sides and matrices built in such arrays move by direct DMA,
    with no staging copy on the host."""
    return _pinned_array(L.load(), shape if isinstance(shape, tuple) else (int(shape),), dtype)


def pinned_csr(a) -> sp.csr_matrix:
    """A copy of the CSR matrix ``a`` whose offsets, column indices and values
    live in page-locked host memory (``pinned_empty``): ``factor_hifde`` of it
    uploads the three arrays by direct DMA while the level-0 analysis runs,
    instead of staging them through the library's pinned buffers.  Offsets
    keep scipy's int32 when they fit."""
    csr = _as_csr(a)
    lib = L.load()
    ipt = np.int32 if csr.indptr.dtype == np.int32 else np.int64
    ip = _pinned_array(lib, csr.indptr.shape, ipt)
    ix = _pinned_array(lib, csr.indices.shape, np.int32)
    va = _pinned_array(lib, csr.data.shape, np.float64)
    ip[...] = csr.indptr
    ix[...] = csr.indices
    va[...] = csr.data
    m = sp.csr_matrix((va, ix, ip), shape=csr.shape, copy=False)
    if any(x.ctypes.data != y.ctypes.data for x, y in ((m.data, va), (m.indices, ix), (m.indptr, ip))):
        raise RuntimeError("scipy copied the page-locked CSR arrays")
    m.has_sorted_indices = True
    m.has_canonical_format = True
    return m


def _factor(a, grid, eps: float, variant: int, spd: bool, skip_levels: int, verify: bool,
            order: str = "auto", exact_max_batches: int = 64, device: Optional[int] = None,
            stream: Optional[int] = None, comm=None, kernel_log: bool = False,
            symbolic: str = "auto", wait: bool = True) -> GeneralizedLDL:
    lib = L.load()
    if not spd:
        raise NotImplementedError("indefinite (Bunch-Kaufman) mode is outside the GPU hot path")
    csr = _as_csr(a)
    # scipy's int32 offsets go to the library as they are (it widens them on
    # its host threads); int64 ones as well
    ip32 = csr.indptr.dtype == np.int32
    indptr = np.ascontiguousarray(csr.indptr, dtype=np.int32 if ip32 else np.int64)
    indices = np.ascontiguousarray(csr.indices, dtype=np.int32)
    data = np.ascontiguousarray(csr.data, dtype=np.float64)
    opt = L.Options()
    lib.hifde_default_options(C.byref(opt), variant)
    opt.skip_levels = int(skip_levels)
    opt.spd = 1
    opt.eps = float(eps)
    opt.order_mode = L.ORDER[order]
    opt.exact_max_batches = int(exact_max_batches)
    if device is None:
        device = comm.device if comm is not None else 0
    opt.device = int(device)
    opt.verify = int(bool(verify))
    opt.stream = stream
    opt.comm = comm.handle if comm is not None else None  # distributed.Comm: sharded sweep
    opt.kernel_log = int(bool(kernel_log))
    opt.symbolic = L.SYMBOLIC[symbolic]  # "host": the host level analysis throughout (A/B tests)
    opt.indptr_int32 = int(ip32)
    # wait=False: the call returns while the factorization runs on a library
    # thread (one GPU); the first use of the factor waits for it and raises
    # what it raised.  apply_inverse of a page-locked host block uploads the
    # right-hand sides meanwhile.
    pending = not wait and comm is None
    opt.async_factor = int(pending)
    h = C.c_void_p()
    code = lib.hifde_factor(indptr.ctypes.data, indices.ctypes.data, data.ctypes.data, csr.shape[0],
                            int(grid.dim), int(grid.n), int(grid.m), int(grid.nlevels),
                            C.byref(opt), C.byref(h))
    if code:
        _raise(lib, code)
    if pending:  # the input arrays must outlive the factorization
        return GeneralizedLDL(h.value, lib, spd, pending=(csr.shape[0], grid.dim, eps, indptr, indices, data, csr))
    return GeneralizedLDL(h.value, lib, spd)


def factor_hifde(a, grid, eps: float, spd: bool = True, skip_levels: int = 0,
                 verify: bool = False, **kw) -> GeneralizedLDL:
    """Interior elimination plus edge (2D) / face (3D) skeletonization
    (src/driver.py:212-225)."""
    return _factor(a, grid, eps, L.VARIANT_HIFDE, spd, skip_levels, verify, **kw)


def factor_hifde3x(a, grid, eps: float, spd: bool = True, skip_levels: int = 1,
                   verify: bool = False, **kw) -> GeneralizedLDL:
    """3D faces + edges with adaptive minimal separators (src/driver.py:228-251)."""
    if grid.dim != 3:
        raise ValueError("factor_hifde3x requires a 3D grid")
    return _factor(a, grid, eps, L.VARIANT_HIFDE3X, spd, skip_levels, verify, **kw)


def factor_mf(a, grid, spd: bool = True, verify: bool = False, **kw) -> GeneralizedLDL:
    """Multifrontal elimination, exact to rounding (src/driver.py:201-209)."""
    return _factor(a, grid, 0.0, L.VARIANT_MF, spd, grid.nlevels, verify, **kw)


def apply_inverse(f: GeneralizedLDL, b) -> np.ndarray:
    return f.apply_inverse(b)


def densify(f: GeneralizedLDL) -> np.ndarray:
    """Dense N x N matrix of the factored operator, F I (src/driver.py:262-264);
    testing oracle for small N."""
    return f.apply(np.eye(f.n))


def device_count() -> int:
    return int(L.load().hifde_device_count())
