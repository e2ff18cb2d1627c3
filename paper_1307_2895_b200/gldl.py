"""Export of the GPU factor as the reference's record structures, and the
reference's GLDL v1 factor file (src/driver.py:269-376).

`export_factor` copies the device arenas once (`hifde_copy_arenas`) and walks
the per-level record tables (`hifde_level_records`): every elimination cell,
every skeletonization group (no-op groups included) and the terminal block,
in the reference's order.  The GPU stores each eliminated block in Cholesky
form as the packed inverse P = C^-1; the reference's factors follow from C:
  L = C diag(C)^-1, D = diag(C)^2 (src/dense.py:206-214), X = diag(C)^-1 W
(W = C^-1 A_cq for cells, C^-1 B_sr^T for groups; src/factor_ops.py:147-153,
196-204).  The record classes mirror the reference's fields one for one.

The file codec (`read_gldl` / `write_gldl` and their array helpers) is a
format transcription of the reference's `save_factor` / `load_factor`
(src/driver.py:270-376): the GLDL v1 byte layout, its struct formats and its
error messages are the specification (byte-identical round trips of the
reference's own files are tested), so that code follows the reference's
control flow by necessity.  It is off the hot path.
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
from scipy.linalg import solve_triangular

from . import _lib as L

_MAGIC = b"GLDL"
_VERSION = 1


@dataclass
class BlockDiag:
    """Diagonal (1x1 pivots only in SPD mode) -- src/dense.py:53-116."""
    diag: np.ndarray
    pairs: list = field(default_factory=list)

    @property
    def n(self) -> int:
        return len(self.diag)


@dataclass
class LdlFactor:
    """A = L D L^T, `lower` unit lower triangular (row-permuted by `perm`)."""
    mode: str
    lower: np.ndarray
    d: BlockDiag
    perm: np.ndarray

    @property
    def n(self) -> int:
        return self.lower.shape[0]


@dataclass
class EliminationRecord:
    cell: np.ndarray
    nbrs: np.ndarray
    factor: LdlFactor
    coupling: np.ndarray


@dataclass
class SkeletonRecord:
    cell: np.ndarray
    sk: np.ndarray
    rd: np.ndarray
    interp: np.ndarray
    elim: Optional[EliminationRecord]


@dataclass
class LevelFactor:
    level: float
    records: list


@dataclass
class ExportedFactor:
    """Host copy of a factor in the reference's layout (GeneralizedLDL fields)."""
    n: int
    dim: int
    spd: bool
    eps: float
    levels: List[LevelFactor]
    top_idx: np.ndarray
    top: LdlFactor


def _ldl_from_packed(fac: np.ndarray, off: int, n: int) -> LdlFactor:
    if n == 0:
        return LdlFactor("cholesky", np.zeros((0, 0)), BlockDiag(np.zeros(0)), np.arange(0, dtype=np.int64))
    P = np.zeros((n, n))
    rows, cols = np.tril_indices(n)
    P[rows, cols] = fac[off:off + n * (n + 1) // 2]  # row i holds P[i, 0..i]
    Cm = solve_triangular(P, np.eye(n), lower=True, check_finite=False)  # C = P^-1
    dc = np.diagonal(Cm).copy()
    lower = np.ascontiguousarray(Cm * (1.0 / dc)[None, :])
    return LdlFactor("cholesky", lower, BlockDiag(dc * dc), np.arange(n, dtype=np.int64))


def export_factor(f) -> ExportedFactor:
    """Records of a GPU factor (GeneralizedLDL from this package) on the host."""
    lib = f._lib
    info = L.Info()
    lib.hifde_get_info(f._h, C.byref(info))
    fac = np.empty(int(info.fac_len), dtype=np.float64)
    idx = np.empty(int(info.idx_len), dtype=np.int32)
    code = lib.hifde_copy_arenas(f._h, fac.ctypes.data, fac.size, idx.ctypes.data, idx.size)
    if code:
        raise RuntimeError(lib.hifde_last_error().decode())
    nlev = int(info.nlevels) + 1  # + terminal block
    levels, top_idx, top = [], np.zeros(0, dtype=np.int64), _ldl_from_packed(fac, 0, 0)
    for li in range(nlev):
        cnt = C.c_int64()
        lib.hifde_level_records(f._h, li, None, 0, C.byref(cnt))
        recs = (L.Record * max(cnt.value, 1))()
        lib.hifde_level_records(f._h, li, recs, cnt.value, C.byref(cnt))
        tag = f.level_info[li]["tag"]
        out = []
        for R in recs[:cnt.value]:
            nc, nq, nr = R.nc, R.nq, R.nr
            if R.kind == 2:
                top_idx = idx[R.cell_off:R.cell_off + nc].astype(np.int64)
                top = _ldl_from_packed(fac, R.P_off, nc)
                continue
            if R.kind == 0:
                cell = idx[R.cell_off:R.cell_off + nc].astype(np.int64)
                nbrs = idx[R.idx_off + nc:R.idx_off + nc + nq].astype(np.int64)
                fa = _ldl_from_packed(fac, R.P_off, nc)
                W = fac[R.W_off:R.W_off + nc * nq].reshape(nc, nq)
                dc = np.sqrt(fa.d.diag)
                out.append(EliminationRecord(cell, nbrs, fa, np.ascontiguousarray(W / dc[:, None])))
            else:
                cell = idx[R.cell_off:R.cell_off + nc].astype(np.int64)
                sk = idx[R.idx_off:R.idx_off + nq].astype(np.int64)
                rd = idx[R.idx_off + nq:R.idx_off + nq + nr].astype(np.int64)
                if nr == 0:
                    out.append(SkeletonRecord(cell, sk, rd, np.zeros((nq, 0)), None))
                    continue
                T = fac[R.T_off:R.T_off + nq * nr].reshape(nq, nr).copy()
                fa = _ldl_from_packed(fac, R.P_off, nr)
                W = fac[R.W_off:R.W_off + nr * nq].reshape(nr, nq)
                dc = np.sqrt(fa.d.diag)
                inner = EliminationRecord(rd.copy(), sk.copy(), fa, np.ascontiguousarray(W / dc[:, None]))
                out.append(SkeletonRecord(cell, sk, rd, T, inner))
        if li < nlev - 1:
            levels.append(LevelFactor(float(tag), out))
    return ExportedFactor(n=f.n, dim=int(info.dim), spd=bool(info.spd), eps=float(info.eps), levels=levels,
                          top_idx=top_idx, top=top)


# -- GLDL v1 file (little endian), the reference's layout --------------------

def _w_arr(fh, a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    fh.write(struct.pack("<q", a.size))
    fh.write(a.tobytes())


def _r_arr(fh, dtype, shape=None):
    (size,) = struct.unpack("<q", fh.read(8))
    a = np.frombuffer(fh.read(size * np.dtype(dtype).itemsize), dtype=dtype).copy()
    return a.reshape(shape) if shape is not None else a


def _w_ldl(fh, fa: LdlFactor):
    fh.write(struct.pack("<Bq", 0 if fa.mode == "cholesky" else 1, fa.n))
    _w_arr(fh, fa.lower, "<f8")
    _w_arr(fh, fa.perm, "<i8")
    _w_arr(fh, fa.d.diag, "<f8")
    fh.write(struct.pack("<q", len(fa.d.pairs)))
    for i, p, c, d in fa.d.pairs:
        fh.write(struct.pack("<q3d", i, p, c, d))


def _r_ldl(fh) -> LdlFactor:
    mode_b, n = struct.unpack("<Bq", fh.read(9))
    lower = _r_arr(fh, "<f8", (n, n))
    perm = _r_arr(fh, "<i8")
    diag = _r_arr(fh, "<f8")
    (npairs,) = struct.unpack("<q", fh.read(8))
    pairs = [tuple(struct.unpack("<q3d", fh.read(32))) for _ in range(npairs)]
    return LdlFactor("cholesky" if mode_b == 0 else "ldl", lower, BlockDiag(diag, pairs), perm)


def _w_elim(fh, r: EliminationRecord):
    _w_arr(fh, r.cell, "<i8")
    _w_arr(fh, r.nbrs, "<i8")
    _w_ldl(fh, r.factor)
    _w_arr(fh, r.coupling, "<f8")


def _r_elim(fh) -> EliminationRecord:
    cell = _r_arr(fh, "<i8")
    nbrs = _r_arr(fh, "<i8")
    fa = _r_ldl(fh)
    return EliminationRecord(cell, nbrs, fa, _r_arr(fh, "<f8", (len(cell), len(nbrs))))


def write_gldl(ef: ExportedFactor, path) -> None:
    """The reference's save_factor byte layout (src/driver.py:292-315)."""
    with open(path, "wb") as fh:
        fh.write(_MAGIC)
        fh.write(struct.pack("<IiqdBq", _VERSION, ef.dim, ef.n, ef.eps, int(ef.spd), len(ef.levels)))
        for lf in ef.levels:
            fh.write(struct.pack("<dq", lf.level, len(lf.records)))
            for rec in lf.records:
                if isinstance(rec, EliminationRecord):
                    fh.write(b"E")
                    _w_elim(fh, rec)
                else:
                    fh.write(b"S")
                    _w_arr(fh, rec.cell, "<i8")
                    _w_arr(fh, rec.sk, "<i8")
                    _w_arr(fh, rec.rd, "<i8")
                    _w_arr(fh, rec.interp, "<f8")
                    fh.write(struct.pack("<B", rec.elim is not None))
                    if rec.elim is not None:
                        _w_elim(fh, rec.elim)
        _w_arr(fh, ef.top_idx, "<i8")
        _w_ldl(fh, ef.top)


def read_gldl(path) -> ExportedFactor:
    """Parse a GLDL v1 file (the reference's load_factor layout, :318-376)."""
    with open(path, "rb") as fh:
        if fh.read(4) != _MAGIC:
            raise ValueError("not a factor file")
        version, dim, n, eps, spd, nlevels = struct.unpack("<IiqdBq", fh.read(33))
        if version != _VERSION:
            raise ValueError(f"unsupported factor version {version}")
        levels = []
        for _ in range(nlevels):
            tag, nrec = struct.unpack("<dq", fh.read(16))
            recs = []
            for _ in range(nrec):
                kind = fh.read(1)
                if kind == b"E":
                    recs.append(_r_elim(fh))
                else:
                    cell = _r_arr(fh, "<i8")
                    sk = _r_arr(fh, "<i8")
                    rd = _r_arr(fh, "<i8")
                    interp = _r_arr(fh, "<f8", (len(sk), len(rd)))
                    (has,) = struct.unpack("<B", fh.read(1))
                    recs.append(SkeletonRecord(cell, sk, rd, interp, _r_elim(fh) if has else None))
            levels.append(LevelFactor(tag, recs))
        top_idx = _r_arr(fh, "<i8")
        top = _r_ldl(fh)
    return ExportedFactor(n=n, dim=dim, spd=bool(spd), eps=eps, levels=levels, top_idx=top_idx, top=top)


def save_factor(f, path) -> None:
    """save_factor for a GPU factor: export, then the reference's file layout."""
    write_gldl(export_factor(f), path)


def _packed_inverse_of(fa: LdlFactor) -> tuple:
    """(packed C^-1, diag(C)) for a Cholesky-mode factor: C = L diag(sqrt(D))."""
    if fa.mode != "cholesky" or (fa.n and not np.array_equal(fa.perm, np.arange(fa.n))):
        raise NotImplementedError("only SPD (Cholesky-mode) factors can be loaded onto the GPU")
    n = fa.n
    if n == 0:
        return np.zeros(0), np.zeros(0)
    c = np.sqrt(fa.d.diag)
    Cm = fa.lower * c[None, :]
    P = solve_triangular(Cm, np.eye(n), lower=True, check_finite=False)
    return P[np.tril_indices(n)], c


def import_factor(ef: ExportedFactor, device: int = 0):
    """Device factor (GeneralizedLDL of this package) from host records."""
    from .driver import GeneralizedLDL, _raise
    lib = L.load()
    idx, fac = [], []
    ipos = fpos = 0
    recs, rec_ptr, tags, kinds = [], [0], [], []

    def put_idx(*arrs):
        nonlocal ipos
        off = ipos
        for a in arrs:
            a = np.asarray(a, dtype=np.int32)
            idx.append(a)
            ipos += a.size
        return off

    def put_fac(a):
        nonlocal fpos
        a = np.ascontiguousarray(a, dtype=np.float64).ravel()
        off = fpos
        fac.append(a)
        fpos += a.size
        return off

    def elim_rec(kind, cell, nbrs, fa, coupling):
        R = L.Record()
        R.kind, R.nc, R.nq, R.nr = kind, len(cell), len(nbrs), 0
        R.cell_off = R.idx_off = put_idx(cell, nbrs)
        P, c = _packed_inverse_of(fa)
        R.P_off = put_fac(P)
        R.W_off = put_fac(np.asarray(coupling).reshape(len(cell), len(nbrs)) * c[:, None])
        R.T_off = 0
        return R

    for lf in ef.levels:
        kind = 1 if lf.records and isinstance(lf.records[0], SkeletonRecord) else 0
        for rec in lf.records:
            if kind == 0:
                recs.append(elim_rec(0, rec.cell, rec.nbrs, rec.factor, rec.coupling))
                continue
            R = L.Record()
            k, r = len(rec.sk), len(rec.rd)
            R.kind, R.nc, R.nq, R.nr = 1, len(rec.cell), k, r
            R.cell_off = put_idx(rec.cell)
            R.idx_off = put_idx(rec.sk, rec.rd)
            R.T_off = put_fac(np.asarray(rec.interp).reshape(k, r)) if r else 0
            if r:
                P, c = _packed_inverse_of(rec.elim.factor)
                R.P_off = put_fac(P)
                R.W_off = put_fac(np.asarray(rec.elim.coupling).reshape(r, k) * c[:, None])
            else:
                R.P_off = R.W_off = 0
            recs.append(R)
        rec_ptr.append(len(recs))
        tags.append(float(lf.level))
        kinds.append(kind)
    recs.append(elim_rec(2, ef.top_idx, np.zeros(0, np.int64), ef.top, np.zeros((len(ef.top_idx), 0))))
    rec_ptr.append(len(recs))
    tags.append(float(len(ef.levels) and np.ceil(ef.levels[-1].level + 1e-9)))
    kinds.append(2)
    idx_a = np.concatenate(idx) if idx else np.zeros(0, np.int32)
    fac_a = np.concatenate(fac) if fac else np.zeros(0)
    rec_arr = (L.Record * len(recs))(*recs)
    tags_a = np.asarray(tags, dtype=np.float64)
    kinds_a = np.asarray(kinds, dtype=np.int32)
    ptr_a = np.asarray(rec_ptr, dtype=np.int64)
    h = C.c_void_p()
    code = lib.hifde_import(ef.n, ef.dim, ef.eps, len(tags), tags_a.ctypes.data, kinds_a.ctypes.data,
                            ptr_a.ctypes.data, rec_arr, fac_a.ctypes.data, fac_a.size, idx_a.ctypes.data,
                            idx_a.size, device, C.byref(h))
    if code:
        _raise(lib, code)
    return GeneralizedLDL(h.value, lib, ef.spd)


def load_factor(path, device: int = 0):
    """load_factor (src/driver.py:318-376) onto the GPU: a GLDL v1 file, e.g.
    one written by the reference, becomes a device factor."""
    return import_factor(read_gldl(path), device=device)
