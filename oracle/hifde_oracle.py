"""CPU oracle for the HIF-DE factor/solve hot path -- TEST INFRASTRUCTURE ONLY.

This module is the parity checker for the B200 path.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it; the product package
(``paper_1307_2895_b200``) never does, and it has no CPU fallback.

It restates, in numpy/scipy, the algorithm of the reference package
``hifde`` 0.1.0 (``/root/reference/pkg/src/hifde``; citations below are
``file:line`` into that tree, ``src/`` = ``pkg/src/hifde/``):

* grid / coefficient fields / five- and seven-point assembly
  (``src/discretize.py:77-192``), plus BASELINE.json's Gaussian
  high-contrast field;
* level partitioning: interior cells, interface Voronoi groups, adaptive
  minimal separators (``src/partition.py:68-227``);
* the level sweep ``factor_hifde`` / ``factor_hifde3x`` / ``factor_mf``
  (``src/driver.py:175-251``) with per-cell elimination and
  skeletonization (``src/factor_ops.py:138-214``), LDL via Cholesky and the
  column-pivoted-QR interpolative decomposition (``src/dense.py:187-264``);
* ``apply_inverse`` / ``apply`` sweeps (``src/driver.py:95-129``,
  ``src/factor_ops.py:47-128``) and PCG (``src/krylov.py:48-77``).

The working matrix is *not* stored the reference's way (mirrored sorted row
lists, ``src/sparse.py``).  It is held as the original stencil matrix plus a
set of live dense "clique blocks": every elimination consumes all blocks
touching its cell and emits one block over its neighbour set (the Schur
update), every skeletonization with redundant DOFs emits one delta block over
its skeletons.  The sparsity pattern this induces is exactly the reference's
(fill is stored even when zero, ``src/sparse.py:10-11``), so neighbour sets,
partitions and the sequential processing order are the reference's; only the
summation order of shared entries differs.  The same data model is what the
CUDA path implements.

Parity of this restatement is pinned against golden vectors produced by the
reference itself (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import os
import time
from contextlib import nullcontext
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

SINGULAR_PIVOT_RTOL = 1e-14          # src/dense.py:38
HIGH_CONTRAST = (1e-2, 1e2)          # src/discretize.py:38
SMOOTH_SIGMA = 4.0                   # src/discretize.py:39
SMOOTH_TRUNCATE = 4.0                # src/discretize.py:40


class OracleFactorizationError(Exception):
    pass


class OracleIndefiniteError(OracleFactorizationError):
    pass


class OracleSingularError(OracleFactorizationError):
    pass


# ---------------------------------------------------------------------------
# grid and problem generation (src/discretize.py)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Grid:
    """n^dim grid, leaf width m, n = 2^nlevels m (src/discretize.py:43-89)."""
    dim: int
    n: int
    m: int
    nlevels: int

    @property
    def side(self) -> int:
        return self.n - 1

    @property
    def ndof(self) -> int:
        return self.side ** self.dim

    @property
    def h(self) -> float:
        return 1.0 / self.n

    def coords(self) -> np.ndarray:
        """1-based integer grid coordinates, first axis fastest."""
        idx = np.arange(self.ndof, dtype=np.int64)
        out = np.empty((self.ndof, self.dim), dtype=np.int64)
        for ax in range(self.dim):
            out[:, ax] = idx % self.side + 1
            idx //= self.side
        return out


def make_grid(dim: int, n: int, m: int) -> Grid:
    """Validated grid (src/discretize.py:77-89)."""
    if dim not in (2, 3):
        raise ValueError("dim must be 2 or 3")
    if m < 2 or n % m:
        raise ValueError("n must be a multiple of m >= 2")
    r = n // m
    L = r.bit_length() - 1
    if (1 << L) != r or L < 1:
        raise ValueError("n/m must be a power of two >= 2")
    return Grid(dim, n, m, L)


def _stag_shape(g: Grid, axis: int):
    return tuple(g.n if i == axis else g.n - 1 for i in range(g.dim))


def constant_coeffs(g: Grid, a0: float = 1.0, b0: float = 0.0):
    """src/discretize.py:111-114."""
    a = tuple(np.full(_stag_shape(g, i), float(a0)) for i in range(g.dim))
    return a, np.full((g.side,) * g.dim, float(b0))


def _smoothed(g: Grid, draw):
    from scipy.ndimage import gaussian_filter
    return [gaussian_filter(draw(_stag_shape(g, i)), sigma=SMOOTH_SIGMA,
                            mode="reflect", truncate=SMOOTH_TRUNCATE)
            for i in range(g.dim)]


def gaussian_contrast_coeffs(g: Grid, seed: int):
    """BASELINE.json high-contrast field: N(0,1) staggered noise smoothed by
    a Gaussian of width 4h, thresholded at zero to {1e-2, 1e2}
    (SURVEY.md section 8(d))."""
    rng = np.random.default_rng(seed)
    sm = _smoothed(g, rng.standard_normal)
    lo, hi = HIGH_CONTRAST
    return tuple(np.where(s <= 0.0, lo, hi) for s in sm), np.zeros((g.side,) * g.dim)


def median_contrast_coeffs(g: Grid, seed: int):
    """The reference's own high_contrast_field (uniform noise, median split,
    src/discretize.py:117-140); used only for golden-vector pinning."""
    rng = np.random.default_rng(seed)
    sm = _smoothed(g, rng.random)
    mu = np.median(np.concatenate([s.ravel() for s in sm]))
    lo, hi = HIGH_CONTRAST
    return tuple(np.where(s <= mu, lo, hi) for s in sm), np.zeros((g.side,) * g.dim)


def assemble_csr(g: Grid, a_arrays, b) -> sp.csr_matrix:
    """Stencil matrix of -div(a grad u) + b u (src/discretize.py:153-192).

    Same floating-point operation sequence as the reference, so the matrix is
    bit-identical: diagonal = b + sum_axis (a_lo + a_hi) n^2, off-diagonal =
    -(a_mid n^2); Dirichlet couplings dropped.
    """
    side, dim = g.side, g.dim
    s2 = float(g.n) * float(g.n)
    diag = np.array(b, dtype=float, copy=True)
    for ax in range(dim):
        a = a_arrays[ax]
        lo = [slice(None)] * dim
        hi = [slice(None)] * dim
        lo[ax] = slice(0, side)
        hi[ax] = slice(1, g.n)
        diag += (a[tuple(lo)] + a[tuple(hi)]) * s2
    ids = np.arange(g.ndof, dtype=np.int64).reshape((side,) * dim, order="F")
    r_list = [np.arange(g.ndof, dtype=np.int64)]
    c_list = [np.arange(g.ndof, dtype=np.int64)]
    v_list = [diag.ravel(order="F")]
    for ax in range(dim):
        a = a_arrays[ax]
        first = [slice(None)] * dim
        inner = [slice(None)] * dim
        first[ax] = slice(0, side - 1)
        inner[ax] = slice(1, side)
        src = ids[tuple(first)].ravel(order="F")
        val = -(a[tuple(inner)] * s2).ravel(order="F")
        dst = src + side ** ax
        r_list += [src, dst]
        c_list += [dst, src]
        v_list += [val, val]
    m = sp.coo_matrix((np.concatenate(v_list),
                       (np.concatenate(r_list), np.concatenate(c_list))),
                      shape=(g.ndof, g.ndof)).tocsr()
    m.sum_duplicates()
    m.sort_indices()
    return m


def make_problem(dim: int, n_interior: int, m: int, field: str = "const",
                 seed: int = 0):
    """BASELINE-style problem: n_interior = n - 1 interior points per axis."""
    g = make_grid(dim, n_interior + 1, m)
    if field == "const":
        a, b = constant_coeffs(g)
    elif field == "gauss_contrast":
        a, b = gaussian_contrast_coeffs(g, seed)
    elif field == "median_contrast":
        a, b = median_contrast_coeffs(g, seed)
    else:
        raise ValueError(field)
    return g, assemble_csr(g, a, b)


# ---------------------------------------------------------------------------
# partitioning (src/partition.py)
# ---------------------------------------------------------------------------

def _split_by_key(dofs: np.ndarray, keys: np.ndarray):
    """Groups of dofs sharing a key; groups in ascending key, members in
    ascending dof order (dofs arrive ascending)."""
    if dofs.size == 0:
        return [], np.empty(0, np.int64)
    order = np.argsort(keys, kind="stable")
    ks = keys[order]
    cut = np.flatnonzero(ks[1:] != ks[:-1]) + 1
    groups = np.split(dofs[order], cut)
    return groups, ks[np.r_[0, cut]]


def interior_groups(g: Grid, ell: int, active: np.ndarray, coords=None):
    """Active DOFs strictly inside each level-ell cell (src/partition.py:68-92)."""
    w = (1 << ell) * g.m
    k = g.n // w
    act = np.flatnonzero(active)
    x = (g.coords() if coords is None else coords)[act]
    inside = np.all(x % w != 0, axis=1)
    key = np.zeros(int(inside.sum()), dtype=np.int64)
    stride = 1
    for ax in range(g.dim):
        key += (x[inside, ax] // w) * stride
        stride *= k
    return _split_by_key(act[inside], key)[0]


def _round_multiple(x2, w, top):
    """Index j in [1, top] of the nearest centre w*j (ties to the lower)."""
    return np.clip((x2 + w - 1) // (2 * w), 1, top)


def _round_half(x2, w, top):
    """Index j in [1, top] of the nearest centre w*(j-1/2) (ties lower)."""
    return np.clip((x2 + 2 * w - 1) // (2 * w), 1, top)


def interface_groups(g: Grid, ell: int, active: np.ndarray, kind: str,
                     coords=None):
    """Voronoi groups about edge (2D) / face or edge (3D) centres, with the
    multi-plane exclusions of src/partition.py:108-181 (doubled integer
    coordinates, lowest family wins distance ties)."""
    dim = g.dim
    if (dim, kind) not in ((2, "edge"), (3, "face"), (3, "edge")):
        raise ValueError(kind)
    w = (1 << ell) * g.m
    k = g.n // w
    act = np.flatnonzero(active)
    x = (g.coords() if coords is None else coords)[act]
    planes = np.sum(x % w == 0, axis=1)
    if dim == 2:
        drop = planes == 2
    elif kind == "face":
        drop = planes >= 2
    else:
        drop = planes == 3
    dofs = act[~drop]
    x2 = 2 * x[~drop]
    nd = dofs.size
    best_d = np.full(nd, np.iinfo(np.int64).max, dtype=np.int64)
    best_key = np.zeros(nd, dtype=np.int64)
    fam_span = (k ** dim) * 2 * dim
    for fam in range(dim):
        d2 = np.zeros(nd, dtype=np.int64)
        key = np.zeros(nd, dtype=np.int64)
        stride = 1
        for ax in range(dim):
            # faces: the family axis is the normal (centre on a plane);
            # edges: the family axis runs along the edge (half offset)
            on_plane = (ax == fam) if kind == "face" else (ax != fam)
            if on_plane:
                j = _round_multiple(x2[:, ax], w, k - 1)
                c2 = 2 * w * j
                span = k - 1
            else:
                j = _round_half(x2[:, ax], w, k)
                c2 = w * (2 * j - 1)
                span = k
            d2 += (x2[:, ax] - c2) ** 2
            key += (j - 1) * stride
            stride *= span
        better = d2 < best_d
        best_d = np.where(better, d2, best_d)
        best_key = np.where(better, fam * fam_span + key, best_key)
    return _split_by_key(dofs, best_key)[0]


def adaptive_groups(g: Grid, ell: int, store: "CliqueStore", coords=None):
    """Minimal-separator interior cells (src/partition.py:184-227): Voronoi to
    cell centres, then every cell in ascending centre order sheds members
    still coupled to a DOF currently owned by another cell."""
    w = (1 << ell) * g.m
    k = g.n // w
    act = np.flatnonzero(store.active)
    x2 = 2 * (g.coords() if coords is None else coords)[act]
    key = np.zeros(act.size, dtype=np.int64)
    stride = 1
    for ax in range(g.dim):
        key += (_round_half(x2[:, ax], w, k) - 1) * stride
        stride *= k
    owner = np.full(store.n, -1, dtype=np.int64)
    owner[act] = key
    groups, keys = _split_by_key(act, key)
    out = []
    for members, gk in zip(groups, keys):
        shed = np.zeros(members.size, dtype=bool)
        # stencil couplings
        nb, row, _ = store.stencil_rows(members)
        o = owner[nb]
        foreign = (o != -1) & (o != gk)
        shed[np.unique(row[foreign])] = True
        # clique-block couplings: a block with a foreign owner sheds every
        # member it contains
        pos = {int(d): i for i, d in enumerate(members)}
        for bid in store.blocks_touching(members):
            bd = store.blk_dofs[bid]
            bd = bd[store.active[bd]]
            ob = owner[bd]
            if np.any((ob != -1) & (ob != gk)):
                for d in bd[ob == gk]:
                    i = pos.get(int(d))
                    if i is not None:
                        shed[i] = True
        if shed.any():
            owner[members[shed]] = -1
        keep = members[~shed]
        if keep.size:
            out.append(keep)
    return out


# ---------------------------------------------------------------------------
# dense kernels (src/dense.py)
# ---------------------------------------------------------------------------

def ldl_spd(block: np.ndarray):
    """SPD LDL^T as unit-lower L and D = diag(chol)^2 (src/dense.py:187-219).
    Returns (L, D, C) with C the Cholesky factor."""
    n = block.shape[0]
    if n == 0:
        return np.zeros((0, 0)), np.zeros(0), np.zeros((0, 0))
    scale = float(np.max(np.abs(np.diag(block))))
    if scale == 0.0:
        scale = float(np.max(np.abs(block)))
    try:
        c = sla.cholesky(block, lower=True, check_finite=False)
    except sla.LinAlgError as exc:
        raise OracleIndefiniteError(str(exc)) from exc
    dc = np.diagonal(c).copy()
    d = dc * dc
    if np.min(np.abs(d)) <= SINGULAR_PIVOT_RTOL * max(scale, 1e-300):
        raise OracleSingularError("singular pivot")
    return c / dc[None, :], d, c


def column_id(mq: np.ndarray, eps: float):
    """Column ID by CPQR with the rank cut of src/dense.py:239-264.
    Returns (sk, rd, T) with sk/rd in pivot order."""
    ncol = mq.shape[1]
    if mq.size == 0 or not np.any(mq):
        return np.arange(0), np.arange(ncol), np.zeros((0, ncol))
    _, r, piv = sla.qr(mq, mode="economic", pivoting=True, check_finite=False)
    rd = np.abs(np.diag(r))
    thr = eps * rd[0] if eps > 0.0 else max(mq.shape) * np.finfo(float).eps * rd[0]
    cut = np.flatnonzero(rd <= thr)
    k = int(cut[0]) if cut.size else rd.size
    t = (sla.solve_triangular(r[:k, :k], r[:k, k:], lower=False, check_finite=False)
         if k else np.zeros((0, ncol)))
    return piv[:k].copy(), piv[k:].copy(), t


# ---------------------------------------------------------------------------
# records (src/factor_ops.py:29-135) in the reference's LDL form
# ---------------------------------------------------------------------------

@dataclass
class ElimRec:
    cell: np.ndarray
    nbrs: np.ndarray
    L: np.ndarray
    D: np.ndarray
    X: np.ndarray      # |cell| x |nbrs| = D^-1 L^-1 A_qc^T

    def nfloats(self):
        return self.L.size + self.D.size + self.X.size

    def fwd(self, v):                       # apply_st, src/factor_ops.py:53-57
        t = sla.solve_triangular(self.L, v[self.cell], lower=True,
                                 unit_diagonal=True, check_finite=False)
        if self.nbrs.size:
            v[self.nbrs] -= self.X.T @ t
        v[self.cell] = t

    def dsolve(self, v):
        v[self.cell] = (v[self.cell].T / self.D).T

    def bwd(self, v):                       # apply_s, src/factor_ops.py:47-51
        t = v[self.cell]
        if self.nbrs.size:
            t = t - self.X @ v[self.nbrs]
        v[self.cell] = sla.solve_triangular(self.L, t, lower=True, trans="T",
                                            unit_diagonal=True, check_finite=False)

    # forward operator pieces (apply_s_inv / apply_s_inv_t / apply_d)
    def fwd_inv_t(self, v):
        t = v[self.cell]
        if self.nbrs.size:
            v[self.nbrs] += self.X.T @ t
        v[self.cell] = self.L @ t

    def dapply(self, v):
        v[self.cell] = (v[self.cell].T * self.D).T

    def bwd_inv(self, v):
        t = self.L.T @ v[self.cell]
        if self.nbrs.size:
            t = t + self.X @ v[self.nbrs]
        v[self.cell] = t


@dataclass
class SkelRec:
    cell: np.ndarray
    sk: np.ndarray
    rd: np.ndarray
    T: np.ndarray       # k x r
    elim: ElimRec | None

    def nfloats(self):
        return self.T.size + (self.elim.nfloats() if self.elim is not None else 0)

    def fwd(self, v):                       # apply_ut, src/factor_ops.py:107-110
        if self.elim is not None:
            v[self.rd] -= self.T.T @ v[self.sk]
            self.elim.fwd(v)

    def dsolve(self, v):
        if self.elim is not None:
            self.elim.dsolve(v)

    def bwd(self, v):                       # apply_u, src/factor_ops.py:102-105
        if self.elim is not None:
            self.elim.bwd(v)
            v[self.sk] -= self.T @ v[self.rd]

    def fwd_inv_t(self, v):
        if self.elim is not None:
            self.elim.fwd_inv_t(v)
            v[self.rd] += self.T.T @ v[self.sk]

    def dapply(self, v):
        if self.elim is not None:
            self.elim.dapply(v)

    def bwd_inv(self, v):
        if self.elim is not None:
            v[self.sk] += self.T @ v[self.rd]
            self.elim.bwd_inv(v)


@dataclass
class OracleFactor:
    """Generalized LDL factor (src/driver.py:64-149)."""
    n: int
    dim: int
    eps: float
    levels: list                 # [(tag, [records])]
    top_idx: np.ndarray
    top_L: np.ndarray
    top_D: np.ndarray
    metrics: dict = field(default_factory=dict)

    def nfloats(self):
        s = self.top_L.size + self.top_D.size
        for _, recs in self.levels:
            s += sum(r.nfloats() for r in recs)
        return s

    def apply_inverse(self, b):
        """src/driver.py:113-129."""
        v = np.array(b, dtype=float, copy=True)
        for _, recs in self.levels:
            for r in recs:
                r.fwd(v)
        for _, recs in self.levels:
            for r in recs:
                r.dsolve(v)
        if self.top_idx.size:
            t = sla.solve_triangular(self.top_L, v[self.top_idx], lower=True,
                                     unit_diagonal=True, check_finite=False)
            t = (t.T / self.top_D).T
            v[self.top_idx] = sla.solve_triangular(self.top_L, t, lower=True, trans="T",
                                                   unit_diagonal=True, check_finite=False)
        for _, recs in reversed(self.levels):
            for r in reversed(recs):
                r.bwd(v)
        return v

    def apply(self, x):
        """src/driver.py:95-111."""
        v = np.array(x, dtype=float, copy=True)
        for _, recs in self.levels:
            for r in recs:
                r.bwd_inv(v)
        for _, recs in self.levels:
            for r in recs:
                r.dapply(v)
        if self.top_idx.size:
            t = self.top_L.T @ v[self.top_idx]
            t = (t.T * self.top_D).T
            v[self.top_idx] = self.top_L @ t
        for _, recs in reversed(self.levels):
            for r in reversed(recs):
                r.fwd_inv_t(v)
        return v

    def skeleton_counts(self):
        """Per skeleton level (tag, sum |sk|) -- the +-2% parity quantity."""
        out = []
        for tag, recs in self.levels:
            if recs and isinstance(recs[0], SkelRec):
                out.append((tag, int(sum(r.sk.size for r in recs))))
            elif not recs and abs(tag - round(tag)) > 1e-9:
                out.append((tag, 0))
        return out


# ---------------------------------------------------------------------------
# the clique-block working matrix
# ---------------------------------------------------------------------------

class CliqueStore:
    """A_work = A0|active + sum of live dense clique blocks |active."""

    def __init__(self, csr: sp.csr_matrix):
        csr = sp.csr_matrix(csr)
        csr.sum_duplicates()
        csr.sort_indices()
        self.n = csr.shape[0]
        self.csr = csr
        self.indptr = csr.indptr.astype(np.int64)
        self.indices = csr.indices.astype(np.int64)
        self.data = csr.data.astype(np.float64)
        self.active = np.ones(self.n, dtype=bool)
        self.blk_dofs: dict[int, np.ndarray] = {}
        self.blk_vals: dict[int, np.ndarray] = {}
        self.member: list[list[int]] = [[] for _ in range(self.n)]
        self._next = 0
        self._pos = np.full(self.n, -1, dtype=np.int64)

    # -- queries -----------------------------------------------------------
    def stencil_rows(self, rows: np.ndarray):
        """(column, local row) pairs of the stencil entries of ``rows``."""
        lo = self.indptr[rows]
        cnt = self.indptr[rows + 1] - lo
        rowid = np.repeat(np.arange(rows.size), cnt)
        off = np.arange(int(cnt.sum())) - np.repeat(np.cumsum(cnt) - cnt, cnt)
        flat = np.repeat(lo, cnt) + off
        return self.indices[flat], rowid, self.data[flat]

    def blocks_touching(self, dofs) -> list[int]:
        s = set()
        for d in dofs:
            s.update(self.member[int(d)])
        return sorted(s)

    def neighbours(self, c: np.ndarray, bids) -> np.ndarray:
        """Active DOFs outside c coupled to c (src/sparse.py:164-173)."""
        nb, _, _ = self.stencil_rows(c)
        parts = [nb] + [self.blk_dofs[b] for b in bids]
        u = np.unique(np.concatenate(parts))
        self._pos[c] = 0
        keep = self.active[u] & (self._pos[u] != 0)
        self._pos[c] = -1
        return u[keep]

    # -- assembly ----------------------------------------------------------
    def _front(self, c, q, bids, only_cols_c: bool, exclude_a0_qq: bool = True):
        nc, nq = c.size, q.size
        nf = nc + nq
        pos = self._pos
        pos[c] = np.arange(nc)
        pos[q] = nc + np.arange(nq)
        ncols = nc if only_cols_c else nf
        f = np.zeros((nf, ncols))
        # original couplings of the c rows, mirrored onto the q rows
        nb, row, val = self.stencil_rows(c)
        pj = pos[nb]
        ok = pj >= 0
        row, pj, val = row[ok], pj[ok], val[ok]
        inc = pj < nc
        np.add.at(f, (row[inc], pj[inc]), val[inc])
        inq = ~inc
        np.add.at(f, (pj[inq], row[inq]), val[inq])
        if not only_cols_c:
            np.add.at(f, (row[inq], pj[inq]), val[inq])
        for b in bids:
            bd = self.blk_dofs[b]
            pb = pos[bd]
            ok = (pb >= 0) & self.active[bd]
            if not ok.any():
                continue
            li = np.flatnonzero(ok)
            pr = pb[li]
            if only_cols_c:
                lc = li[pr < nc]
                f[np.ix_(pr, pb[lc])] += self.blk_vals[b][np.ix_(li, lc)]
            else:
                f[np.ix_(pr, pr)] += self.blk_vals[b][np.ix_(li, li)]
        pos[c] = -1
        pos[q] = -1
        return f

    def _add_block(self, dofs: np.ndarray, vals: np.ndarray) -> int:
        bid = self._next
        self._next += 1
        self.blk_dofs[bid] = dofs
        self.blk_vals[bid] = vals
        for d in dofs:
            self.member[int(d)].append(bid)
        return bid

    def _drop_block(self, bid: int):
        for d in self.blk_dofs[bid]:
            self.member[int(d)].remove(bid)
        del self.blk_dofs[bid]
        del self.blk_vals[bid]

    # -- the two per-cell transforms (src/factor_ops.py:138-214) -------------
    def eliminate(self, c: np.ndarray) -> ElimRec:
        bids = self.blocks_touching(c)
        q = self.neighbours(c, bids)
        nc = c.size
        f = self._front(c, q, bids, only_cols_c=False)
        L, D, C = ldl_spd(f[:nc, :nc])
        if q.size:
            w = sla.solve_triangular(C, f[:nc, nc:], lower=True, check_finite=False)
            x = w / np.diagonal(C)[:, None]
            u = f[nc:, nc:] - w.T @ w
            u = 0.5 * (u + u.T)
        else:
            x = np.zeros((nc, 0))
        for b in bids:
            self._drop_block(b)
        if q.size:
            self._add_block(q.copy(), u)
        self.active[c] = False
        return ElimRec(c.copy(), q, L, D, x)

    def skeletonize(self, c: np.ndarray, eps: float) -> SkelRec:
        bids = self.blocks_touching(c)
        q = self.neighbours(c, bids)
        nc = c.size
        m = self._front(c, q, bids, only_cols_c=True)
        sk0, rd0, t0 = column_id(m[nc:], eps)
        so = np.argsort(sk0, kind="stable")
        ro = np.argsort(rd0, kind="stable")
        lsk, lrd = sk0[so], rd0[ro]
        t = t0[np.ix_(so, ro)]
        if lrd.size == 0:
            return SkelRec(c.copy(), c[lsk], c[lrd], t, None)
        acc = m[:nc]
        a_rr = acc[np.ix_(lrd, lrd)]
        a_sr = acc[np.ix_(lsk, lrd)]
        a_ss = acc[np.ix_(lsk, lsk)]
        b_rr = a_rr - t.T @ a_sr - a_sr.T @ t + t.T @ (a_ss @ t)
        b_rr = 0.5 * (b_rr + b_rr.T)
        b_sr = a_sr - a_ss @ t
        L, D, C = ldl_spd(b_rr)
        if lsk.size:
            w = sla.solve_triangular(C, b_sr.T, lower=True, check_finite=False)
            x = w / np.diagonal(C)[:, None]
            delta = -(w.T @ w)
            self._add_block(c[lsk].copy(), 0.5 * (delta + delta.T))
        else:
            x = np.zeros((lrd.size, 0))
        self.active[c[lrd]] = False
        elim = ElimRec(c[lrd].copy(), c[lsk].copy(), L, D, x)
        return SkelRec(c.copy(), c[lsk].copy(), c[lrd].copy(), t, elim)

    def top_block(self):
        s = np.flatnonzero(self.active)
        a0 = self.csr[s][:, s].toarray()
        pos = self._pos
        pos[s] = np.arange(s.size)
        for b, bd in self.blk_dofs.items():
            ok = self.active[bd]
            if ok.any():
                p = pos[bd[ok]]
                a0[np.ix_(p, p)] += self.blk_vals[b][np.ix_(ok, ok)]
        pos[s] = -1
        return s, a0


# ---------------------------------------------------------------------------
# drivers (src/driver.py:175-251)
# ---------------------------------------------------------------------------

def _schedule(g: Grid, variant: str, skip_levels: int, store: CliqueStore, coords):
    L = g.nlevels
    for ell in range(L):
        if variant == "hifde3x" and ell > 0:
            cells = adaptive_groups(g, ell, store, coords)
        else:
            cells = interior_groups(g, ell, store.active, coords)
        yield float(ell), cells, False
        if variant == "mf":
            continue
        if variant == "hifde":
            if ell >= skip_levels:
                kind = "edge" if g.dim == 2 else "face"
                yield ell + 0.5, interface_groups(g, ell, store.active, kind, coords), True
        else:
            yield ell + 1.0 / 3.0, interface_groups(g, ell, store.active, "face", coords), True
            if ell >= skip_levels:
                yield ell + 2.0 / 3.0, interface_groups(g, ell, store.active, "edge", coords), True


def _cell_loop_threads():
    """BLAS capped at one thread for the cell sweep unless HIFDE_NUM_THREADS
    overrides (src/driver.py:35-41,183)."""
    try:
        from threadpoolctl import threadpool_limits
    except ImportError:  # pragma: no cover
        return nullcontext()
    cap = os.environ.get("HIFDE_NUM_THREADS")
    return threadpool_limits(limits=int(cap) if cap else 1)


def factor(csr, g: Grid, eps: float, variant: str = "hifde",
           skip_levels: int | None = None, spd: bool = True) -> OracleFactor:
    """Sequential (reference-order) HIF-DE factorization.

    variant: "hifde" (src/driver.py:212-225, skip_levels default 0),
    "hifde3x" (src/driver.py:228-251, default 1) or "mf" (:201-209).
    """
    if not spd:
        raise NotImplementedError("indefinite (Bunch-Kaufman) mode is out of scope")
    if variant == "hifde3x" and g.dim != 3:
        raise ValueError("hifde3x requires a 3D grid")
    if skip_levels is None:
        skip_levels = 1 if variant == "hifde3x" else 0
    if variant == "mf":
        eps = 0.0
    t0 = time.perf_counter()
    store = CliqueStore(csr)
    coords = g.coords()
    levels = []
    trace = [(-1.0, int(store.active.sum()))]
    level_times = []
    with _cell_loop_threads():
        for tag, cells, is_skel in _schedule(g, variant, skip_levels, store, coords):
            tl = time.perf_counter()
            if is_skel:
                recs = [store.skeletonize(c, eps) for c in cells]
            else:
                recs = [store.eliminate(c) for c in cells]
            levels.append((tag, recs))
            trace.append((tag, int(store.active.sum())))
            level_times.append((tag, time.perf_counter() - tl))
    s, a_top = store.top_block()
    L, D, _ = ldl_spd(a_top)
    f = OracleFactor(store.n, g.dim, eps, levels, s, L, D)
    f.metrics = {
        "s_top": int(s.size),
        "active_trace": trace,
        "level_seconds": level_times,
        "m_f_bytes": 8 * f.nfloats(),
        "t_f_seconds": time.perf_counter() - t0,
    }
    return f


def pcg(a, b, precond=None, tol: float = 1e-12, max_iter: int = 1000):
    """Preconditioned CG on the relative residual (src/krylov.py:48-77).
    Returns (x, iterations, relative residual, converged)."""
    mv = (lambda v: a @ v)
    pc = precond if precond is not None else (lambda v: v)
    b = np.asarray(b, dtype=float)
    bn = np.linalg.norm(b)
    if bn == 0.0:
        return np.zeros_like(b), 0, 0.0, True
    x = np.zeros_like(b)
    r = b.copy()
    z = pc(r)
    p = z.copy()
    rz = float(r @ z)
    res = 1.0
    for it in range(1, max_iter + 1):
        ap = mv(p)
        alpha = rz / float(p @ ap)
        x += alpha * p
        r -= alpha * ap
        res = np.linalg.norm(r) / bn
        if res <= tol:
            return x, it, res, True
        z = pc(r)
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, max_iter, res, False


def relative_residual(csr, x_of_b, b) -> float:
    """||A F^-1 b - b|| / ||b|| (column-wise max for blocks)."""
    y = csr @ x_of_b
    r = np.linalg.norm(y - b, axis=0) / np.linalg.norm(b, axis=0)
    return float(np.max(r))
