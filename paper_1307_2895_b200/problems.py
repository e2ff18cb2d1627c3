"""Problem generation: grids, coefficient fields and stencil assembly.

Mirrors the reference's discretization API (``src/discretize.py:43-192``:
``GridConfig``, ``build_grid``, ``constant_field``, ``high_contrast_field``,
``CoeffField``, ``assemble``) so benchmark and test inputs can be generated on
a machine without the reference.  ``assemble`` performs the reference's exact
floating-point sequence, so the matrix is bit-identical (pinned by the golden
fixtures' CSR digests).  This is input generation, not the hot path; it
returns a SciPy CSR matrix, which is what the factor entry points consume.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import scipy.sparse as sp

HIGH_CONTRAST_VALUES = (1e-2, 1e2)


@dataclass(frozen=True)
class GridConfig:
    dim: int
    n: int
    m: int
    nlevels: int
    h: float

    @property
    def ndof(self) -> int:
        return (self.n - 1) ** self.dim

    @property
    def side(self) -> int:
        return self.n - 1


def build_grid(dim: int, n: int, m: int) -> GridConfig:
    if dim not in (2, 3):
        raise ValueError(f"dim must be 2 or 3, got {dim}")
    if m < 2:
        raise ValueError(f"leaf width m must be >= 2, got {m}")
    if n % m:
        raise ValueError(f"n={n} is not a multiple of m={m}")
    ratio = n // m
    L = ratio.bit_length() - 1
    if (1 << L) != ratio or L < 1:
        raise ValueError(f"n={n} is not m={m} times a power of two (>= 2)")
    return GridConfig(dim, n, m, L, 1.0 / n)


@dataclass
class CoeffField:
    a: tuple
    b: np.ndarray
    contrast_ratio: Optional[float] = None


def _stag(g: GridConfig, axis: int):
    return tuple(g.n if i == axis else g.n - 1 for i in range(g.dim))


def constant_field(g: GridConfig, a0: float = 1.0, b0: float = 0.0) -> CoeffField:
    return CoeffField(tuple(np.full(_stag(g, i), float(a0)) for i in range(g.dim)),
                      np.full((g.side,) * g.dim, float(b0)))


def _smooth(g: GridConfig, noise):
    from scipy.ndimage import gaussian_filter
    return [gaussian_filter(noise(_stag(g, i)), sigma=4.0, mode="reflect", truncate=4.0)
            for i in range(g.dim)]


def gaussian_contrast_field(g: GridConfig, seed: int) -> CoeffField:
    """BASELINE.json high-contrast field: seeded N(0,1) white noise on the
    staggered grid, Gaussian-smoothed with width 4h, thresholded at zero to
    a in {1e-2, 1e2}; b = 0."""
    rng = np.random.default_rng(seed)
    lo, hi = HIGH_CONTRAST_VALUES
    a = tuple(np.where(s <= 0.0, lo, hi) for s in _smooth(g, rng.standard_normal))
    return CoeffField(a, np.zeros((g.side,) * g.dim), hi / lo)


def high_contrast_field(g: GridConfig, seed: int) -> CoeffField:
    """The reference's own variant: uniform noise split at the median
    (src/discretize.py:129-140)."""
    rng = np.random.default_rng(seed)
    sm = _smooth(g, rng.random)
    mu = np.median(np.concatenate([s.ravel() for s in sm]))
    lo, hi = HIGH_CONTRAST_VALUES
    return CoeffField(tuple(np.where(s <= mu, lo, hi) for s in sm),
                      np.zeros((g.side,) * g.dim), hi / lo)


def assemble(g: GridConfig, field: CoeffField) -> sp.csr_matrix:
    """Five-/seven-point matrix of -div(a grad u) + b u, Dirichlet BCs."""
    side, dim = g.side, g.dim
    n2 = float(g.n) * float(g.n)
    diag = np.array(field.b, dtype=float, copy=True)
    for ax in range(dim):
        sl_lo = tuple(slice(0, side) if i == ax else slice(None) for i in range(dim))
        sl_hi = tuple(slice(1, g.n) if i == ax else slice(None) for i in range(dim))
        diag += (field.a[ax][sl_lo] + field.a[ax][sl_hi]) * n2
    ids = np.arange(g.ndof, dtype=np.int64).reshape((side,) * dim, order="F")
    rows, cols, vals = [ids.ravel(order="F")], [ids.ravel(order="F")], [diag.ravel(order="F")]
    for ax in range(dim):
        head = tuple(slice(0, side - 1) if i == ax else slice(None) for i in range(dim))
        tail = tuple(slice(1, side) if i == ax else slice(None) for i in range(dim))
        i0 = ids[head].ravel(order="F")
        w = -(field.a[ax][tail] * n2).ravel(order="F")
        j0 = i0 + side ** ax
        rows += [i0, j0]
        cols += [j0, i0]
        vals += [w, w]
    m = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(g.ndof, g.ndof)).tocsr()
    m.sum_duplicates()
    m.sort_indices()
    return m


def baseline_problem(config: int, seed: int = 0):
    """(grid, A, eps, variant, nrhs) for BASELINE.json configs 1-5."""
    table = {
        1: (2, 128, 8, "const", 1e-6, "hifde", 1),
        2: (2, 512, 8, "gauss", 1e-9, "hifde", 16),
        3: (2, 2048, 8, "const", 1e-6, "hifde", 64),
        4: (3, 64, 4, "const", 1e-6, "hifde3x", 16),
        5: (3, 128, 4, "gauss", 1e-3, "hifde3x", 32),
    }
    dim, n, m, fld, eps, variant, nrhs = table[config]
    g = build_grid(dim, n, m)
    field = constant_field(g) if fld == "const" else gaussian_contrast_field(g, seed)
    return g, assemble(g, field), eps, variant, nrhs
