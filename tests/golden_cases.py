"""Shared helpers: load committed golden fixtures and rebuild their inputs
without the reference (the GPU box has no /root/reference)."""

from __future__ import annotations

import glob
import hashlib
import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden_names(include_big: bool = False):
    names = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz"))
                   if not p.endswith("_idx.npz"))  # record index sets, not cases
    if not include_big:
        names = [n for n in names if not n.startswith("cfg")]
    return names


def load(name: str) -> dict:
    with np.load(os.path.join(GOLDEN_DIR, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def csr_digest(csr) -> str:
    h = hashlib.sha256()
    for arr in (csr.indptr.astype(np.int64), csr.indices.astype(np.int64),
                csr.data.astype(np.float64)):
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


def build_problem(gd: dict):
    """(grid, csr) for a golden case, via the oracle's problem generator."""
    from oracle import hifde_oracle as O
    dim, n, m = int(gd["dim"]), int(gd["n"]), int(gd["m"])
    g = O.make_grid(dim, n, m)
    fld = str(gd["field"])
    seed = int(gd["seed"])
    if fld == "const":
        a, b = O.constant_coeffs(g)
    elif fld == "median":
        a, b = O.median_contrast_coeffs(g, seed)
    else:
        a, b = O.gaussian_contrast_coeffs(g, seed)
    return g, O.assemble_csr(g, a, b)


def rhs(gd: dict, n: int):
    return np.random.default_rng(1).standard_normal((n, int(gd["nrhs"])))


def skip_levels(gd: dict):
    s = int(gd["skip_levels"])
    return None if s < 0 else s


def ranks_within(got, ref, rel=0.02, abs_slack=1):
    """Per-level skeleton counts within +-rel of the reference (BASELINE
    criterion); tiny levels get a one-DOF slack."""
    got = np.asarray(got, dtype=float)
    ref = np.asarray(ref, dtype=float)
    if got.shape != ref.shape:
        return False
    return bool(np.all(np.abs(got - ref) <= np.maximum(rel * ref, abs_slack)))
