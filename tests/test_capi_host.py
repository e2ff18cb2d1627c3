"""CPU-side checks of the C ABI library: it loads, exports every symbol the
public header declares, and its host partitioner reproduces the reference's
partition semantics (against the oracle restatement).  No GPU compute."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import hifde_oracle as O
from paper_1307_2895_b200 import _lib as L
from paper_1307_2895_b200._build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build()
    return L.load()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "hifde_gpu.h")).read()
    return sorted(set(re.findall(r"\b(hifde_[a-z_]+)\s*\(", src)))


def test_exports_every_header_symbol(lib):
    syms = header_symbols()
    assert set(syms) == set(L.EXPORTS)
    for s in syms:
        assert hasattr(lib, s), s


def test_version_and_device_count(lib):
    assert b"sm_100a" in lib.hifde_version()
    assert lib.hifde_device_count() >= 0


def test_bad_arguments_rejected_without_gpu(lib):
    opt = L.Options()
    lib.hifde_default_options(C.byref(opt), L.VARIANT_HIFDE3X)
    assert opt.skip_levels == 1 and opt.spd == 1
    h = C.c_void_p()
    ip = np.zeros(2, np.int64)
    ix = np.zeros(1, np.int32)
    va = np.zeros(1)
    # hifde3x on a 2D grid -> ValueError class (BADARG), before touching CUDA
    code = lib.hifde_factor(ip.ctypes.data, ix.ctypes.data, va.ctypes.data, 1, 2, 2, 2, 0,
                            C.byref(opt), C.byref(h))
    assert code == L.HIFDE_BADARG
    assert b"3D" in lib.hifde_last_error()


def _partition(lib, dim, n, m, ell, kind, active):
    N = active.size
    members = np.zeros(N, np.int32)
    offsets = np.zeros(N + 1, np.int64)
    act = np.ascontiguousarray(active.astype(np.uint8))
    ng = lib.hifde_partition(dim, n, m, ell, kind, act.ctypes.data, members.ctypes.data, N,
                             offsets.ctypes.data, N + 1)
    assert ng >= 0
    return [members[offsets[i]:offsets[i + 1]].tolist() for i in range(ng)]


CASES = [(2, 16, 2), (2, 32, 4), (2, 64, 8), (3, 8, 2), (3, 16, 4), (3, 16, 2)]


@pytest.mark.parametrize("dim,n,m", CASES)
def test_partition_matches_reference_semantics(lib, dim, n, m):
    g = O.make_grid(dim, n, m)
    rng = np.random.default_rng(dim * 100 + n + m)
    for trial in range(3):
        active = np.ones(g.ndof, bool) if trial == 0 else rng.random(g.ndof) < 0.6
        for ell in range(g.nlevels):
            got = _partition(lib, dim, n, m, ell, 0, active)
            ref = [c.tolist() for c in O.interior_groups(g, ell, active)]
            assert got == ref
            kinds = [(1, "edge")] if dim == 2 else [(2, "face"), (1, "edge")]
            for code, kind in kinds:
                got = _partition(lib, dim, n, m, ell, code, active)
                ref = [c.tolist() for c in O.interface_groups(g, ell, active, kind)]
                assert got == ref, (dim, n, m, ell, kind)


@pytest.mark.parametrize("dim,n,m", [(2, 512, 8), (3, 64, 4)])
def test_partition_large_grids_parallel_buckets(lib, dim, n, m):
    """Grids above the 65536-DOF threshold take the parallel bucket path
    (per-thread counts, prefix, scatter): same groups, same member order."""
    g = O.make_grid(dim, n, m)
    rng = np.random.default_rng(7)
    for active in (np.ones(g.ndof, bool), rng.random(g.ndof) < 0.7):
        for ell in (0, 1):
            got = _partition(lib, dim, n, m, ell, 0, active)
            ref = [c.tolist() for c in O.interior_groups(g, ell, active)]
            assert got == ref
            code, kind = (1, "edge") if dim == 2 else (2, "face")
            got = _partition(lib, dim, n, m, ell, code, active)
            ref = [c.tolist() for c in O.interface_groups(g, ell, active, kind)]
            assert got == ref
