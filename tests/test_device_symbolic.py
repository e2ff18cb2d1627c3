"""The device symbolic pass (partition, neighbour sets, task tables and block
bookkeeping on the GPU, csrc/symbolic.cu) against the host analysis
(csrc/runtime.cu, partition.cpp): both must give the same factor, record for
record and bit for bit -- the same groups, neighbour sets, skeletons, block
ids (hence summation orders) and values."""

import numpy as np
import pytest

import paper_1307_2895_b200 as H
from paper_1307_2895_b200 import gldl

pytestmark = pytest.mark.gpu

CASES = [
    # dim, n, m, field, eps, variant, order
    (2, 32, 4, "const", 1e-6, "hifde", "auto"),
    (2, 64, 8, "gauss", 1e-9, "hifde", "auto"),
    (2, 64, 4, "gauss", 1e-6, "hifde", "snapshot"),
    (2, 128, 8, "const", 1e-6, "hifde", "exact"),
    (2, 32, 4, "const", 0.0, "mf", "auto"),
    (3, 16, 4, "const", 1e-6, "hifde", "auto"),
    (3, 16, 4, "gauss", 1e-3, "hifde3x", "auto"),
    (3, 32, 4, "gauss", 1e-3, "hifde3x", "auto"),
]


def _problem(dim, n, m, field):
    g = H.build_grid(dim, n, m)
    fld = H.constant_field(g) if field == "const" else H.gaussian_contrast_field(g, seed=3)
    return g, H.assemble(g, fld)


def _factor(g, a, eps, variant, order, symbolic):
    if variant == "mf":
        return H.factor_mf(a, g, symbolic=symbolic)
    fac = H.factor_hifde3x if variant == "hifde3x" else H.factor_hifde
    return fac(a, g, eps, order=order, symbolic=symbolic)


def _same(a, b, what):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, what
    assert np.array_equal(a, b), what


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}d_n{c[1]}_m{c[2]}_{c[3]}_{c[5]}_{c[6]}" for c in CASES])
def test_device_symbolic_bitwise_equals_host(case):
    dim, n, m, field, eps, variant, order = case
    g, a = _problem(dim, n, m, field)
    fd = _factor(g, a, eps, variant, order, "auto")
    fh = _factor(g, a, eps, variant, order, "host")
    assert fd.metrics["skeleton_counts"] == fh.metrics["skeleton_counts"]
    assert fd.metrics["s_top"] == fh.metrics["s_top"]
    assert fd.metrics["m_f_bytes"] == fh.metrics["m_f_bytes"]
    assert [t for t, _ in fd.metrics["active_trace"]] == [t for t, _ in fh.metrics["active_trace"]]
    assert fd.metrics["active_trace"] == fh.metrics["active_trace"]
    ed, eh = gldl.export_factor(fd), gldl.export_factor(fh)
    assert len(ed.levels) == len(eh.levels)
    for ld, lh in zip(ed.levels, eh.levels):
        assert ld.level == lh.level and len(ld.records) == len(lh.records)
        for rd, rh in zip(ld.records, lh.records):
            _same(rd.cell, rh.cell, "cell")
            if isinstance(rh, gldl.SkeletonRecord):
                _same(rd.sk, rh.sk, "sk")
                _same(rd.rd, rh.rd, "rd")
                _same(rd.interp, rh.interp, "T")
                rd, rh = rd.elim, rh.elim
                if rh is None:
                    assert rd is None
                    continue
            _same(rd.nbrs, rh.nbrs, "nbrs")
            _same(rd.factor.lower, rh.factor.lower, "L")
            _same(rd.factor.d.diag, rh.factor.d.diag, "D")
            _same(rd.coupling, rh.coupling, "X")
    _same(ed.top_idx, eh.top_idx, "top")
    b = np.random.default_rng(0).standard_normal((g.ndof, 3))
    _same(fd.apply_inverse(b), fh.apply_inverse(b), "solve")


def test_device_symbolic_full_size_config2_bitwise():
    """Config 2 at full size: device and host analysis give the same solve."""
    g, a, eps, variant, nrhs = H.baseline_problem(2)
    fd = H.factor_hifde(a, g, eps)
    fh = H.factor_hifde(a, g, eps, symbolic="host")
    assert fd.metrics["skeleton_counts"] == fh.metrics["skeleton_counts"]
    b = np.random.default_rng(0).standard_normal((g.ndof, 4))
    _same(fd.apply_inverse(b), fh.apply_inverse(b), "solve")
