"""GLDL v1 factor files and record export (hifde_level_records /
hifde_copy_arenas): the reference's own factor files (tests/golden/*.gldl,
written by its save_factor, src/driver.py:292-315) are the fixtures."""

import os

import numpy as np
import pytest

from paper_1307_2895_b200 import gldl
from tests import golden_cases as G

HERE = os.path.join(os.path.dirname(__file__), "golden")
CASES = ["g2d_n16_m2", "g2d_n32_m4", "g3d_n8_m2"]


@pytest.mark.parametrize("name", CASES)
def test_gldl_writer_reproduces_reference_bytes(name, tmp_path):
    """read_gldl + write_gldl round-trips the reference's file byte for byte."""
    src = os.path.join(HERE, f"{name}.gldl")
    ef = gldl.read_gldl(src)
    out = tmp_path / "copy.gldl"
    gldl.write_gldl(ef, out)
    assert open(src, "rb").read() == open(out, "rb").read()
    gd = G.load(name)
    assert ef.n == int(np.prod([int(gd["n"]) - 1] * int(gd["dim"])))
    assert [lf.level for lf in ef.levels] == [float(t) for t in gd["level_tags"]]
    assert len(ef.top_idx) == int(gd["s_top"])


def _close(a, b, rtol):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape
    if a.size == 0:
        return
    scale = max(np.abs(b).max(), 1e-300)
    assert np.abs(a - b).max() <= rtol * scale, np.abs(a - b).max() / scale


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_export_matches_reference_records(name, tmp_path):
    """The GPU factor, exported, equals the reference's factor record by
    record: identical index sets (cells, neighbours, skeletons, redundant
    DOFs, top block) and L, D, X, T within 1e-7 of each record's scale."""
    import paper_1307_2895_b200 as H
    gd = G.load(name)
    _, csr = G.build_problem(gd)
    g = H.build_grid(int(gd["dim"]), int(gd["n"]), int(gd["m"]))
    f = H.factor_hifde(csr, g, float(gd["eps"]), order="exact")
    ref = gldl.read_gldl(os.path.join(HERE, f"{name}.gldl"))
    ours = gldl.export_factor(f)
    assert (ours.n, ours.dim, ours.spd) == (ref.n, ref.dim, ref.spd)
    assert ours.eps == pytest.approx(ref.eps)
    assert [lf.level for lf in ours.levels] == pytest.approx([lf.level for lf in ref.levels])
    for lo, lr in zip(ours.levels, ref.levels):
        assert len(lo.records) == len(lr.records), lo.level
        for ro, rr in zip(lo.records, lr.records):
            assert type(ro).__name__ == type(rr).__name__
            np.testing.assert_array_equal(ro.cell, rr.cell)
            if isinstance(rr, gldl.EliminationRecord):
                eo, er = ro, rr
            else:
                np.testing.assert_array_equal(ro.sk, rr.sk)
                np.testing.assert_array_equal(ro.rd, rr.rd)
                _close(ro.interp, rr.interp, 1e-7)
                assert (ro.elim is None) == (rr.elim is None)
                if rr.elim is None:
                    continue
                eo, er = ro.elim, rr.elim
            np.testing.assert_array_equal(eo.cell, er.cell)
            np.testing.assert_array_equal(eo.nbrs, er.nbrs)
            _close(eo.factor.lower, er.factor.lower, 1e-7)
            _close(eo.factor.d.diag, er.factor.d.diag, 1e-7)
            _close(eo.coupling, er.coupling, 1e-7)
    np.testing.assert_array_equal(ours.top_idx, ref.top_idx)
    _close(ours.top.lower, ref.top.lower, 1e-7)
    _close(ours.top.d.diag, ref.top.d.diag, 1e-7)
    # save_factor writes what export_factor returns, in the reference layout
    path = tmp_path / "ours.gldl"
    H.save_factor(f, path)
    back = gldl.read_gldl(path)
    assert len(back.levels) == len(ours.levels)
    np.testing.assert_array_equal(back.top_idx, ours.top_idx)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_load_reference_factor_onto_gpu(name, tmp_path):
    """load_factor of the reference's own file: the GPU sweeps of the loaded
    factor reproduce the reference's apply_inverse on the golden vectors, and
    a save/load round trip of a GPU factor keeps its operator."""
    import paper_1307_2895_b200 as H
    gd = G.load(name)
    _, csr = G.build_problem(gd)
    f = H.load_factor(os.path.join(HERE, f"{name}.gldl"))
    b = G.rhs(gd, f.n)
    x = f.apply_inverse(b)
    ref = gd["x_oneshot"]
    assert np.linalg.norm(x - ref) <= 1e-10 * np.linalg.norm(ref)
    xa = np.random.default_rng(2).standard_normal(f.n)
    ax = csr @ xa
    err = np.linalg.norm(f.apply(xa) - ax) / np.linalg.norm(ax)
    assert err <= 1.01 * float(gd["apply_err"]) + 1e-14
    assert f.metrics["s_top"] == int(gd["s_top"])
    # GPU factor -> file -> GPU factor
    g = H.build_grid(int(gd["dim"]), int(gd["n"]), int(gd["m"]))
    f0 = H.factor_hifde(csr, g, float(gd["eps"]))
    path = tmp_path / "gpu.gldl"
    H.save_factor(f0, path)
    f1 = H.load_factor(path)
    y0, y1 = f0.apply_inverse(b), f1.apply_inverse(b)
    assert np.linalg.norm(y1 - y0) <= 1e-10 * np.linalg.norm(y0)
