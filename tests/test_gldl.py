"""GLDL v1 factor files and record export (hifde_level_records /
hifde_copy_arenas): the reference's own factor files (tests/golden/*.gldl,
written by its save_factor, src/driver.py:292-315) are the fixtures."""

import os

import numpy as np
import pytest

from paper_1307_2895_b200 import gldl
from tests import golden_cases as G

HERE = os.path.join(os.path.dirname(__file__), "golden")
CASES = ["g2d_n16_m2", "g2d_n32_m4", "g3d_n8_m2", "g3d_n16_m4_x_gauss"]
# record values (L, D, X, T) against the reference's, relative to each record's
# scale: FP64 rounding of the same pivots and the same ID (2D), a little more
# for the deeper 3D eliminations
VALUE_RTOL = {"g2d_n16_m2": 1e-11, "g2d_n32_m4": 1e-11, "g3d_n8_m2": 1e-10, "g3d_n16_m4_x_gauss": 1e-9}


def _factor_case(H, gd, csr, **kw):
    g = H.build_grid(int(gd["dim"]), int(gd["n"]), int(gd["m"]))
    if str(gd["variant"]) == "hifde3x":
        return H.factor_hifde3x(csr, g, float(gd["eps"]), **kw)
    return H.factor_hifde(csr, g, float(gd["eps"]), **kw)


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
    DOFs, top block) and L, D, X, T within VALUE_RTOL of each record's
    scale.  The hifde3x case (random coefficients: no pivot ties) pins the
    adaptive separators (src/partition.py:184-227) index for index."""
    import paper_1307_2895_b200 as H
    gd = G.load(name)
    _, csr = G.build_problem(gd)
    f = _factor_case(H, gd, csr, order="exact")
    rtol = VALUE_RTOL[name]
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
                _close(ro.interp, rr.interp, rtol)
                assert (ro.elim is None) == (rr.elim is None)
                if rr.elim is None:
                    continue
                eo, er = ro.elim, rr.elim
            np.testing.assert_array_equal(eo.cell, er.cell)
            np.testing.assert_array_equal(eo.nbrs, er.nbrs)
            _close(eo.factor.lower, er.factor.lower, rtol)
            _close(eo.factor.d.diag, er.factor.d.diag, rtol)
            _close(eo.coupling, er.coupling, rtol)
    np.testing.assert_array_equal(ours.top_idx, ref.top_idx)
    _close(ours.top.lower, ref.top.lower, rtol)
    _close(ours.top.d.diag, ref.top.d.diag, rtol)
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
    f0 = _factor_case(H, gd, csr)
    path = tmp_path / "gpu.gldl"
    H.save_factor(f0, path)
    f1 = H.load_factor(path)
    y0, y1 = f0.apply_inverse(b), f1.apply_inverse(b)
    assert np.linalg.norm(y1 - y0) <= 1e-10 * np.linalg.norm(y0)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["g3d_n32_m4_x_gauss"])
def test_export_matches_reference_index_sets(name):
    """A larger hifde3x case (31^3, three adaptive levels): every record's
    index sets -- cells, neighbours, skeletons, redundant DOFs -- and the top
    block equal the reference's (tests/golden/<name>_idx.npz, from its own
    factor): the adaptive separators (src/partition.py:184-227), neighbour
    sets and the sequential-order truncation are bit-exact."""
    import paper_1307_2895_b200 as H
    gd = G.load(name)
    _, csr = G.build_problem(gd)
    f = _factor_case(H, gd, csr, order="exact")
    ours = gldl.export_factor(f)
    with np.load(os.path.join(HERE, f"{name}_idx.npz")) as z:
        ref = {k: z[k] for k in z.files}
    assert [lf.level for lf in ours.levels] == pytest.approx(list(ref["tags"]))
    for li, lf in enumerate(ours.levels):
        got = {"cell": [], "nbrs": [], "sk": [], "rd": []}
        for r in lf.records:
            e = r if isinstance(r, gldl.EliminationRecord) else r.elim
            got["cell"].append(np.asarray(r.cell, dtype=np.int64))
            got["nbrs"].append(np.asarray(e.nbrs if e is not None else [], dtype=np.int64))
            got["sk"].append(np.asarray(getattr(r, "sk", []), dtype=np.int64))
            got["rd"].append(np.asarray(getattr(r, "rd", []), dtype=np.int64))
        for k, v in got.items():
            ptr = np.cumsum([0] + [len(x) for x in v])
            np.testing.assert_array_equal(ptr, ref[f"l{li}_{k}_ptr"], err_msg=f"level {lf.level} {k} sizes")
            flat = np.concatenate(v) if v else np.zeros(0, np.int64)
            np.testing.assert_array_equal(flat, ref[f"l{li}_{k}"], err_msg=f"level {lf.level} {k}")
    np.testing.assert_array_equal(ours.top_idx, ref["top_idx"])
