"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import hifde_oracle as O
from tests import golden_cases as G

NAMES = G.golden_names()


@pytest.mark.parametrize("name", NAMES)
def test_problem_generator_bit_identical(name):
    gd = G.load(name)
    _, csr = G.build_problem(gd)
    assert G.csr_digest(csr) == str(gd["csr_sha256"])


@pytest.mark.parametrize("name", NAMES)
def test_oracle_matches_reference(name):
    gd = G.load(name)
    g, csr = G.build_problem(gd)
    eps = float(gd["eps"])
    f = O.factor(csr, g, eps, str(gd["variant"]), G.skip_levels(gd))
    # level structure
    assert np.allclose([t for t, _ in f.levels], gd["level_tags"])
    counts = [c for _, c in f.skeleton_counts()]
    assert G.ranks_within(counts, gd["skel_ranks"]), (counts, gd["skel_ranks"])
    assert abs(f.metrics["s_top"] - int(gd["s_top"])) <= max(1, 0.02 * int(gd["s_top"]))
    # factorization criterion: residual within 10x of the reference's
    b = G.rhs(gd, g.ndof)
    x = f.apply_inverse(b)
    resid = np.linalg.norm(csr @ x - b, axis=0) / np.linalg.norm(b, axis=0)
    assert np.all(resid <= 10 * gd["oneshot_resid"] + 1e-14)
    # solution criterion on PCG-converged solutions
    u, its, res, ok = O.pcg(csr, b[:, 0], f.apply_inverse, tol=1e-12)
    assert ok
    if "u_pcg" in gd:
        ref = gd["u_pcg"]
        diff = np.linalg.norm(u - ref) / np.linalg.norm(ref)
        assert diff <= max(10 * eps, 1e-10), diff
    assert abs(its - int(gd["pcg_iters"])) <= max(1, int(0.2 * int(gd["pcg_iters"])))


def test_oracle_exact_on_reference_trace():
    """On the 2D golden cases the restatement reproduces the reference's
    active-DOF trace and factor size exactly."""
    for name in ("g2d_n16_m2", "g2d_n32_m4", "g2d_cfg1", "g2d_n32_m4_mf"):
        gd = G.load(name)
        g, csr = G.build_problem(gd)
        f = O.factor(csr, g, float(gd["eps"]), str(gd["variant"]), G.skip_levels(gd))
        assert [t[1] for t in f.metrics["active_trace"]] == gd["trace"].tolist()
        assert f.metrics["m_f_bytes"] == int(gd["m_f_bytes"])


def test_mf_is_exact():
    gd = G.load("g2d_n32_m4_mf")
    g, csr = G.build_problem(gd)
    f = O.factor(csr, g, 0.0, "mf")
    b = G.rhs(gd, g.ndof)
    x = f.apply_inverse(b)
    assert np.linalg.norm(csr @ x - b) / np.linalg.norm(b) <= 1e-12


def test_dense_kernel_known_answers():
    """Hand values of the reference's dense-kernel tests
    (tests/test_dense_kernels.py:13-21,74-82)."""
    L, D, _ = O.ldl_spd(np.array([[4.0]]))
    assert D[0] == pytest.approx(4.0)
    L, D, _ = O.ldl_spd(np.array([[2.0, 1.0], [1.0, 2.0]]))
    assert D.tolist() == pytest.approx([2.0, 1.5]) and L[1, 0] == pytest.approx(0.5)
    sk, rd, t = O.column_id(np.array([[1.0, 2.0], [2.0, 4.0]]), 1e-12)
    assert sk.tolist() == [1] and rd.tolist() == [0] and float(t[0, 0]) == pytest.approx(0.5)
    sk, rd, t = O.column_id(np.zeros((3, 2)), 1e-6)
    assert sk.size == 0 and rd.tolist() == [0, 1]
    with pytest.raises(O.OracleIndefiniteError):
        O.ldl_spd(np.array([[1.0, 2.0], [2.0, 1.0]]))
