"""GPU parity: the sm_100a path (through the C ABI) against the reference's
golden vectors and the CPU oracle on the same seeded inputs.

BASELINE.json criteria, as written in the tests:
  * factorization: ||A F^-1 x - x|| / ||x|| <= 10 x the reference's value;
  * solution: ||u_gpu - u_ref|| / ||u_ref|| <= 10 eps on PCG-converged
    solutions (tol 1e-12, each preconditioned by its own factor; SURVEY.md
    appendix E shows one-shot solutions of two valid factors differ by > 10 eps);
  * skeleton ranks: per-level sum |sk| within +-2% of the reference.
"""

import numpy as np
import pytest

import paper_1307_2895_b200 as H
from oracle import hifde_oracle as O
from tests import golden_cases as G

pytestmark = pytest.mark.gpu

NAMES = G.golden_names()


def _grid(gd):
    return H.build_grid(int(gd["dim"]), int(gd["n"]), int(gd["m"]))


def _factor(gd, csr, **kw):
    g = _grid(gd)
    variant = str(gd["variant"])
    eps = float(gd["eps"])
    skip = G.skip_levels(gd)
    if variant == "mf":
        return g, H.factor_mf(csr, g, **kw)
    if variant == "hifde3x":
        return g, H.factor_hifde3x(csr, g, eps, **({} if skip is None else {"skip_levels": skip}), **kw)
    return g, H.factor_hifde(csr, g, eps, **({} if skip is None else {"skip_levels": skip}), **kw)


@pytest.mark.parametrize("order", ["auto", "snapshot"])
@pytest.mark.parametrize("name", NAMES)
def test_gpu_matches_reference_golden(name, order):
    gd = G.load(name)
    _, csr = G.build_problem(gd)
    assert G.csr_digest(csr) == str(gd["csr_sha256"])
    g, f = _factor(gd, csr, order=order)
    eps = float(gd["eps"])
    tags = [t for t, _ in f.metrics["active_trace"][1:]]
    assert np.allclose(tags, gd["level_tags"])
    counts = [c for _, c in f.metrics["skeleton_counts"]]
    # default ("auto") ordering must meet BASELINE's +-2%; the opt-in snapshot
    # ordering is allowed the +2.5%-class drift SURVEY.md appendix D measured
    # for loose-eps 3D coarse levels
    rel = 0.02 if order == "auto" else 0.04
    assert G.ranks_within(counts, gd["skel_ranks"], rel=rel), (counts, gd["skel_ranks"].tolist())
    s_ref = int(gd["s_top"])
    assert abs(f.metrics["s_top"] - s_ref) <= max(1, rel * s_ref)
    b = G.rhs(gd, g.ndof)
    x = f.apply_inverse(b)
    resid = np.linalg.norm(csr @ x - b, axis=0) / np.linalg.norm(b, axis=0)
    tol = 10 * gd["oneshot_resid"] + (1e-13 if str(gd["variant"]) == "mf" else 1e-14)
    assert np.all(resid <= tol), (resid, gd["oneshot_resid"])
    rep = H.pcg(csr, b[:, 0], f.apply_inverse, tol=1e-12)
    assert rep.converged
    if "u_pcg" in gd:
        ref = gd["u_pcg"]
        diff = np.linalg.norm(rep.x - ref) / np.linalg.norm(ref)
        assert diff <= max(10 * eps, 1e-10), diff
    assert abs(rep.n_i - int(gd["pcg_iters"])) <= max(1, int(0.2 * int(gd["pcg_iters"])))


@pytest.mark.parametrize("name", NAMES)
def test_apply_matches_reference_golden(name):
    """F x through the GPU factor (GeneralizedLDL.apply, src/driver.py:95-111):
    ||F x - A x|| / ||A x|| within 10x the reference's on the golden vector,
    and apply inverts apply_inverse."""
    gd = G.load(name)
    _, csr = G.build_problem(gd)
    g, f = _factor(gd, csr)
    xa = np.random.default_rng(2).standard_normal(g.ndof)
    ax = csr @ xa
    err = np.linalg.norm(f.apply(xa) - ax) / np.linalg.norm(ax)
    assert err <= 10 * float(gd["apply_err"]) + 1e-13, (err, float(gd["apply_err"]))
    b = G.rhs(gd, g.ndof)
    back = f.apply(f.apply_inverse(b))
    assert np.linalg.norm(back - b) <= 1e-9 * np.linalg.norm(b)
    y = np.empty_like(b)
    y2 = f.apply(b)
    for j in range(b.shape[1]):  # vector and block right-hand sides agree
        y[:, j] = f.apply(b[:, j])
    assert np.allclose(y, y2, rtol=1e-12, atol=1e-14 * np.abs(y2).max())


@pytest.mark.parametrize("name", ["g2d_n64_m8_gauss", "g2d_n64_m4_hc", "g3d_n16_m4_x_gauss", "g2d_cfg1"])
def test_pcg_gpu_matches_reference(name):
    """Device-resident PCG (hifde_pcg) against the reference's pcg on its own
    factor (src/krylov.py:48-77): iteration count and the converged solution."""
    gd = G.load(name)
    _, csr = G.build_problem(gd)
    g, f = _factor(gd, csr)
    b = G.rhs(gd, g.ndof)[:, 0]
    rep = H.pcg_gpu(f, csr, b, tol=1e-12)
    host = H.pcg(csr, b, f.apply_inverse, tol=1e-12)
    assert rep.converged and host.converged
    assert abs(rep.n_i - host.n_i) <= 1
    assert abs(rep.n_i - int(gd["pcg_iters"])) <= max(1, int(0.2 * int(gd["pcg_iters"])))
    assert np.linalg.norm(csr @ rep.x - b) <= 1e-12 * np.linalg.norm(b) * 1.0001
    if "u_pcg" in gd:
        ref = gd["u_pcg"]
        assert np.linalg.norm(rep.x - ref) / np.linalg.norm(ref) <= max(10 * float(gd["eps"]), 1e-10)
    zero = H.pcg_gpu(f, csr, np.zeros(g.ndof))
    assert zero.converged and zero.n_i == 0 and not zero.x.any()


@pytest.mark.parametrize("name", [n for n in NAMES if n != "g3d_n32_m4_x"])
def test_error_estimators_match_reference(name):
    """estimate_apply_error / estimate_solve_error (src/krylov.py:153-201) on
    the device, same start vectors: the reference's estimates on its own
    factor, to the power iteration's 1e-2 stopping tolerance."""
    gd = G.load(name)
    if "e_a" not in gd:
        pytest.skip("no estimator golden")
    _, csr = G.build_problem(gd)
    g, f = _factor(gd, csr)
    ea = H.estimate_apply_error(csr, f, seed=0)
    es = H.estimate_solve_error(csr, f, seed=0)
    assert ea.converged == bool(gd["e_a_conv"]) and es.converged == bool(gd["e_s_conv"])
    for got, ref in ((ea.value, float(gd["e_a"])), (es.value, float(gd["e_s"]))):
        assert abs(got - ref) <= 0.05 * ref + 200 * np.finfo(float).eps, (got, ref)  # MF: rounding level
    # iteration counts are meaningful unless the operator error is rounding noise (MF)
    if float(gd["e_a"]) > 1e-12:
        assert abs(ea.iterations - int(gd["e_a_iters"])) <= 2
    if float(gd["e_s"]) > 1e-12:
        assert abs(es.iterations - int(gd["e_s_iters"])) <= 2


def test_densify_and_gmres():
    """densify (F I, src/driver.py:262-264) and right-preconditioned GMRES
    (src/krylov.py:80-137) on the GPU factor: the dense operator matches A
    to the factor's accuracy, GMRES converges like PCG."""
    gd = G.load("g2d_n16_m2")
    _, csr = G.build_problem(gd)
    g, f = _factor(gd, csr)
    Fd = H.densify(f)
    A = csr.toarray()
    assert Fd.shape == A.shape
    assert np.linalg.norm(Fd - A) <= 10 * float(gd["apply_err"]) * np.linalg.norm(A) + 1e-12
    assert np.allclose(Fd, Fd.T, rtol=0, atol=1e-12 * np.abs(A).max())
    b = G.rhs(gd, g.ndof)[:, 0]
    rep = H.gmres(csr, b, f.apply_inverse, tol=1e-12)
    assert rep.converged and np.linalg.norm(csr @ rep.x - b) <= 1.01e-12 * np.linalg.norm(b)
    assert abs(rep.n_i - H.pcg(csr, b, f.apply_inverse, tol=1e-12).n_i) <= 2


def test_apply_large_cells_round_trip():
    """apply on factors with cells beyond the one-CTA paths (blocked inverse,
    tiled solve records): still the exact inverse of apply_inverse."""
    g = H.build_grid(3, 24, 3)
    a = H.assemble(g, H.gaussian_contrast_field(g, seed=1))
    f = H.factor_mf(a, g)
    b = np.random.default_rng(3).standard_normal((g.ndof, 3))
    assert np.linalg.norm(f.apply(f.apply_inverse(b)) - b) <= 1e-9 * np.linalg.norm(b)
    assert np.linalg.norm(f.apply(b) - a @ b) <= 1e-10 * np.linalg.norm(a @ b)


@pytest.mark.parametrize("name", ["g2d_n32_m4", "g2d_n64_m4_hc", "g3d_n16_m4_x_hc", "g3d_n16_m2_x"])
def test_gpu_exact_order_matches_oracle(name):
    """In exact (reference) order the GPU's ranks equal the sequential oracle's
    and the factors agree as operators."""
    gd = G.load(name)
    _, csr = G.build_problem(gd)
    g, f = _factor(gd, csr, order="exact")
    og = O.make_grid(int(gd["dim"]), int(gd["n"]), int(gd["m"]))
    fo = O.factor(csr, og, float(gd["eps"]), str(gd["variant"]), G.skip_levels(gd))
    ranks = [c for _, c in f.metrics["skeleton_counts"]]
    ranks_o = [c for _, c in fo.skeleton_counts()]
    assert G.ranks_within(ranks, ranks_o, rel=0.005), (ranks, ranks_o)
    assert f.metrics["m_f_bytes"] == pytest.approx(fo.metrics["m_f_bytes"], rel=0.02)
    b = G.rhs(gd, g.ndof)
    x, xo = f.apply_inverse(b), fo.apply_inverse(b)
    r = np.max(np.linalg.norm(csr @ x - b, axis=0) / np.linalg.norm(b, axis=0))
    ro = np.max(np.linalg.norm(csr @ xo - b, axis=0) / np.linalg.norm(b, axis=0))
    assert r <= 10 * ro + 1e-14
    y, yo = f.apply(b), fo.apply(b)  # the factored operators agree
    assert np.linalg.norm(y - yo) <= 1e-6 * np.linalg.norm(yo)


def test_mf_exact_and_matches_oracle_operator():
    g = H.build_grid(2, 32, 4)
    a = H.assemble(g, H.high_contrast_field(g, seed=3))
    f = H.factor_mf(a, g)
    fo = O.factor(a, O.make_grid(2, 32, 4), 0.0, "mf")
    b = np.random.default_rng(0).standard_normal((g.ndof, 3))
    x = f.apply_inverse(b)
    assert np.linalg.norm(a @ x - b) / np.linalg.norm(b) <= 1e-12
    assert np.linalg.norm(x - fo.apply_inverse(b)) <= 1e-10 * np.linalg.norm(x)
    assert f.metrics["s_top"] == fo.metrics["s_top"]


def test_mf_top_separator_count():
    """MF top block is the top-level cross, 2(n-1)-1 DOFs (tests/test_driver.py:35-40)."""
    g = H.build_grid(2, 64, 4)
    a = H.assemble(g, H.constant_field(g))
    f = H.factor_mf(a, g)
    assert f.metrics["s_top"] == 2 * (64 - 1) - 1
    assert f.metrics["s_top"] == f.metrics["active_trace"][-1][1]


@pytest.mark.parametrize("dim,n,m", [(2, 256, 8), (3, 16, 2), (3, 24, 3)])
def test_mf_large_top_cell_blocked_inverse(dim, n, m):
    """Top cells wider than the thread-per-column inverse limit (320) take the
    blocked packed inverse (ragged last panel included); MF stays exact."""
    g = H.build_grid(dim, n, m)
    a = H.assemble(g, H.gaussian_contrast_field(g, seed=1))
    f = H.factor_mf(a, g)
    assert f.metrics["s_top"] > 320
    b = np.random.default_rng(0).standard_normal((g.ndof, 2))
    x = f.apply_inverse(b)
    assert np.max(np.linalg.norm(a @ x - b, axis=0) / np.linalg.norm(b, axis=0)) <= 1e-10


def test_single_dof_grid():
    g = H.GridConfig(dim=2, n=2, m=2, nlevels=0, h=0.5)
    a = H.assemble(g, H.constant_field(g))
    f = H.factor_mf(a, g)
    assert f.apply_inverse(np.array([16.0]))[0] == pytest.approx(1.0)


def test_vector_and_block_rhs_agree():
    g = H.build_grid(2, 64, 4)
    a = H.assemble(g, H.gaussian_contrast_field(g, seed=2))
    f = H.factor_hifde(a, g, 1e-9)
    rng = np.random.default_rng(4)
    B = rng.standard_normal((g.ndof, 5))
    X = f.apply_inverse(B)
    for j in range(5):
        xj = f.apply_inverse(B[:, j])
        assert np.allclose(xj, X[:, j], rtol=1e-12, atol=1e-14 * np.abs(X).max())
    lin = f.apply_inverse(2.5 * B[:, 0] - 1.5 * B[:, 1])
    assert np.allclose(lin, 2.5 * X[:, 0] - 1.5 * X[:, 1], atol=1e-10 * np.abs(X).max())
    # zero right-hand side
    assert not f.apply_inverse(np.zeros(g.ndof)).any()


def test_indefinite_block_raises():
    """tests/test_driver.py:214-221: a strongly negative shift makes a leaf
    block indefinite -> IndefiniteBlockError in SPD mode."""
    g = H.build_grid(2, 4, 2)
    fld = H.constant_field(g)
    fld.b[0, 0] = -1e4
    a = H.assemble(g, fld)
    with pytest.raises(H.IndefiniteBlockError):
        H.factor_mf(a, g)


def test_failed_factorizations_release_device_memory():
    """A factorization that raises (IndefiniteBlockError from the level-0
    cells of a large grid) frees its working buffers (Factorizer::release_all):
    repeated failures leave the device's free memory flat, so a caller that
    catches the error and retries does not run out of HBM."""
    import torch
    g = H.build_grid(2, 512, 8)
    fld = H.constant_field(g)
    fld.b[100:140, 100:140] = -1e4
    a = H.assemble(g, fld)
    with pytest.raises(H.IndefiniteBlockError):
        H.factor_hifde(a, g, 1e-6)
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(4):
        with pytest.raises(H.IndefiniteBlockError):
            H.factor_hifde(a, g, 1e-6)
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 <= 64 << 20, (free0 - free1) / 2**20


def test_int32_and_int64_csr_offsets_agree():
    """options.indptr_int32: scipy's int32 offsets go in as they are and are
    widened by the library; the factor is bit-identical to the one from
    int64 offsets (both through the C ABI)."""
    import ctypes as C
    from paper_1307_2895_b200 import _lib as L
    lib = L.load()
    g = H.build_grid(2, 256, 8)
    a = H.assemble(g, H.gaussian_contrast_field(g, seed=3))
    ix = np.ascontiguousarray(a.indices, dtype=np.int32)
    va = np.ascontiguousarray(a.data, dtype=np.float64)
    b = np.random.default_rng(2).standard_normal((g.ndof, 3))
    out = []
    for ip in (np.ascontiguousarray(a.indptr, dtype=np.int32), np.ascontiguousarray(a.indptr, dtype=np.int64)):
        opt = L.Options()
        lib.hifde_default_options(C.byref(opt), L.VARIANT_HIFDE)
        opt.eps = 1e-9
        opt.indptr_int32 = int(ip.dtype == np.int32)
        h = C.c_void_p()
        assert lib.hifde_factor(ip.ctypes.data, ix.ctypes.data, va.ctypes.data, g.ndof, g.dim, g.n, g.m,
                                g.nlevels, C.byref(opt), C.byref(h)) == 0
        f = H.GeneralizedLDL(h.value, lib, True)
        out.append((f.metrics["skeleton_counts"], f.apply_inverse(b)))
        f.close()
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1], out[1][1])


def test_hifde3x_rejects_2d():
    g = H.build_grid(2, 8, 2)
    a = H.assemble(g, H.constant_field(g))
    with pytest.raises(ValueError):
        H.factor_hifde3x(a, g, 1e-6)


def test_tiny_eps_behaves_like_mf():
    g = H.build_grid(2, 16, 2)
    a = H.assemble(g, H.constant_field(g))
    f = H.factor_hifde(a, g, 1e-15)
    b = np.random.default_rng(5).standard_normal(g.ndof)
    x = f.apply_inverse(b)
    assert np.linalg.norm(a @ x - b) / np.linalg.norm(b) <= 1e-12


def test_verify_noninteracting_passes():
    g = H.build_grid(3, 16, 4)
    a = H.assemble(g, H.constant_field(g))
    f = H.factor_hifde3x(a, g, 1e-6, verify=True)
    assert f.metrics["s_top"] > 0


@pytest.mark.parametrize("name", ["cfg2", "cfg4", "cfg3", "cfg5"])
def test_full_size_config_against_reference(name):
    """BASELINE configs at full size against the reference's own run
    (tests/golden/<cfg>.npz): per-level ranks within +-2%, s_top, one-shot
    residual within 10x, PCG iteration count within 10% (+-1), and the
    PCG(tol 1e-12)-converged solution within 10 eps of the reference's."""
    import os
    if not os.path.exists(os.path.join(G.GOLDEN_DIR, name + ".npz")):
        pytest.skip(f"golden {name} not generated")
    gd = G.load(name)
    g, csr = G.build_problem(gd)
    assert G.csr_digest(csr) == str(gd["csr_sha256"])
    gg = _grid(gd)
    fac = H.factor_hifde3x if str(gd["variant"]) == "hifde3x" else H.factor_hifde
    f = fac(csr, gg, float(gd["eps"]))
    counts = [c for _, c in f.metrics["skeleton_counts"]]
    assert G.ranks_within(counts, gd["skel_ranks"]), (counts, gd["skel_ranks"].tolist())
    s_ref = int(gd["s_top"])
    assert abs(f.metrics["s_top"] - s_ref) <= max(1, 0.02 * s_ref)
    b = G.rhs(gd, gg.ndof)
    x = f.apply_inverse(b)
    resid = np.linalg.norm(csr @ x - b, axis=0) / np.linalg.norm(b, axis=0)
    assert np.all(resid <= 10 * gd["oneshot_resid"]), (resid, gd["oneshot_resid"])
    rep = H.pcg(csr, b[:, 0], f.apply_inverse, tol=1e-12, max_iter=500)
    assert rep.converged
    its = int(gd["pcg_iters"])
    assert abs(rep.n_i - its) <= max(1, round(0.1 * its)), (rep.n_i, its)
    # BASELINE's solution criterion on the PCG-converged solutions: the
    # reference's u_pcg is stored in float64 (configs 2, 4) or float32
    # (configs 3, 5; storage rounding <= 6e-8 relative, far below 10 eps)
    assert "u_pcg" in gd, "golden lacks the PCG solution (regenerate with make_golden.py --big)"
    ref = gd["u_pcg"].astype(np.float64)
    diff = np.linalg.norm(rep.x - ref) / float(gd["u_pcg_norm"])
    assert diff <= 10 * float(gd["eps"]), (diff, 10 * float(gd["eps"]))


def test_many_and_odd_rhs_counts():
    """Right-hand-side blocks of 1, 3, 17 and 64 columns (tile widths 16/32,
    the 1-RHS matrix-vector paths) give the same columns as one-at-a-time
    solves, for a factor with large (tiled) records."""
    g = H.build_grid(3, 16, 2)
    a = H.assemble(g, H.gaussian_contrast_field(g, seed=3))
    f = H.factor_hifde3x(a, g, 1e-6)
    rng = np.random.default_rng(5)
    B = rng.standard_normal((g.ndof, 64))
    X = f.apply_inverse(B)
    for k in (1, 3, 17):
        Xk = f.apply_inverse(B[:, :k])
        assert np.allclose(Xk, X[:, :k], rtol=1e-12, atol=1e-13 * np.abs(X).max())
    for j in (0, 31, 63):
        assert np.allclose(f.apply_inverse(B[:, j]), X[:, j], rtol=1e-12, atol=1e-13 * np.abs(X).max())
    Y = f.apply(B[:, :17])
    assert np.allclose(Y[:, 5], f.apply(B[:, 5]), rtol=1e-12, atol=1e-13 * np.abs(Y).max())
    # beyond 64 columns: DMMA record products in 64-column chunks plus a remainder
    B2 = rng.standard_normal((g.ndof, 100))
    X2 = f.apply_inverse(B2)
    for lo, hi in ((0, 64), (64, 100), (99, 100)):
        Xk = f.apply_inverse(np.ascontiguousarray(B2[:, lo:hi]))
        assert np.allclose(Xk, X2[:, lo:hi], rtol=1e-12, atol=1e-13 * np.abs(X2).max())


def test_concurrent_solves_are_reentrant():
    """A finished factor serves concurrent apply_inverse calls from several
    host threads (each on the factor's stream, serialized by the library)."""
    import threading
    g = H.build_grid(2, 64, 4)
    a = H.assemble(g, H.constant_field(g))
    f = H.factor_hifde(a, g, 1e-9)
    rng = np.random.default_rng(6)
    Bs = [rng.standard_normal((g.ndof, 4)) for _ in range(6)]
    ref = [f.apply_inverse(B) for B in Bs]
    out = [None] * len(Bs)
    def work(i):
        out[i] = f.apply_inverse(Bs[i])
    ts = [threading.Thread(target=work, args=(i,)) for i in range(len(Bs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for x, y in zip(out, ref):
        assert np.array_equal(x, y)


def test_api_errors_are_reference_exceptions():
    """Shape errors raise ValueError (src/driver.py:237-238 style); hifde3x on
    2D and closed factors are rejected."""
    g = H.build_grid(2, 32, 4)
    a = H.assemble(g, H.constant_field(g))
    f = H.factor_hifde(a, g, 1e-6)
    with pytest.raises(ValueError):
        f.apply_inverse(np.ones(g.ndof + 1))
    with pytest.raises(ValueError):
        f.apply(np.ones((g.ndof - 1, 2)))
    with pytest.raises(ValueError):
        H.factor_hifde3x(a, g, 1e-6)
    x = f.apply_inverse(np.ones(g.ndof))
    assert np.isfinite(x).all()


_SOLVE_DUMP = r'''
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1307_2895_b200 as H
out = {}
for dim, n, m, eps, var in [(2, 64, 8, 1e-6, "hifde"), (2, 256, 8, 1e-9, "hifde"), (2, 512, 8, 1e-6, "hifde"),
                            (3, 16, 4, 1e-6, "hifde3x"), (3, 32, 4, 1e-6, "hifde3x")]:
    g = H.build_grid(dim, n, m)
    a = H.assemble(g, H.gaussian_contrast_field(g, seed=5))
    f = (H.factor_hifde if var == "hifde" else H.factor_hifde3x)(a, g, eps)
    for nrhs in (2, 3, 8, 16, 17, 32, 40, 48, 64):
        b = np.random.default_rng(nrhs).standard_normal((g.ndof, nrhs))
        out[f"{dim}_{n}_{nrhs}"] = f.apply_inverse(b)
np.savez(sys.argv[1], **out)
'''


@pytest.mark.gpu
def test_small_record_solve_kernels_match_general(tmp_path):
    """The fine-level record kernels (single load phase; DMMA tiles from 8
    right-hand sides) against the general record kernels
    (HIFDE_NO_SOLVE_SMALL, read once per process, hence the subprocesses):
    the same solutions to FP64 rounding of a different summation order."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    files = []
    for i, env in enumerate(({}, {"HIFDE_NO_SOLVE_SMALL": "1"})):
        fn = str(tmp_path / f"x{i}.npz")
        r = subprocess.run([sys.executable, "-c", _SOLVE_DUMP, fn], capture_output=True, text=True, cwd=root,
                           env=dict(os.environ, **env), timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        files.append(np.load(fn))
    for k in files[0].files:
        x, y = files[0][k], files[1][k]
        assert np.linalg.norm(x - y) <= 1e-12 * np.linalg.norm(y), (k, np.linalg.norm(x - y) / np.linalg.norm(y))


def test_pipelined_record_kernels_bit_identical(tmp_path):
    """The persistent pipelined elimination-record kernels (TMA bulk loads
    into a stage ring, producer/consumer mbarriers) run the one-record
    kernels' DMMA tiles in the same order: solutions identical bit for bit
    to those with HIFDE_NO_SOLVE_PIPE (8/16/64 RHS take the pipeline on the
    2D levels with 592+ records)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    files = []
    for i, env in enumerate(({}, {"HIFDE_NO_SOLVE_PIPE": "1"})):
        fn = str(tmp_path / f"p{i}.npz")
        r = subprocess.run([sys.executable, "-c", _SOLVE_DUMP, fn], capture_output=True, text=True, cwd=root,
                           env=dict(os.environ, **env), timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        files.append(np.load(fn))
    for k in files[0].files:
        assert np.array_equal(files[0][k], files[1][k]), k


_FACTOR_DUMP = r'''
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1307_2895_b200 as H
out = {}
for dim, n, m, eps, var, seed in [(2, 512, 8, 1e-9, "hifde", 5), (2, 2048, 8, 1e-9, "hifde", 0),
                                  (3, 64, 4, 1e-3, "hifde3x", 2)]:
    g = H.build_grid(dim, n, m)
    a = H.assemble(g, H.gaussian_contrast_field(g, seed=seed))
    f = (H.factor_hifde if var == "hifde" else H.factor_hifde3x)(a, g, eps)
    b = np.random.default_rng(7).standard_normal((g.ndof, 3))
    out[f"{dim}_{n}_x"] = f.apply_inverse(b)
    out[f"{dim}_{n}_k"] = np.array([c for _, c in f.metrics["skeleton_counts"]])
np.savez(sys.argv[1], **out)
'''


def test_warp_skeleton_kernel_bit_identical(tmp_path):
    """Snapshot levels run their groups on smaller thread teams than the
    lane split they keep -- one warp per tiny group (skel_warp_kernel),
    64-thread CTAs for the 128-thread split, 256 for the 512-thread one
    (skel_team_kernel): ranks and solutions identical bit for bit to the
    full-size CTAs' (HIFDE_NO_SKEL_WARP), on random-coefficient problems
    whose fine levels drop DOFs (2D 511^2 and 2047^2 at eps 1e-9, 3D 63^3
    at eps 1e-3; the 2047^2 grid's levels 0.5-2.5 are snapshot levels)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    files = []
    for i, env in enumerate(({}, {"HIFDE_NO_SKEL_WARP": "1"})):
        fn = str(tmp_path / f"w{i}.npz")
        r = subprocess.run([sys.executable, "-c", _FACTOR_DUMP, fn], capture_output=True, text=True, cwd=root,
                           env=dict(os.environ, **env), timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        files.append(np.load(fn))
    for k in files[0].files:
        assert np.array_equal(files[0][k], files[1][k]), k


_CERT_DUMP = r'''
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1307_2895_b200 as H
out = {}
for dim, n, m, eps, var, seed in [(2, 512, 8, 1e-6, "hifde", 5), (2, 1024, 8, 1e-5, "hifde", 1),
                                  (2, 256, 4, 1e-3, "hifde", 3), (3, 32, 4, 1e-3, "hifde3x", 2),
                                  (3, 32, 2, 1e-2, "hifde", 4)]:
    g = H.build_grid(dim, n, m)
    a = H.assemble(g, H.gaussian_contrast_field(g, seed=seed))
    f = (H.factor_hifde if var == "hifde" else H.factor_hifde3x)(a, g, eps)
    b = np.random.default_rng(7).standard_normal((g.ndof, 3))
    out[f"{dim}_{n}_{eps}_x"] = f.apply_inverse(b)
    out[f"{dim}_{n}_{eps}_k"] = np.array([c for _, c in f.metrics["skeleton_counts"]])
np.savez(sys.argv[1], **out)
'''


def test_full_rank_certificate_changes_nothing(tmp_path):
    """Small groups whose neighbour block is certified full rank (Gram
    matrix minus (16 eps |R_11|)^2 I positive definite) skip the pivoted QR:
    the record is the one the QR ends in (rank nc, nothing eliminated), so
    ranks and solutions are identical bit for bit to HIFDE_NO_RANK_CERT, on
    random-coefficient problems from eps 1e-6 (config 3's) to eps 1e-2,
    where small groups do drop DOFs and must fail the certificate."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    files = []
    for i, env in enumerate(({}, {"HIFDE_NO_RANK_CERT": "1"})):
        fn = str(tmp_path / f"c{i}.npz")
        r = subprocess.run([sys.executable, "-c", _CERT_DUMP, fn], capture_output=True, text=True, cwd=root,
                           env=dict(os.environ, **env), timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        files.append(np.load(fn))
    for k in files[0].files:
        assert np.array_equal(files[0][k], files[1][k]), k


def test_pipelined_host_solve_matches_one_block_solve():
    """Page-locked host right-hand sides take the pipelined solve (column
    chunks: strided H2D DMA, sweep, D2H pieces scattered into the caller's
    columns, all overlapped); it must equal the one-block solve of the same
    pageable data."""
    import torch
    g, a, eps, variant, nrhs = H.baseline_problem(2)
    f = H.factor_hifde(a, g, eps)
    b = torch.from_numpy(np.random.default_rng(3).standard_normal((g.ndof, 64))).pin_memory()
    x1 = f.apply_inverse(b.numpy())
    x2 = f.apply_inverse(b.numpy().copy())
    assert np.linalg.norm(x1 - x2) <= 1e-13 * np.linalg.norm(x2)
    b40 = torch.from_numpy(np.random.default_rng(4).standard_normal((g.ndof, 40))).pin_memory()
    y1 = f.apply_inverse(b40.numpy())
    y2 = f.apply_inverse(b40.numpy().copy())
    assert np.linalg.norm(y1 - y2) <= 1e-13 * np.linalg.norm(y2)


def test_pinned_csr_factor_bit_identical():
    """pinned_csr: the CSR's arrays in page-locked pool blocks (direct DMA in
    factor_hifde, no host staging) give the same factor as scipy's pageable
    arrays, bit for bit; pinned_empty arrays feed the host solve."""
    g, a, eps, variant, nrhs = H.baseline_problem(2)
    ap = H.pinned_csr(a)
    assert ap.indptr.dtype == a.indptr.dtype and (ap != a).nnz == 0
    f0 = H.factor_hifde(a, g, eps)
    f1 = H.factor_hifde(ap, g, eps)
    assert f0.metrics["skeleton_counts"] == f1.metrics["skeleton_counts"]
    b = H.pinned_empty((g.ndof, 16))
    b[...] = np.random.default_rng(9).standard_normal((g.ndof, 16))
    x0, x1 = f0.apply_inverse(b), f1.apply_inverse(b)
    assert np.array_equal(x0, x1)
    f0.close()
    f1.close()


def test_host_output_paths_agree_and_pool_recycles():
    """Large host results land in page-locked blocks of the library's pool
    (hifde_host_alloc): the DMA-straight-in result must equal the staged copy
    into a pageable caller buffer (hifde_solve on a plain numpy array) and the
    device-resident solve, and a freed block must serve the next solve."""
    import ctypes as C
    import torch
    g, a, eps, variant, nrhs = H.baseline_problem(2)
    f = H.factor_hifde(a, g, eps)
    b = torch.from_numpy(np.random.default_rng(5).standard_normal((g.ndof, 32))).pin_memory()
    x_pool = f.apply_inverse(b.numpy())
    assert x_pool.base is not None and x_pool.flags.writeable
    x_page = np.empty((g.ndof, 32))
    code = f._lib.hifde_solve(f.handle, b.numpy().ctypes.data, x_page.ctypes.data, g.ndof, 32, 0, None)
    assert code == 0
    bd = b.cuda()
    xd = torch.empty_like(bd)
    f.apply_inverse_device(bd.data_ptr(), xd.data_ptr(), 32)
    torch.cuda.synchronize()
    x_dev = xd.cpu().numpy()
    for x in (x_pool, x_page):
        assert np.linalg.norm(x - x_dev) <= 1e-13 * np.linalg.norm(x_dev)
    ptr = x_pool.ctypes.data
    del x_pool
    import gc
    gc.collect()
    x_again = f.apply_inverse(b.numpy())
    assert x_again.ctypes.data == ptr
    assert np.linalg.norm(x_again - x_dev) <= 1e-13 * np.linalg.norm(x_dev)
    y = f.apply(x_again)  # apply's output takes the pool as well
    assert np.linalg.norm(y - b.numpy()) <= 1e-8 * np.linalg.norm(b.numpy())


@pytest.mark.parametrize("dim,n,m,eps,variant,symbolic",
                         [(2, 256, 8, 1e-6, "hifde", "auto"), (3, 32, 4, 1e-3, "hifde3x", "auto"),
                          (2, 128, 4, 1e-6, "hifde", "host")])
def test_device_resident_csr_factor_bit_identical(dim, n, m, eps, variant, symbolic):
    """options.input_on_device (the bench's timed path): the CSR arrays
    already in HBM.  The host copy of the pattern is taken asynchronously
    while the device symbolic pass runs and waited for at the hand-over to
    the host analysis (hifde3x: level 1) or the end of the run; the factor
    and its solves are those of the host-CSR call, bit for bit."""
    import ctypes as C

    import torch

    from paper_1307_2895_b200 import _lib
    g = H.build_grid(dim, n, m)
    a = H.assemble(g, H.gaussian_contrast_field(g, seed=3))
    fac = H.factor_hifde if variant == "hifde" else H.factor_hifde3x
    f_host = fac(a, g, eps, symbolic=symbolic)
    dev = torch.device("cuda", 0)
    ip = torch.from_numpy(a.indptr.astype(np.int64)).to(dev)
    ix = torch.from_numpy(a.indices.astype(np.int32)).to(dev)
    va = torch.from_numpy(a.data.astype(np.float64)).to(dev)
    torch.cuda.synchronize()
    lib = _lib.load()
    b = np.random.default_rng(5).standard_normal((g.ndof, 3))
    x_host = f_host.apply_inverse(b)
    for _ in range(2):  # twice: the cached page-locked pattern buffers are reused
        opt = _lib.Options()
        lib.hifde_default_options(C.byref(opt), _lib.VARIANT_HIFDE if variant == "hifde" else _lib.VARIANT_HIFDE3X)
        opt.eps = eps
        opt.device = 0
        opt.input_on_device = 1
        opt.symbolic = _lib.SYMBOLIC[symbolic]
        h = C.c_void_p()
        code = lib.hifde_factor(ip.data_ptr(), ix.data_ptr(), va.data_ptr(), g.ndof, g.dim, g.n, g.m, g.nlevels,
                                C.byref(opt), C.byref(h))
        assert code == 0, lib.hifde_last_error().decode()
        f_dev = H.GeneralizedLDL(h.value, lib, True)
        assert f_dev.metrics["skeleton_counts"] == f_host.metrics["skeleton_counts"]
        assert np.array_equal(f_dev.apply_inverse(b), x_host)
        f_dev.close()
    f_host.close()


def test_wait_false_factor_overlaps_and_matches():
    """factor_hifde(..., wait=False) returns while the factorization runs on
    a library thread; apply_inverse of a page-locked host block queues its
    uploads at once and waits for the factor before the sweep.  Factor,
    metrics and solutions are those of the blocking call, bit for bit; a
    failing factorization raises the reference's exception at first use; a
    pending factor can be closed without being waited for."""
    import torch
    g = H.build_grid(2, 512, 8)
    a = H.assemble(g, H.gaussian_contrast_field(g, seed=2))
    f0 = H.factor_hifde(a, g, 1e-6)
    b = np.random.default_rng(3).standard_normal((g.ndof, 32))       # 67 MB: the pipelined host solve
    bp = torch.from_numpy(b).pin_memory()
    x0 = f0.apply_inverse(bp.numpy())
    for _ in range(3):
        f1 = H.factor_hifde(a, g, 1e-6, wait=False)
        x1 = f1.apply_inverse(bp.numpy())                            # uploads first, then waits
        assert np.array_equal(x0, x1)
        assert f1.metrics["skeleton_counts"] == f0.metrics["skeleton_counts"]
        assert f1.metrics["m_f_bytes"] == f0.metrics["m_f_bytes"]
        del x1
        f1.close()
    f2 = H.factor_hifde(a, g, 1e-6, wait=False)
    assert np.array_equal(f2.apply_inverse(b[:, :3]), f0.apply_inverse(b[:, :3]))  # plain path: waits first
    f2.close()
    f3 = H.factor_hifde(a, g, 1e-6, wait=False)
    assert f3.wait().metrics["s_top"] == f0.metrics["s_top"]
    f3.close()
    H.factor_hifde(a, g, 1e-6, wait=False).close()                   # never waited for
    g3 = H.build_grid(3, 32, 4)                                       # hifde3x: hand-over to the host analysis
    a3 = H.assemble(g3, H.gaussian_contrast_field(g3, seed=1))
    b3 = np.random.default_rng(4).standard_normal((g3.ndof, 4))
    f3 = H.factor_hifde3x(a3, g3, 1e-3)
    f3a = H.factor_hifde3x(a3, g3, 1e-3, wait=False)
    assert np.array_equal(f3a.apply_inverse(b3), f3.apply_inverse(b3))
    assert f3a.metrics["skeleton_counts"] == f3.metrics["skeleton_counts"]
    f3a.close()
    f3.close()
    gs = H.build_grid(2, 4, 2)
    fld = H.constant_field(gs)
    fld.b[0, 0] = -1e4
    bad = H.assemble(gs, fld)
    fb = H.factor_mf(bad, gs, wait=False)
    with pytest.raises(H.IndefiniteBlockError):
        fb.apply_inverse(np.ones(gs.ndof))
    fb.close()
    fb = H.factor_mf(bad, gs, wait=False)
    with pytest.raises(H.IndefiniteBlockError):
        fb.wait()
    fb.close()
    f0.close()
