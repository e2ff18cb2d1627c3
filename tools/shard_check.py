"""Sharded factor (emulated ranks on one GPU) against the unsharded factor:
bitwise equality of the factor arena, ranks and solve results."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1307_2895_b200 as H
from paper_1307_2895_b200 import distributed as D
from paper_1307_2895_b200 import _lib as L
import ctypes as C


def arenas(f):
    info = L.Info()
    f._lib.hifde_get_info(f.handle, C.byref(info))
    fac = np.empty(info.fac_len)
    idx = np.empty(info.idx_len, dtype=np.int32)
    f._lib.hifde_copy_arenas(f.handle, fac.ctypes.data, fac.size, idx.ctypes.data, idx.size)
    return fac, idx


def case(dim, n, m, eps, variant, contrast, ranks):
    g = H.build_grid(dim, n, m)
    a = H.assemble(g, H.gaussian_contrast_field(g, seed=3) if contrast else H.constant_field(g, 1.0, 0.0))
    fac = {"hifde": H.factor_hifde, "hifde3x": H.factor_hifde3x, "mf": lambda a, g, e, **k: H.factor_mf(a, g, **k)}[variant]
    b = np.random.default_rng(0).standard_normal((g.ndof, 3))
    f0 = fac(a, g, eps)
    x0 = f0.apply_inverse(b)
    F0, I0 = arenas(f0)
    r0 = f0.metrics["skeleton_counts"]
    for P in ranks:
        c = D.emulated_comm(P)
        t = time.perf_counter()
        f = fac(a, g, eps, comm=c)
        dt = time.perf_counter() - t
        x = f.apply_inverse(b)
        Fp, Ip = arenas(f)
        same_f = Fp.shape == F0.shape and np.array_equal(Fp.view(np.int64), F0.view(np.int64))
        same_i = np.array_equal(Ip, I0)
        same_x = np.array_equal(x, x0)
        rel = np.linalg.norm(x - x0) / np.linalg.norm(x0)
        res = np.linalg.norm(a @ x - b) / np.linalg.norm(b)
        print(f"{variant} d{dim} n{n} P={P}: fac bitwise {same_f} idx {same_i} x bitwise {same_x} "
              f"rel {rel:.2e} resid {res:.2e} ranks same {f.metrics['skeleton_counts'] == r0} "
              f"xfer {f.metrics['xfer_bytes']/1e6:.2f} MB  {dt*1e3:.1f} ms", flush=True)
        f.close()
        c.close()


if __name__ == "__main__":
    case(2, 64, 8, 1e-6, "hifde", True, [2, 3, 4, 8])
    case(2, 64, 8, 0.0, "mf", False, [2, 4])
    case(3, 16, 4, 1e-6, "hifde3x", False, [2, 4, 8])
    case(2, 512, 8, 1e-9, "hifde", True, [4])
    case(3, 32, 4, 1e-6, "hifde3x", True, [8])
