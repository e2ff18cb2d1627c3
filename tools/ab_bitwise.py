"""Factor a few cases with the library at $HIFDE_LIB_PATH and print a digest
of the exported factor (GLDL bytes) and of a solve: run twice (A/B builds)
and compare the digests."""
import hashlib, io, os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1307_2895_b200 as H
from paper_1307_2895_b200 import gldl
cases = [(2, 64, 8, 1e-6, True, "hifde"), (2, 128, 8, 1e-9, True, "hifde"), (3, 16, 4, 1e-6, False, "hifde3x"),
         (2, 512, 8, 1e-9, True, "hifde")]
for dim, n, m, eps, hc, var in cases:
    g = H.build_grid(dim, n, m)
    a = H.assemble(g, H.gaussian_contrast_field(g, seed=3) if hc else H.constant_field(g, 1.0, 0.0))
    f = (H.factor_hifde if var == "hifde" else H.factor_hifde3x)(a, g, eps)
    p = os.path.join(tempfile.gettempdir(), f"ab_{os.getpid()}.gldl")
    gldl.save_factor(f, p)
    d1 = hashlib.sha256(open(p, "rb").read()).hexdigest()[:16]
    os.remove(p)
    x = f.apply_inverse(np.random.default_rng(0).standard_normal((g.ndof, 2)))
    d2 = hashlib.sha256(x.tobytes()).hexdigest()[:16]
    print(f"d{dim} n{n} {var}: factor {d1} solve {d2} ranks {[c for _, c in f.metrics['skeleton_counts']]}", flush=True)
