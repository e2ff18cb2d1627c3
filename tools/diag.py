"""Quick GPU-vs-oracle diagnostic on small cases (prints, never asserts)."""
import sys, os, time, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1307_2895_b200 as H
from oracle import hifde_oracle as O

def run(dim, n, m, eps, variant, field="const", order="auto"):
    g = H.build_grid(dim, n, m)
    fld = H.constant_field(g) if field == "const" else H.gaussian_contrast_field(g, 0)
    a = H.assemble(g, fld)
    try:
        t = time.time()
        f = (H.factor_hifde if variant == "hifde" else H.factor_hifde3x if variant == "hifde3x" else (lambda a, g, e, **k: H.factor_mf(a, g, **k)))(a, g, eps, order=order)
        tg = time.time() - t
    except Exception:
        traceback.print_exc(); return
    t = time.time()
    fo = O.factor(a, O.make_grid(dim, n, m), eps, variant)
    to = time.time() - t
    b = np.random.default_rng(1).standard_normal((g.ndof, 2))
    x = f.apply_inverse(b); xo = fo.apply_inverse(b)
    r = np.max(np.linalg.norm(a @ x - b, axis=0) / np.linalg.norm(b, axis=0))
    ro = np.max(np.linalg.norm(a @ xo - b, axis=0) / np.linalg.norm(b, axis=0))
    print(f"{dim}D n={n} m={m} eps={eps} {variant} {field} {order}: t_gpu={tg:.3f}s t_or={to:.2f}s "
          f"resid gpu={r:.3e} oracle={ro:.3e} dx={np.linalg.norm(x-xo)/np.linalg.norm(xo):.2e} "
          f"sL {f.metrics['s_top']}/{fo.metrics['s_top']} mf {f.metrics['m_f_bytes']}/{fo.metrics['m_f_bytes']}")
    print("   ranks gpu", [c for _, c in f.metrics["skeleton_counts"]], " oracle", [c for _, c in fo.skeleton_counts()])
    print("   trace gpu", [t for _, t in f.metrics["active_trace"]])
    print("   trace ora", [t for _, t in fo.metrics["active_trace"]], flush=True)

if __name__ == "__main__":
    print("devices", H.device_count())
    run(2, 8, 2, 0.0, "mf")
    run(2, 16, 2, 1e-6, "hifde")
    run(2, 32, 4, 1e-6, "hifde", order="exact")
    run(2, 64, 8, 1e-9, "hifde", "gauss")
    run(2, 128, 8, 1e-6, "hifde")
    run(3, 8, 2, 1e-6, "hifde")
    run(3, 16, 4, 1e-3, "hifde3x", "gauss", order="exact")
    run(3, 16, 2, 1e-6, "hifde3x", order="exact")
