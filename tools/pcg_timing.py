"""Factor + device PCG (tol 1e-12) of a BASELINE config: factor time, PCG
iterations and seconds, per-iteration cost (the reference's config-5 use)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1307_2895_b200 as H
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
g, a, eps, variant, nrhs = H.baseline_problem(cfg)
fac = H.factor_hifde if variant == "hifde" else H.factor_hifde3x
b = np.random.default_rng(1).standard_normal(g.ndof)
for rep in range(2):
    t0 = time.perf_counter()
    f = fac(a, g, eps)
    t1 = time.perf_counter()
    r = H.pcg_gpu(f, a, b, tol=1e-12)
    t2 = time.perf_counter()
    print(f"cfg{cfg} N={g.ndof}: factor {t1-t0:.3f} s, pcg {r.n_i} it {t2-t1:.3f} s "
          f"({1e3*(t2-t1)/max(r.n_i,1):.2f} ms/it), resid {np.linalg.norm(a@r.x-b)/np.linalg.norm(b):.2e}, "
          f"converged {r.converged}", flush=True)
    f.close()
