"""End-to-end step through the public API with host arrays (bench.py's e2e):
factor(host CSR) + apply_inverse(host 16-RHS block), wall time per step."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1307_2895_b200 as H
g, a, eps, variant, nrhs = H.baseline_problem(2)
b = np.random.default_rng(1).standard_normal((g.ndof, nrhs))
ts, tf, tsol = [], [], []
for rep in range(12):
    t0 = time.perf_counter()
    f = H.factor_hifde(a, g, eps)
    t1 = time.perf_counter()
    x = f.apply_inverse(b)
    t2 = time.perf_counter()
    f.close()
    if rep >= 2:
        ts.append(t2 - t0); tf.append(t1 - t0); tsol.append(t2 - t1)
print(f"e2e step ms: median {1e3*np.median(ts):.2f} min {1e3*min(ts):.2f} | factor {1e3*np.median(tf):.2f} | solve {1e3*np.median(tsol):.2f}")
