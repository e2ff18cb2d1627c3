"""Short profiling target: factor + 16-RHS solve of BASELINE cfg2, twice."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1307_2895_b200 as H
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
g, a, eps, variant, nrhs = H.baseline_problem(cfg)
b = np.random.default_rng(1).standard_normal((g.ndof, nrhs))
fac = H.factor_hifde if variant == "hifde" else H.factor_hifde3x
for _ in range(2):
    f = fac(a, g, eps)
    x = f.apply_inverse(b)
    f.close()
print("resid", float(np.max(np.linalg.norm(a @ x - b, axis=0) / np.linalg.norm(b, axis=0))))
