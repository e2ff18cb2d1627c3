import os, sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1307_2895_b200 as H
for cfg in (1, 2):
    g, a, eps, variant, nrhs = H.baseline_problem(cfg)
    f = H.factor_hifde(a, g, eps)
    b = np.random.default_rng(0).standard_normal(g.ndof)
    x = f.apply_inverse(b)
    print(cfg, [c for _, c in f.metrics["skeleton_counts"]], np.linalg.norm(a @ x - b) / np.linalg.norm(b), flush=True)
