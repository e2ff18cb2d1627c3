import sys, numpy as np
sys.path.insert(0, '.')
import paper_1307_2895_b200 as H
from tests import golden_cases as G
gd = G.load(sys.argv[1] if len(sys.argv) > 1 else "g3d_n32_m4_x")
g0, csr = G.build_problem(gd)
g = H.build_grid(int(gd["dim"]), int(gd["n"]), int(gd["m"]))
f = H.factor_hifde3x(csr, g, float(gd["eps"]))
print("ok", f.skeleton_counts if hasattr(f, "skeleton_counts") else "")
