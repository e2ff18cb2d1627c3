"""Exact-order skeleton timeline of a config (host analysis path, which
passes the HIFDE_SKEL_TLOG timestamp buffer)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_2895_b200 as H
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
g, a, eps, variant, nrhs = H.baseline_problem(cfg)
fac = H.factor_hifde if variant == "hifde" else H.factor_hifde3x
f = fac(a, g, eps, symbolic="host")
f = fac(a, g, eps, symbolic="host")
print(f.metrics["skeleton_counts"])
