"""One factorization of a BASELINE config (profiling target; warm-up first)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_2895_b200 as H
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
g, a, eps, variant, nrhs = H.baseline_problem(cfg)
fac = H.factor_hifde if variant == "hifde" else H.factor_hifde3x
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    fac(a, g, eps).close()
