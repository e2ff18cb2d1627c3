"""Profiling target: one factor of a BASELINE config with a chosen skeleton
ordering (auto / exact / snapshot), after one warm-up factor."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_2895_b200 as H
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
order = sys.argv[2] if len(sys.argv) > 2 else "auto"
g, a, eps, variant, nrhs = H.baseline_problem(cfg)
fac = H.factor_hifde if variant == "hifde" else H.factor_hifde3x
for _ in range(2):
    f = fac(a, g, eps, order=order)
    print("gpu ms", sum(d["gpu_seconds"] for d in f.level_info) * 1e3,
          [round(d["gpu_seconds"] * 1e3, 3) for d in f.level_info if d["kind"] == 1])
    f.close()
