import os, sys, faulthandler
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(50, exit=True)
import numpy as np
import paper_1307_2895_b200 as H
g = H.build_grid(2, 32, 4)
a = H.assemble(g, H.constant_field(g))
f = H.factor_hifde(a, g, 1e-6)
print("small ok", f.metrics["s_top"], flush=True)
g, a, eps, v, nrhs = H.baseline_problem(1)
f = H.factor_hifde(a, g, eps)
print("cfg1 ok", f.metrics["s_top"], flush=True)
