"""One factor + one device-resident RHS-block solve of a BASELINE config
(for ncu captures: the first launches of each kernel are the fine levels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1307_2895_b200 as H
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
g, a, eps, variant, nrhs = H.baseline_problem(cfg)
fac = H.factor_hifde if variant == "hifde" else H.factor_hifde3x
f = fac(a, g, eps)
b = torch.from_numpy(np.random.default_rng(1).standard_normal((g.ndof, nrhs))).cuda()
x = torch.empty_like(b)
f.apply_inverse_device(b.data_ptr(), x.data_ptr(), nrhs)
torch.cuda.synchronize()
print("ok", f.metrics["skeleton_counts"])
