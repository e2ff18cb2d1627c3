import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_1307_2895_b200 as H
cfg = int(sys.argv[1])
g, a, eps, variant, nrhs = H.baseline_problem(cfg)
fac = H.factor_hifde if variant == "hifde" else H.factor_hifde3x
f = fac(a, g, eps)
b = torch.randn(g.ndof, 1, dtype=torch.float64, device="cuda"); x = torch.empty_like(b)
torch.cuda.synchronize()
f.apply_inverse_device(b.data_ptr(), x.data_ptr(), 1)
torch.cuda.synchronize()
