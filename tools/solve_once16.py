"""One 16-RHS device solve of a BASELINE config's factor (profiling target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1307_2895_b200 as H
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
k = int(sys.argv[2]) if len(sys.argv) > 2 else 16
g, a, eps, variant, nrhs = H.baseline_problem(cfg)
fac = H.factor_hifde if variant == "hifde" else H.factor_hifde3x
f = fac(a, g, eps)
b = torch.randn(g.ndof, k, dtype=torch.float64, device="cuda"); x = torch.empty_like(b)
torch.cuda.synchronize()
f.apply_inverse_device(b.data_ptr(), x.data_ptr(), k)
torch.cuda.synchronize()
