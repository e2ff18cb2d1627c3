"""Factor cfg2 once, then 3 device-resident 16-RHS solves (profiling target)."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1307_2895_b200 as H
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
g, a, eps, variant, nrhs = H.baseline_problem(cfg)
fac = H.factor_hifde if variant == "hifde" else H.factor_hifde3x
f = fac(a, g, eps)
b = torch.randn(g.ndof, nrhs, dtype=torch.float64, device="cuda")
x = torch.empty_like(b)
for _ in range(3):
    f.apply_inverse_device(b.data_ptr(), x.data_ptr(), nrhs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st = torch.cuda.Stream()  # events and solves on one non-default stream
e0.record(st)
for _ in range(5):
    f.apply_inverse_device(b.data_ptr(), x.data_ptr(), nrhs, st.cuda_stream)
e1.record(st); torch.cuda.synchronize()
print("solve ms", e0.elapsed_time(e1) / 5)
