"""Per-level kernel log of a BASELINE config: the factorization (phase 0)
and one device-resident solve (phase 1), CUDA events around each level's
launches (hifde_kernel_stats).  usage: tools/solve_levels.py CFG [NRHS] [PHASE]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1307_2895_b200 as H
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
nrhs_over = int(sys.argv[2]) if len(sys.argv) > 2 else 0
phase = int(sys.argv[3]) if len(sys.argv) > 3 else 1
g, a, eps, variant, nrhs = H.baseline_problem(cfg)
nrhs = nrhs_over or nrhs
fac = H.factor_hifde if variant == "hifde" else H.factor_hifde3x
fac(a, g, eps, kernel_log=True).close()  # warm-up (first-call allocations, page faults)
f = fac(a, g, eps, kernel_log=True)
b = torch.from_numpy(np.random.default_rng(1).standard_normal((g.ndof, nrhs))).cuda()
x = torch.empty_like(b)
for _ in range(3):
    f.apply_inverse_device(b.data_ptr(), x.data_ptr(), nrhs)
torch.cuda.synchronize()
st = f.kernel_stats(phase)
tot = sum(k["seconds"] for k in st)
print(f"cfg{cfg} {nrhs} RHS: {'solve' if phase else 'factor'} kernels {tot * 1e3:.2f} ms")
for k in sorted(st, key=lambda k: -k["seconds"])[:40]:
    print(f"  {k['name']:24s} tag {k['tag']:6.3f} {k['seconds'] * 1e3:7.3f} ms  {k['gbytes'] / k['seconds']:7.1f} GB/s  "
          f"{k['gflop'] / k['seconds'] * 1e-3:6.2f} TF/s")
