"""Device timeline of one factorization's logged launches (CUDA events, ms
from the first launch) plus the host-phase profile: shows what sits on the
critical path and what overlaps (second-stream symbolic analysis, deferred
inverses).

usage: python tools/factor_timeline.py CFG [pinned]   (prints to stderr; pinned: the CSR
in page-locked memory, H.pinned_csr)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_2895_b200 as H
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
g, a, eps, variant, nrhs = H.baseline_problem(cfg)
if len(sys.argv) > 2 and sys.argv[2] == "pinned":
    a = H.pinned_csr(a)
fac = H.factor_hifde if variant == "hifde" else H.factor_hifde3x
for _ in range(2):  # warm-up: first-call allocations, page faults
    fac(a, g, eps, kernel_log=True).close()
os.environ["HIFDE_PROFILE"] = "1"
fac(a, g, eps, kernel_log=True).close()
