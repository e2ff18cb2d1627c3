"""Where the end-to-end (public API, host buffers) time of a config goes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1307_2895_b200 as H
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
g, a, eps, variant, nrhs = H.baseline_problem(cfg)
fac = H.factor_hifde if variant == "hifde" else H.factor_hifde3x
b = np.random.default_rng(1).standard_normal((g.ndof, nrhs))
bp = torch.from_numpy(b).pin_memory()
dev = torch.device("cuda", 0)
ap = H.pinned_csr(a)
for rep in range(3):
    torch.cuda.synchronize()
    tp = time.perf_counter(); fp = fac(ap, g, eps); tq = time.perf_counter(); fp.close()
    t0 = time.perf_counter(); f = fac(a, g, eps); t1 = time.perf_counter()
    x = f.apply_inverse(bp.numpy()); t2 = time.perf_counter()
    x2 = f.apply_inverse(b); t3 = time.perf_counter()
    bd = torch.from_numpy(b).to(dev); xd = torch.empty_like(bd); torch.cuda.synchronize()
    t4 = time.perf_counter(); f.apply_inverse_device(bd.data_ptr(), xd.data_ptr(), nrhs); torch.cuda.synchronize(); t5 = time.perf_counter()
    h = bp.to(dev, non_blocking=True); torch.cuda.synchronize(); t6 = time.perf_counter()
    o = torch.empty(bp.shape, dtype=bp.dtype).pin_memory(); torch.cuda.synchronize(); t7 = time.perf_counter()
    o.copy_(h); torch.cuda.synchronize(); t8 = time.perf_counter()
    e = np.empty_like(b); e[...] = 0; t9 = time.perf_counter()
    print(f"rep {rep}: factor(pinned CSR) {1e3*(tq-tp):.1f} ms | factor(host CSR) {1e3*(t1-t0):.1f} ms | solve(pinned in) {1e3*(t2-t1):.1f} | solve(pageable in) {1e3*(t3-t2):.1f} | "
          f"device solve {1e3*(t5-t4):.1f} | raw H2D pinned {1e3*(t6-t5):.1f} | raw D2H pinned {1e3*(t8-t7):.1f} | "
          f"first-touch {b.nbytes/2**20:.0f} MiB {1e3*(t9-t8):.1f}", flush=True)
    f.close()
