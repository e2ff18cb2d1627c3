"""Config 3 ranks, residual and factor time against the exact-order threshold
(options.exact_max_batches): which levels run in the reference's sequential
order and what the others cost in ranks."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1307_2895_b200 as H
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
g, a, eps, variant, nrhs = H.baseline_problem(cfg)
gd = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", f"cfg{cfg}.npz"))
ref = [int(c) for c in gd["skel_ranks"]]
print("reference", ref)
b = np.random.default_rng(1).standard_normal((g.ndof, 2))
fac = H.factor_hifde if variant == "hifde" else H.factor_hifde3x
for emb in (64, 40, 20, 8, 1):
    for rep in range(2):
        t0 = time.perf_counter()
        f = fac(a, g, eps, exact_max_batches=emb)
        t1 = time.perf_counter()
        if rep == 0:
            f.close()
    x = f.apply_inverse(b)
    res = float(np.max(np.linalg.norm(a @ x - b, axis=0) / np.linalg.norm(b, axis=0)))
    ranks = [c for _, c in f.metrics["skeleton_counts"]]
    dev = [f"{100.0 * (r - q) / q:+.2f}%" for r, q in zip(ranks, ref)] if ref else None
    print(f"exact_max_batches {emb:3d}: t_f {(t1 - t0) * 1e3:.1f} ms (host CSR) resid {res:.3e} ranks {ranks} vs ref {dev}", flush=True)
    f.close()
