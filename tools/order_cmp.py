"""Exact vs snapshot ordering of a config: per-level ranks, residual, GPU time."""
import sys, numpy as np
sys.path.insert(0, ".")
import paper_1307_2895_b200 as H
cfg = int(sys.argv[1])
g, a, eps, variant, nrhs = H.baseline_problem(cfg)
fac = H.factor_hifde if variant == "hifde" else H.factor_hifde3x
b = np.random.default_rng(1).standard_normal((g.ndof, 2))
res = {}
for order in ["auto", "snapshot"]:
    for r in range(2):
        f = fac(a, g, eps, order=order)
        gpu = sum(d["gpu_seconds"] for d in f.level_info)
        if r == 0:
            f.close()
    x = f.apply_inverse(b)
    rr = float(np.max(np.linalg.norm(a @ x - b, axis=0) / np.linalg.norm(b, axis=0)))
    res[order] = [c for _, c in f.metrics["skeleton_counts"]]
    print(order, "gpu ms", round(gpu * 1e3, 1), "resid", rr, "ranks", res[order], flush=True)
    f.close()
print("dev %", [round(100 * (s - e) / e, 2) for e, s in zip(res["auto"], res["snapshot"])])
