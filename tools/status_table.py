"""Status table of the five BASELINE configs on this GPU: factor wall time
(host arrays, median of reps after a warm-up), GPU event time, solve time
for the configured RHS block, one-shot residual against the reference's and
the largest per-level rank deviation from the reference (tests/golden)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")
import numpy as np
import paper_1307_2895_b200 as H

HERE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
for cfg in [int(c) for c in (sys.argv[1:] or ["1", "2", "3", "4", "5"])]:
    g, a, eps, variant, nrhs = H.baseline_problem(cfg)
    fac = H.factor_hifde if variant == "hifde" else H.factor_hifde3x
    reps = 3 if g.ndof < 3_000_000 else 2
    walls, gpus = [], []
    for r in range(reps + 1):
        t = time.perf_counter()
        f = fac(a, g, eps)
        w = time.perf_counter() - t
        if r:
            walls.append(w)
            gpus.append(sum(d["gpu_seconds"] for d in f.level_info))
        if r < reps:
            f.close()
    b = np.random.default_rng(1).standard_normal((g.ndof, nrhs))
    f.apply_inverse(b)
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        x = f.apply_inverse(b)
        ts.append(time.perf_counter() - t)
    xr = np.random.default_rng(7).standard_normal(g.ndof)
    res = float(np.linalg.norm(a @ f.apply_inverse(xr) - xr) / np.linalg.norm(xr))
    name = "g2d_cfg1" if cfg == 1 else f"cfg{cfg}"
    gd = np.load(os.path.join(HERE, name + ".npz"), allow_pickle=True)
    ref = [int(v) for v in gd["skel_ranks"]]
    mine = [c for _, c in f.metrics["skeleton_counts"]]
    dev = max(abs(m - r) / max(r, 1) for m, r in zip(mine, ref)) if ref else 0.0
    print(f"cfg{cfg} N={g.ndof} factor wall {1e3*np.median(walls):.1f} ms (gpu {1e3*np.median(gpus):.1f} ms) "
          f"solve {nrhs} rhs {1e3*min(ts):.2f} ms (host arrays) oneshot resid {res:.2e} "
          f"(ref {float(np.max(gd['oneshot_resid'])):.2e}) max rank dev {100*dev:.2f}% sL {f.metrics['s_top']}", flush=True)
    f.close()
