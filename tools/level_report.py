"""Per-level host/GPU timing of one BASELINE config factor (HIFDE_PROFILE=1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("HIFDE_PROFILE", "1")
import numpy as np
import paper_1307_2895_b200 as H

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
g, a, eps, variant, nrhs = H.baseline_problem(cfg)
fac = H.factor_hifde if variant == "hifde" else H.factor_hifde3x
for r in range(reps):
    t = time.perf_counter()
    f = fac(a, g, eps)
    tf = time.perf_counter() - t
    b = np.random.default_rng(1).standard_normal((g.ndof, nrhs))
    t = time.perf_counter()
    x = f.apply_inverse(b)
    ts = time.perf_counter() - t
    res = np.max(np.linalg.norm(a @ x - b, axis=0) / np.linalg.norm(b, axis=0))
    print(f"cfg{cfg} rep{r}: factor {tf*1e3:.1f} ms solve {ts*1e3:.1f} ms resid {res:.3e} sL {f.metrics['s_top']} "
          f"ranks {[c for _, c in f.metrics['skeleton_counts']]}", flush=True)
    for d in f.level_info:
        print(f"   tag {d['tag']:.3f} kind {d['kind']} groups {d['ngroups']} front {d['max_front']} "
              f"gpu {d['gpu_seconds']*1e3:.3f} ms  gflop {d['gflop']:.3f} gbytes {d['gbytes']:.4f}", flush=True)
    f.close()
