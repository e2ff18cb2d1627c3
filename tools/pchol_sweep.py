"""GPU time and ranks of configs 4 / 5 for each pivoted-Cholesky launch mode
(HIFDE_PCHOL_CL), each in its own process."""
import os, subprocess, sys, json
code = r'''
import sys, json, numpy as np
sys.path.insert(0, ".")
import paper_1307_2895_b200 as H
cfg = int(sys.argv[1])
g, a, eps, variant, nrhs = H.baseline_problem(cfg)
fac = H.factor_hifde if variant == "hifde" else H.factor_hifde3x
gs = []
for r in range(3):
    f = fac(a, g, eps)
    gs.append(sum(d["gpu_seconds"] for d in f.level_info))
    ranks = [c for _, c in f.metrics["skeleton_counts"]]
    f.close()
print(json.dumps({"gpu_ms": 1e3 * min(gs[1:]), "ranks": ranks}))
'''
for cfg in sys.argv[1:]:
    for mode in ["0", "2", "4", "8", "16", ""]:
        env = dict(os.environ)
        if mode:
            env["HIFDE_PCHOL_CL"] = mode
        r = subprocess.run([sys.executable, "-c", code, cfg], capture_output=True, text=True, env=env, timeout=600)
        line = [l for l in r.stdout.splitlines() if l.startswith("{")]
        print(f"cfg{cfg} mode {mode or 'default'}:", line[-1] if line else r.stderr[-400:], flush=True)
