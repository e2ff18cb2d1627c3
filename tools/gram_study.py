"""Ranks / residual / time of a config with the CPQR path and the Gram path
(HIFDE_GRAM_MIN_EPS lowered), run as two subprocesses."""
import json, os, subprocess, sys
cfg = sys.argv[1] if len(sys.argv) > 1 else "4"
code = r'''
import sys, time, json, numpy as np
sys.path.insert(0, ".")
import paper_1307_2895_b200 as H
g, a, eps, variant, nrhs = H.baseline_problem(%s)
fac = H.factor_hifde if variant == "hifde" else H.factor_hifde3x
b = np.random.default_rng(1).standard_normal((g.ndof, 2))
ts = []
for r in range(3):
    t = time.perf_counter(); f = fac(a, g, eps); ts.append(time.perf_counter() - t)
    if r < 2: f.close()
x = f.apply_inverse(b)
res = float(np.max(np.linalg.norm(a @ x - b, axis=0) / np.linalg.norm(b, axis=0)))
print(json.dumps({"t": min(ts[1:]), "ranks": [c for _, c in f.metrics["skeleton_counts"]], "resid": res,
                  "gpu": sum(d["gpu_seconds"] for d in f.level_info)}))
''' % cfg
out = {}
for name, env in [("cpqr", {}), ("gram", {"HIFDE_GRAM_MIN_EPS": "1e-9"})]:
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=e)
    line = [l for l in r.stdout.splitlines() if l.startswith("{")]
    out[name] = json.loads(line[-1]) if line else r.stderr[-500:]
    print(name, out[name], flush=True)
a, b = out["cpqr"], out["gram"]
if isinstance(a, dict) and isinstance(b, dict):
    print("rank dev %:", [round(100 * (y - x) / max(x, 1), 3) for x, y in zip(a["ranks"], b["ranks"])])
