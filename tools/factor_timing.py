"""Repeated factor timing of a BASELINE config: min / median of host wall
time, and the per-level host-phase profile of the fastest repetition.

usage: python tools/factor_timing.py CFG [REPS] [host|auto]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1307_2895_b200 as H
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
sym = sys.argv[3] if len(sys.argv) > 3 else "auto"
g, a, eps, variant, nrhs = H.baseline_problem(cfg)
fac = H.factor_hifde if variant == "hifde" else H.factor_hifde3x
ts, best, best_t = [], None, 1e9
for r in range(reps):
    t = time.perf_counter()
    f = fac(a, g, eps, symbolic=sym)
    dt = time.perf_counter() - t
    ts.append(dt)
    print(f"  rep {r}: wall {dt*1e3:8.2f} ms  gpu-sum {sum(d['gpu_seconds'] for d in f.level_info)*1e3:8.2f} ms  "
          f"level-wall-sum {sum(d['seconds'] for d in f.level_info)*1e3:8.2f}", flush=True)
    if r > 0 and dt < best_t:
        best_t, best, skel = dt, f.level_info, f.metrics["skeleton_counts"]
    f.close()
ts = np.array(ts[1:]) * 1e3
print(f"cfg{cfg} symbolic={sym} factor ms: min {ts.min():.2f} median {np.median(ts):.2f} max {ts.max():.2f}")
gpu = sum(d["gpu_seconds"] for d in best) * 1e3
host = sum(d["seconds"] for d in best) * 1e3
print(f"fastest rep: sum level wall {host:.2f} ms, sum level gpu {gpu:.2f} ms; ranks {[c for _, c in skel]}")
for d in best:
    print(f"  tag {d['tag']:.3f} kind {d['kind']} groups {d['ngroups']:6d} wall {d['seconds']*1e3:7.3f} gpu {d['gpu_seconds']*1e3:7.3f}")
