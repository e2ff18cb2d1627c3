"""Skeleton-rank drift of snapshot vs exact (reference) group ordering,
against the reference's golden per-level ranks."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1307_2895_b200 as H
from tests import golden_cases as G

for name in sys.argv[1:] or ["g2d_cfg1", "cfg2", "g2d_n64_m8_gauss", "g3d_n16_m4_x_hc", "g3d_n16_m4_x_gauss", "g3d_n32_m4_x"]:
    gd = G.load(name)
    g = H.build_grid(int(gd["dim"]), int(gd["n"]), int(gd["m"]))
    _, a = G.build_problem(gd)
    ref = gd["skel_ranks"].tolist()
    for order in ("exact", "snapshot"):
        fac = H.factor_hifde3x if str(gd["variant"]) == "hifde3x" else H.factor_hifde
        f = fac(a, g, float(gd["eps"]), order=order)
        got = [c for _, c in f.metrics["skeleton_counts"]]
        dev = [f"{100*(x-y)/y:+.2f}%" for x, y in zip(got, ref)]
        ngroups = [d["ngroups"] for d in f.level_info if d["kind"] == 1]
        print(f"{name:20s} {order:8s} groups={ngroups} dev={dev}", flush=True)
