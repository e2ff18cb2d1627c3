"""Device vs host symbolic analysis: first differing record per level."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1307_2895_b200 as H
from paper_1307_2895_b200 import gldl
dim, n, m = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (2, 32, 4)
g = H.build_grid(dim, n, m)
a = H.assemble(g, H.constant_field(g))
fac = H.factor_hifde
eps = 1e-6
fd = fac(a, g, eps, symbolic="auto")
fh = fac(a, g, eps, symbolic="host")
print("dev ", fd.metrics["skeleton_counts"], fd.metrics["active_trace"])
print("host", fh.metrics["skeleton_counts"], fh.metrics["active_trace"])
for i, (d1, d2) in enumerate(zip(fd.level_info, fh.level_info)):
    print(i, {k: (d1[k], d2[k]) for k in ("tag", "ngroups", "nskel", "nredundant", "active_after", "max_front") if d1[k] != d2[k]})
ed, eh = gldl.export_factor(fd), gldl.export_factor(fh)
for ld, lh in zip(ed.levels, eh.levels):
    print("level", ld.level, len(ld.records), len(lh.records))
    for j, (rd, rh) in enumerate(zip(ld.records, lh.records)):
        bad = []
        if not np.array_equal(rd.cell, rh.cell): bad.append(("cell", rd.cell, rh.cell))
        if isinstance(rh, gldl.SkeletonRecord) and isinstance(rd, gldl.SkeletonRecord):
            if not np.array_equal(rd.sk, rh.sk): bad.append(("sk", rd.sk, rh.sk))
            if not np.array_equal(rd.rd, rh.rd): bad.append(("rd", rd.rd, rh.rd))
            e1, e2 = rd.elim, rh.elim
        else:
            e1, e2 = rd, rh
        if e1 is not None and e2 is not None and not np.array_equal(e1.nbrs, e2.nbrs):
            bad.append(("nbrs", e1.nbrs, e2.nbrs))
        if bad:
            print("  record", j, bad[:2])
            break
