"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ grid/block])."""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = collections.OrderedDict()
for r in rows[1:]:
    e = d.setdefault(r[ii], {"name": r[ki].split("(")[0].replace("void ", "")})
    e[r[mi]] = r[vi]
lim = int(sys.argv[2]) if len(sys.argv) > 2 else 10 ** 9
tot = 0.0
agg = collections.Counter()
for n, (k, v) in enumerate(d.items()):
    if n >= lim: break
    t = float(v.get("gpu__time_duration.sum", "0").replace(",", "")) / 1e3
    tot += t
    agg[v["name"]] += t
    if len(sys.argv) > 3:
        print(f"{k:>5} {v['name'][:45]:45s} grid {v.get('launch__grid_size', ''):>7} {t:9.2f} us")
for name, t in agg.most_common():
    print(f"{t:10.1f} us  {100 * t / tot:5.1f}%  {name}")
print(f"total {tot:.1f} us over {min(lim, len(d))} launches")
