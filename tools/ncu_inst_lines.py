"""Top CUDA source lines of an ncu `--page source --csv --print-source cuda,sass`
dump by executed warp instructions (with their share of the stall samples)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 45
agg = collections.defaultdict(lambda: [0, 0, ''])
fname, cur, H = '', None, None
for r in rows:
    if r and r[0] in ('File Path', 'File Name'):
        fname = r[1].split('/')[-1]
        continue
    if r and r[0] == 'Line No':
        H = r
        ie = H.index('Instructions Executed')
        si = H.index('Warp Stall Sampling (All Samples)')
        continue
    if H is None or len(r) <= max(ie, si):
        continue
    if r[0]:
        cur = (fname, r[0])
        agg[cur][2] = r[1].strip()[:90]
    if cur is None:
        continue
    try:
        agg[cur][0] += int(r[ie])
        agg[cur][1] += int(r[si])
    except ValueError:
        pass
tot = sum(v[0] for v in agg.values())
smp = sum(v[1] for v in agg.values())
print('total inst', tot, 'samples', smp)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * v[0] / tot:5.1f}% inst {100 * v[1] / max(smp, 1):5.1f}% smp {k[0]}:{k[1]}  {v[2]}")
