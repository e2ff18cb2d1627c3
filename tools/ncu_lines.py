"""Aggregate an ncu `--page source --csv --print-source cuda,sass` dump to
CUDA source lines: warp-stall samples and the top stall reasons per line."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = next(i for i, r in enumerate(rows) if 'Warp Stall Sampling (All Samples)' in r)
H = rows[hdr]
ci = H.index('Warp Stall Sampling (All Samples)')
stalls = [(j, h) for j, h in enumerate(H) if h.startswith('stall_') and 'Not Issued' not in h]
agg = collections.defaultdict(lambda: [0, collections.Counter(), ''])
fname = ''
cur = None
for r in rows[hdr + 1:]:
    if len(r) < 3:
        if r and r[0] == 'File Path': fname = r[1].split('/')[-1]
        continue
    if r[0] == 'File Path': fname = r[1].split('/')[-1]; continue
    if r[0] == 'Line No': continue
    if r[0]:
        cur = (fname, int(r[0]) if r[0].isdigit() else r[0]); agg[cur][2] = r[1].strip()[:70]
    if cur is None: continue
    try: s = int(r[ci])
    except ValueError: continue
    agg[cur][0] += s
    for j, h in stalls:
        try: agg[cur][1][h[6:]] += int(r[j])
        except ValueError: pass
tot = sum(v[0] for v in agg.values())
print(f"total samples {tot}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    rs = ', '.join(f"{n} {c}" for n, c in v[1].most_common(3))
    print(f"{v[0]:7d} {100*v[0]/tot:5.1f}%  {k[0]}:{k[1]:<5}  {v[2]:<70} [{rs}]")
