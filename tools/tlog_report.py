"""Analyse HIFDE_SKEL_TLOG dumps of the exact-order skeleton kernel:
per-group phase durations and the critical chain (flag latency vs work)."""
import sys, glob, numpy as np
for fn in sorted(glob.glob(sys.argv[1] + "/tlog_*.bin")):
    raw = open(fn, "rb").read()
    nt, npred, grid = np.frombuffer(raw[:24], dtype=np.int64)
    o = 24
    t = np.frombuffer(raw[o:o + nt * 128], dtype=np.uint64).reshape(nt, 16).astype(np.int64); o += nt * 128
    cyc = t[:, 8:12].astype(float); cyc2 = t[:, 12:15].astype(float); t = t[:, :8]
    pp = np.frombuffer(raw[o:o + (nt + 1) * 8], dtype=np.int64); o += (nt + 1) * 8
    pr = np.frombuffer(raw[o:o + npred * 4], dtype=np.int32)
    t0 = t[:, 0].min()
    t = (t - t0) / 1e3  # us
    zero = t[:, 4] - t[:, 1]; norms = t[:, 5] - t[:, 4]; loop = t[:, 6] - t[:, 5]; post = t[:, 2] - t[:, 6]
    asm = t[:, 1] - t[:, 0]
    work = t[:, 2] - t[:, 1]
    tail = t[:, 3] - t[:, 2]
    # latency from the last predecessor's publish to this group's wait end
    lat = []
    crit = np.zeros(nt)
    for j in range(nt):
        ps = pr[pp[j]:pp[j + 1]]
        if len(ps):
            last = t[ps, 2].max()
            lat.append(t[j, 1] - last)
    lat = np.array(lat) if lat else np.zeros(1)
    # walk back the critical chain from the last publish
    j = int(np.argmax(t[:, 2])); chain = [j]
    while pp[j + 1] > pp[j]:
        ps = pr[pp[j]:pp[j + 1]]
        j = int(ps[np.argmax(t[ps, 2])]); chain.append(j)
    chain = chain[::-1]
    cw = sum(work[c] for c in chain)
    print(f"{fn.split('/')[-1]}: groups {nt} grid {grid} span {t[:, 3].max():.1f} us | "
          f"assemble med {np.median(asm):.1f} | cpqr (wait->publish) med {np.median(work):.1f} max {work.max():.1f} | "
          f"tail med {np.median(tail):.1f} | flag latency med {np.median(lat):.1f} | chain {len(chain)} groups, "
          f"work on chain {cw:.1f} us, chain end {t[chain[-1], 2]:.1f} us, first wait end {t[chain[0], 1]:.1f}\n"
          f"    cpqr cycles (warp 0, summed over steps) median: pivot {np.median(cyc[:,0]):.0f} householder {np.median(cyc[:,1]):.0f} update {np.median(cyc[:,2]):.0f} barrier {np.median(cyc[:,3]):.0f} | update: dot {np.median(cyc2[:,0]):.0f} upd {np.median(cyc2[:,1]):.0f} acc-red {np.median(cyc2[:,2]):.0f}\n"
          f"    after wait: zero rows {np.median(zero):.1f} | (tsqr+)norms {np.median(norms):.1f} | cpqr loop {np.median(loop):.1f} | to publish {np.median(post):.1f}")
