"""Symbolize a HIFDE_SAMPLE host profile: self time by innermost library
frame (samples whose leaf is outside the library are attributed to the
innermost library frame and tagged [ext]) and inclusive time by function."""
import collections, subprocess, sys

path = sys.argv[1]
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_1307_2895_b200/libhifde_gpu.so"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
rows = [l.split()[2:] for l in open(path) if not l.startswith("#")]  # drop handler + signal frame
addrs = sorted({a for r in rows for a in r if a != "x"})
sym = {}
if addrs:
    out = subprocess.run(["addr2line", "-f", "-C", "-i", "-e", lib] + [hex(int(a, 16) - 1) for a in addrs],
                         capture_output=True, text=True).stdout.split("\n")
    # with -i, inlined frames add extra pairs; take the first (innermost) function per address
    # by re-running without -i for a clean 1:1 mapping
    out = subprocess.run(["addr2line", "-f", "-C", "-e", lib] + [hex(int(a, 16) - 1) for a in addrs],
                         capture_output=True, text=True).stdout.split("\n")
    for i, a in enumerate(addrs):
        fn = out[2 * i] if 2 * i < len(out) else "?"
        fn = fn.replace("(anonymous namespace)::", "").split("(")[0][:90]
        loc = out[2 * i + 1].split("/")[-1] if 2 * i + 1 < len(out) else ""
        sym[a] = (fn, loc)
self_c, incl = collections.Counter(), collections.Counter()
for r in rows:
    inner = next((a for a in r if a != "x"), None)
    if inner is None:
        self_c["[outside library]"] += 1
        continue
    tag = "" if r[0] != "x" else " [ext]"
    self_c[sym[inner][0] + tag] += 1
    seen = set()
    for a in r:
        if a == "x":
            continue
        fn = sym[a][0]
        if fn not in seen:
            incl[fn] += 1
            seen.add(fn)
n = len(rows)
print(f"{n} samples")
print("--- self (innermost library frame)")
for k, v in self_c.most_common(top):
    print(f"{v:6d} {100*v/n:5.1f}%  {k}")
print("--- inclusive")
for k, v in incl.most_common(top):
    print(f"{v:6d} {100*v/n:5.1f}%  {k}")
