"""Symbolize a HIFDE_SAMPLE file against the in-tree library: inclusive
sample counts per function (first N frames of our own code).

usage: python tools/host_sample_report.py FILE [TOP]"""
import collections, os, subprocess, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = os.path.join(root, "paper_1307_2895_b200", "libhifde_gpu.so")
stacks = []
for line in open(sys.argv[1]):
    if line.startswith("#"):
        continue
    fr = [t for t in line.split() if t != "x"]
    if fr:
        stacks.append(fr)
addrs = sorted({a for s in stacks for a in s})
# return addresses: look up the call site (address - 1)
q = [hex(int(a, 16) - 1) for a in addrs]
res = subprocess.run(["addr2line", "-f", "-C", "-e", lib] + q, capture_output=True, text=True).stdout.split("\n")
name = {a: (res[2 * i][:90], res[2 * i + 1].split("/")[-1]) for i, a in enumerate(addrs)}
incl = collections.Counter()
leaf = collections.Counter()
for s in stacks:
    seen = set()
    ours = [name[a] for a in s]
    ours = [o for o in ours if "on_prof" not in o[0]]
    if ours:
        leaf[ours[0]] += 1
    for o in ours:
        if o[0] not in seen:
            seen.add(o[0])
            incl[o[0]] += 1
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print("samples", len(stacks))
print("-- leaf (function, line)")
for k, v in leaf.most_common(top):
    print(f"{v:6d} {k[0]}  {k[1]}")
print("-- inclusive")
for k, v in incl.most_common(top):
    print(f"{v:6d} {k}")
