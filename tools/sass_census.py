"""Per-kernel SASS census of libqcs_b200.so (cuobjdump -sass): the mnemonics
that back DESIGN.md's hardware claims -- TMA bulk copies (UBLKCP) and their
mbarrier transactions (SYNCS), cp.async (LDGSTS), FP64 arithmetic (DMUL, DADD,
and DFMA, which must be absent: -fmad=false keeps the reference's FMA-free
arithmetic), warp shuffles and votes, tensor-core ops (none: the path is
integer / FP64).  usage: python tools/sass_census.py [lib] > profiles/r2_sass_census.txt"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1811_05140_b200/libqcs_b200.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
keys = ["UBLKCP", "SYNCS", "LDGSTS", "DFMA", "DMUL", "DADD", "SHFL", "VOTE", "BAR", "LDS", "STS", "UTC", "HMMA"]
per = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        per[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m:
        op = m.group(1)
        for k in keys:
            if op.startswith(k):
                per[cur][k] += 1


def short(name):
    d = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    return d[:90]


print(f"{'kernel':92s} " + " ".join(f"{k:>7s}" for k in keys))
for f, c in per.items():
    if sum(c.values()) == 0:
        continue
    print(f"{short(f):92s} " + " ".join(f"{c[k]:7d}" for k in keys))
tot = collections.Counter()
for c in per.values():
    tot.update(c)
print(f"{'TOTAL':92s} " + " ".join(f"{tot[k]:7d}" for k in keys))
