"""Aggregate an ncu source page of k_stream (csrc/qcs_stream.cuh) into the kernel's regions
(dev tool): share of warp-stall samples and of executed warp instructions per region, and
warp instructions per walk step (one complex element per lane).
usage: ncu_regions.py REPORT [STEPS]   (STEPS: complex elements of the launch / 32)"""
import collections
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
steps = float(sys.argv[2]) if len(sys.argv) > 2 else None
SRC = "paper_1811_05140_b200/csrc/qcs_stream.cuh"
MARKS = [
    (r"^struct TokReader", "token reader (slow paths)"),
    (r"^struct StreamCommit", "encoder-side commit"),
    (r"^struct StreamPlaneOut", "prologue / per-step uniform tests"),
    (r"// A\. stage", "A input staging (TMA)"),
    (r"auto walk = ", "walk setup"),
    (r"auto next2 = ", "token reader (joint fast path)"),
    (r"auto gate_snap = ", "scale + gate + snap"),
    (r"auto slow_step = ", "reference step (unproven)"),
    (r"auto emit_any = ", "token emission (general)"),
    (r"auto sums = ", "sum-of-squares units"),
    (r"// element 0:", "element 0"),
    (r"for \(int k = 1; k < SUB", "quantize"),
    (r"two code tokens, nothing else", "token emission (fast path)"),
    (r"Mprev\[0\] = M0;", "walk tail"),
    (r"// B\. main pass", "B main pass call"),
    (r"// C\. first elements", "C first elements, runs, lead tokens"),
    (r"// exclusive sum-scan of the lanes' bytes", "C byte scan + side index"),
    (r"// D\. stored sum", "D stored sum (events)"),
    (r"// E\. token bytes out", "E packed copy-out"),
    (r"// ladder early exit", "tail"),
]
lines = open(SRC).read().splitlines()
starts = []
for pat, name in MARKS:
    for i, l in enumerate(lines):
        if re.search(pat, l):
            starts.append((i + 1, name))
            break
starts.sort()
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
fname = hdr = None
agg = collections.defaultdict(lambda: [0, 0])
for line in out:
    r = next(csv.reader([line]))
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[2] == "-":
        a = agg[(fname, int(r[0]))]
        a[0] += int(r[4])
        a[1] += int(r[7] or 0)
res = collections.defaultdict(lambda: [0, 0])
for (f, ln), (s, i) in agg.items():
    name = "other: " + f
    if f == "qcs_stream.cuh":
        name = "head"
        for st, nm in starts:
            if ln >= st:
                name = nm
    res[name][0] += s
    res[name][1] += i
tot = sum(v[0] for v in res.values())
toti = sum(v[1] for v in res.values())
print(f"{rep}: {tot} samples, {toti / 1e6:.0f}M warp instructions" + (f", {toti / steps:.0f} per step" if steps else ""))
for k, (s, i) in sorted(res.items(), key=lambda x: -x[1][0]):
    print(f"  {k:42s} stall samples {100 * s / tot:5.1f}%   inst {100 * i / toti:5.1f}%" +
          (f"   {i / steps:6.1f} per step" if steps else ""))
