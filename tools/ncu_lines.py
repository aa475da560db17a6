"""Aggregate ncu source-page samples per CUDA source line, summed over every
profiled launch in the report (dev tool).  usage: ncu_lines.py REP [TOP]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
fname = None
hdr = None
agg = collections.defaultdict(lambda: [0, 0, ""])
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
        a[2] = r[1].strip()
tot = sum(v[0] for v in agg.values())
toti = sum(v[1] for v in agg.values())
print("total samples", tot, "inst", toti)
for (f, ln), (s, ie, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100*s/tot:5.1f}% {100*ie/toti:5.1f}%i {f}:{ln:<5d} {src[:90]}")
