"""Aggregate ncu source-page samples per CUDA source line (dev tool)."""
import csv, subprocess, sys, collections
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
fname = None
rows = []
hdr = None
for line in out:
    r = next(csv.reader([line]))
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[2] == "-":
        rows.append((fname, int(r[0]), r[1].strip(), int(r[4]), int(r[7] or 0)))
tot = sum(x[3] for x in rows)
print("total samples", tot)
for f, ln, src, s, ie in sorted(rows, key=lambda x: -x[3])[:top]:
    print(f"{100*s/tot:5.1f}% {ie:>10d} {f}:{ln:<5d} {src[:90]}")
