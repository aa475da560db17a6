"""Aggregate ncu source-line instruction counts and stall samples into k_fused phases (dev tool)."""
import csv, subprocess, sys, collections, re
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
fname = None; hdr = None; rows = []
for line in out:
    r = next(csv.reader([line]))
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr and len(r) == len(hdr) and r[2] == "-":
        rows.append((fname, int(r[0]), int(r[4]), int(r[7] or 0)))
# phase boundaries: line numbers of QCS_PHASE markers in qcs_fused.cuh
src = open("paper_1811_05140_b200/csrc/qcs_fused.cuh").read().splitlines()
marks = [(i + 1, int(m.group(1))) for i, l in enumerate(src) for m in [re.search(r"QCS_PHASE\((\d)\);", l)] if m]
def phase(f, ln):
    if f != "qcs_fused.cuh":
        return "helper:" + f
    p = -1
    for l, k in marks:
        if ln > l:
            p = k
    return {-1: "0 input/prologue", 0: "1 rounds", 1: "2 final", 2: "3 sum", 3: "4 tokcount", 4: "5 write", 5: "6 carry", 6: "7 tail"}.get(p, str(p))
agg = collections.defaultdict(lambda: [0, 0])
for f, ln, smp, ie in rows:
    k = phase(f, ln)
    if f == "qcs_fused.cuh" and 95 <= ln <= 320:
        k = "helpers in qcs_fused (scans/sumsq)"
    agg[k][0] += smp; agg[k][1] += ie
ts = sum(v[0] for v in agg.values()); ti = sum(v[1] for v in agg.values())
for k, (smp, ie) in sorted(agg.items()):
    print(f"{k:40s} samples {100*smp/ts:5.1f}%  inst {100*ie/ti:5.1f}%  ({ie/1e6:.1f}M)")
print("total inst", ti)
