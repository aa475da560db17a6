"""Aggregate an ncu source page of k_fused into encoder phases (dev tool).

usage: ncu_phases.py REPORT [GIT_REV]
Lines of the kernel body are attributed by the QCS_PHASE markers, helper
functions by their own ranges, for the qcs_fused.cuh of GIT_REV (the source
the report was captured from; default the working tree).  Prints, per kernel
variant and phase, the share of warp-stall samples, of not-issued samples
and of executed warp instructions."""
import collections
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
rev = sys.argv[2] if len(sys.argv) > 2 else None
CSRC = "paper_1811_05140_b200/csrc/"


def source(name):
    p = CSRC + name
    return (subprocess.run(["git", "show", f"{rev}:{p}"], capture_output=True, text=True).stdout
            if rev else open(p).read()).splitlines()


src = source("qcs_fused.cuh")
kstart = next(i + 1 for i, l in enumerate(src) if "void fused_body(" in l or "k_fused(FusedArgs a)" in l)
marks = [(i + 1, int(m.group(1))) for i, l in enumerate(src) for m in [re.search(r"QCS_PHASE\((\d)\);", l)] if m]
names = {-1: "0 input", 0: "1 rounds", 1: "2 final", 2: "3 sum", 3: "4 tokcount", 4: "5 write", 5: "6 carry", 6: "7 tail"}
funcs = [(i + 1, m.group(1)) for i, l in enumerate(src)
         for m in [re.match(r"__device__ __forceinline__ \S+&? (\w+)\(", l)] if m]


def fn_ranges(lines):
    return [(i + 1, m.group(1)) for i, l in enumerate(lines)
            for m in [re.match(r"(?:template.*)?__device__ __forceinline__ [\w:<>]+&? (\w+)\(", l)] if m]


helper_funcs = {f: fn_ranges(source(f)) for f in ("qcs_codec.cuh", "qcs_device.cuh")}


def phase(f, ln):
    if f in helper_funcs:
        name = "?"
        for l0, n in helper_funcs[f]:
            if l0 <= ln:
                name = n
        return f"{f}:{name}"
    if f != "qcs_fused.cuh":
        return "helper " + f
    if ln < kstart:
        name = "?"
        for l0, n in funcs:
            if l0 <= ln:
                name = n
        return "fn " + name
    p = -1
    for l, k in marks:
        if ln > l:
            p = k
    return names.get(p, str(p))


out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
fname = func = hdr = None
agg = collections.defaultdict(lambda: collections.defaultdict(lambda: [0, 0, 0]))
for line in out:
    r = next(csv.reader([line]))
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        func = ("LOCAL" if r[1].endswith("(int)1>(qcs::FusedArgs)") else
                "RAW" if "k_fused" in r[1] else r[1].split("(")[0].replace("<unnamed>::", ""))
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[2] == "-":
        a = agg[func][phase(fname, int(r[0]))]
        a[0] += int(r[4])
        a[1] += int(r[5])
        a[2] += int(r[7] or 0)
for func, ph in agg.items():
    ts = sum(v[0] for v in ph.values()) or 1
    tn = sum(v[1] for v in ph.values()) or 1
    ti = sum(v[2] for v in ph.values()) or 1
    print(f"== {func}: {ts} samples, {ti / 1e6:.0f}M warp instructions")
    for k, (s_, n_, i_) in sorted(ph.items(), key=lambda kv: -kv[1][0]):
        print(f"  {k:28s} stall {100 * s_ / ts:5.1f}%  not-issued {100 * n_ / tn:5.1f}%  inst {100 * i_ / ti:5.1f}%")
