"""Summarise ncu --set full reports into profiles/ (dev tool).

usage: ncu_summary.py OUT_JSON NAME=REPORT[:INDEX] ...
For each named launch: duration, DRAM bytes, issue/warp activity, executed
warp instructions, registers, grid, FP64 pipe, top stall reasons (pc-sampling
shares), shared-memory bank conflicts."""
import csv
import json
import subprocess
import sys

KEYS = {
    "duration_ns": ("gpu__time_duration.sum", 1.0),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "inst_executed": ("smsp__inst_executed.sum", 1.0),
    "registers": ("launch__registers_per_thread", 1.0),
    "grid": ("launch__grid_size", 1.0),
    "block": ("launch__block_size", 1.0),
    "fp64_pipe_pct": ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 1.0),
    "smem_bank_conflicts_ld": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", 1.0),
}
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e3, "usecond": 1e3, "ns": 1.0, "nsecond": 1.0, "ms": 1e6, "msecond": 1e6}


def rows_of(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def summarise(rep, idx):
    h, units, rows = rows_of(rep)
    r = rows[idx]
    col = {n: i for i, n in enumerate(h)}
    out = {"kernel": r[col["Kernel Name"]][:80]}
    for k, (m, _) in KEYS.items():
        if m in col:
            v = r[col[m]].replace(",", "")
            try:
                out[k] = float(v) * UNIT.get(units[col[m]], 1.0)
            except ValueError:
                out[k] = v
    st = {n[len("smsp__pcsamp_warps_issue_stalled_"):]: float(r[i] or 0) for n, i in col.items()
          if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued")}
    tot = sum(st.values()) or 1.0
    out["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:6]}
    return out


res = {}
for arg in sys.argv[2:]:
    name, spec = arg.split("=", 1)
    rep, _, idx = spec.partition(":")
    res[name] = summarise(rep, int(idx or 0))
with open(sys.argv[1], "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res, indent=1))
