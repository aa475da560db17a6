"""Write profiles/traffic_k_fused_c3.json from an ncu --set full report of one
k_fused launch of the C3 bench: DRAM bytes read + written per launch (the
bench's roofline.traffic) and the launch's algorithmic C_in + C_out when given.
usage: traffic_from_ncu.py REPORT [out.json]"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else "profiles/traffic_k_fused_c3.json"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
vals = rows[2:]
res = []
for v in vals:
    d = dict(zip(h, v))
    u = dict(zip(h, units))

    def num(k):
        x = float(d[k].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u[k], 1)
        return x * scale

    res.append({"kernel": d.get("Kernel Name", ""), "dram_read": num("dram__bytes_read.sum"),
                "dram_write": num("dram__bytes_write.sum"),
                "duration_ns": num("gpu__time_duration.sum") * (1e3 if u["gpu__time_duration.sum"] == "usecond" else
                                                                1e6 if u["gpu__time_duration.sum"] == "msecond" else 1),
                "grid": d.get("launch__grid_size"), "regs": d.get("launch__registers_per_thread"),
                "warps_active_pct": d.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
                "issue_active_pct": d.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                "warp_inst": d.get("smsp__inst_executed.sum")})
t = sum(r["dram_read"] + r["dram_write"] for r in res) / max(1, len(res))
doc = {"traffic_bytes": t, "launches": res, "source": rep}
if len(sys.argv) > 3:  # records json of the same command (tools/profile_c3.py QCS_PROFILE_OUT): C_in + C_out
    recs = json.load(open(sys.argv[3]))
    alg = recs[int(sys.argv[4]) if len(sys.argv) > 4 else 1]
    doc["algorithmic_bytes"] = alg["c_in"] + alg["c_out"]
    doc["traffic_per_algorithmic_byte"] = t / doc["algorithmic_bytes"]
json.dump(doc, open(out, "w"), indent=1)
print(json.dumps({"traffic_bytes": t, "n": len(res)}))
