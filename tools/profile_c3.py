"""C3-shaped profiling workload (tools/ncu runs): the QFT-n last-stage window
on 2^20-amplitude strides from the closed-form stage state (bench.py's C3
headline at a smaller n: the same per-CTA work).  Prints per-gate device time,
the encoder's phase-cycle counters and the codec counters.
usage: python tools/profile_c3.py [n=28] [gates=4]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1811_05140_b200 as q  # noqa: E402
from paper_1811_05140_b200 import circuit as cc  # noqa: E402
from paper_1811_05140_b200.stage import load_stage_state  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
ng = int(sys.argv[2]) if len(sys.argv) > 2 else 4
s = 20
prog = cc.build_qft(n)
x = next(cc.splitmix64(n)) & ((1 << n) - 1)
g0 = len(prog.gates) - n
delta = cc.pow2_bound(1e-3, n)
lad, th = q.ErrorBoundLadder.make([delta]), q.RatioThreshold(1.0)
st = load_stage_state(q, n, s, x, g0, lad, th, 0)
st.profile(1)
t0 = time.perf_counter()
m = q.apply_program_range(st, prog, g0, g0 + ng, lad, th)
wall = time.perf_counter() - t0
import json  # noqa: E402
with open(os.environ.get("QCS_PROFILE_OUT", "/dev/null"), "w") as f:
    json.dump([{"gate": r.gate_index, "elapsed_ns": r.elapsed_ns, "c_in": r.compressed_in, "c_out": r.bytes_after,
                "amp_updates": r.bytes_before // 16} for r in m.records], f)
for r in m.records:
    print(f"gate {r.gate_index}: {r.elapsed_ns / 1e6:.2f} ms, {r.bytes_before // 16 / (r.elapsed_ns * 1e-9):.3e} amp/s, "
          f"C_in {r.compressed_in} C_out {r.bytes_after}")
print("kernel times", st.kernel_times())
print("counters", st.counters())
print(f"wall {wall:.3f} s")
