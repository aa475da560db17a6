"""Per-gate report of the streaming kernel (dev tool): slots it encoded, slots it left to the
legacy encoder and why.  usage: python tools/debug/dbg_stream.py"""
import os, sys
sys.path.insert(0, os.getcwd())
os.environ["QCS_STREAM"] = "2"
import paper_1811_05140_b200 as q
from paper_1811_05140_b200 import circuit as cc
n, s = 13, 13
prog = cc.build_qft(n)
lad, th = q.ErrorBoundLadder.make([cc.pow2_bound(1e-3, n)]), q.RatioThreshold(1.0)
st = q.CompressedState.basis_state(q.StateGeometry.make(n, s), 0x5a5) if hasattr(q, "CompressedState") else None
print(type(st))
prev = (0, 0)
pw = None
for i, g in enumerate(prog.gates):
    q.apply_program_range(st, prog, i, i + 1, lad, th)
    c = st.counters()
    cur = (c["stream_slots"], c["stream_left_slots"])
    w = c["stream_left_why"]
    dw = {k: w[k] - (pw[k] if pw else 0) for k in w}
    pw = w
    print(i, g.label, "streamed", cur[0] - prev[0], "left", cur[1] - prev[1], {k: v for k, v in dw.items() if v})
    prev = cur
