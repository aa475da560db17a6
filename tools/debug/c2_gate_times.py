"""Per-gate device time of one Grover iteration of C2 (dev tool)."""
import os, sys
sys.path.insert(0, os.getcwd())
import paper_1811_05140_b200 as q
from paper_1811_05140_b200 import circuit as cc
n, s = 24, 16
prog = cc.build_grover_gate_form(n, next(cc.splitmix64(7)) & ((1 << n) - 1), 6)
lad, th = q.ErrorBoundLadder.make([cc.pow2_bound(1e-4, n)]), q.RatioThreshold(1.0)
st = q.CompressedState.basis_state(q.StateGeometry.make(n, s), 0)
m = q.apply_program_range(st, prog, 0, len(prog.gates), lad, th)
recs = m.records
g0 = n + 4 * 50
for r in recs[g0:g0 + 50]:
    print(r.gate_index, prog.gates[r.gate_index].label, f"{r.elapsed_ns/1e3:.0f} us")
print("counters", st.counters())
