"""Diagnostic: dump the encoder input planes (split path) of given slots after
gate index G of the C2 circuit to gpurun_out/x_dump.npz.  QCS_SPLIT_LOCAL=1."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1811_05140_b200 as q  # noqa: E402
from paper_1811_05140_b200 import circuit as cc  # noqa: E402
from paper_1811_05140_b200.engine import lib  # noqa: E402

n, s = 24, 16
marked = next(cc.splitmix64(7)) & ((1 << n) - 1)
prog = cc.build_grover_gate_form(n, marked, 64)
delta = cc.pow2_bound(1e-4, n)
lad, th = q.ErrorBoundLadder.make([delta]), q.RatioThreshold(1.0)
st = q.CompressedState.basis_state(q.StateGeometry.make(n, s), 0)
G = int(sys.argv[1])
slots = [int(x) for x in sys.argv[2:]]
q.apply_program_range(st, prog, 0, G + 1, lad, th)
L = lib()
L.qcs_debug_read_x.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
out = {}
for sl in slots:
    x = np.empty(2 << s)
    assert L.qcs_debug_read_x(st._h, sl, x.ctypes.data) == 0
    out[f"s{sl}"] = x
    out[f"blk{sl}"] = np.frombuffer(st.export_blocks(sl)[0], dtype=np.uint8)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
np.savez(os.path.join(ROOT, "gpurun_out", "x_dump.npz"), delta=delta, **out)
print("saved", slots, prog.gates[G].label)
