"""Diagnostic (not a test): per-CTA phase cycles of the encoder for each gate
of one C2 Grover iteration; dumps the input planes of the slowest stride of
the slowest gate to gpurun_out/slow_stride.npz.  Run on the GPU box with
QCS_CTA_TRACE=1."""
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
it = int(sys.argv[1]) if len(sys.argv) > 1 else 4
q.apply_program_range(st, prog, 0, n + it * 50, lad, th)
L = lib()
L.qcs_debug_cta_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
worst = (0, None, None)
names = ("input", "rounds", "final", "sum", "tokcount", "write", "tail", "x")
for gi in range(n + it * 50, n + it * 50 + 50):
    g = prog.gates[gi]
    before = {}
    m = q.apply_program_range(st, prog, gi, gi + 1, lad, th)
    tr = np.zeros((256, 8), dtype=np.uint64)
    L.qcs_debug_cta_trace(st._h, tr.ctypes.data, 256)
    tot = tr[:, :7].sum(axis=1)
    k = int(tot.argmax())
    print(f"gate {gi} {g.label:10s} {m.records[0].elapsed_ns/1e3:8.1f} us  slowest slot {k} "
          f"{tot[k]/1.965e3:8.1f} us  median {np.median(tot)/1.965e3:7.1f} us  "
          + " ".join(f"{nm}={tr[k, i]/1.965e3:.0f}" for i, nm in enumerate(names[:7])))
    if m.records[0].elapsed_ns > worst[0]:
        worst = (m.records[0].elapsed_ns, gi, k)
print("worst", worst, "marked", marked, "marked stride", marked >> s)
