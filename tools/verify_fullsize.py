"""Full-size parity run against the unmodified reference (oracle/_ref):
runs a BASELINE configuration completely on the GPU engine and on the
reference's CPU build, compares every GateRecord field except wall time and
the final amplitudes bit for bit, and prints a JSON summary.
Usage: python tools/verify_fullsize.py C2   (or C1)"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import paper_1811_05140_b200 as q  # noqa: E402
from oracle import Reference  # noqa: E402
from paper_1811_05140_b200 import circuit as cc  # noqa: E402
from paper_1811_05140_b200 import metrics as mm  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
if cfg == "C1":
    n, s, basis, eps = 20, 14, 552808, 1e-3
    prog = cc.build_qft(n)
else:
    n, s, basis, eps = 24, 16, 0, 1e-4
    prog = cc.build_grover_gate_form(n, next(cc.splitmix64(7)) & ((1 << n) - 1), 64)
ladder = [cc.pow2_bound(eps, n)]
ref = Reference()
t0 = time.time()
ref_csv, ref_amps, summ = ref.run(cc.print_circuit(prog), s, basis, ladder, 1.0, workers=0)
t_ref = time.time() - t0
t0 = time.time()
st = q.CompressedState.basis_state(q.StateGeometry.make(n, s), basis)
m = q.apply_program_range(st, prog, 0, len(prog.gates), q.ErrorBoundLadder.make(ladder), q.RatioThreshold(1.0))
t_gpu = time.time() - t0
csv = mm.emit_csv(m.records, with_elapsed=False)
amps = st.to_amplitudes()
same_csv = csv == mm.strip_elapsed(ref_csv)
same_amps = amps.tobytes() == ref_amps.tobytes()
print(json.dumps({
    "config": cfg, "n_qubits": n, "stride_bits": s, "gates": len(prog.gates), "delta": ladder[0],
    "gate_records_identical": same_csv, "amplitudes_bitwise_identical": same_amps,
    "compressed_bytes_gpu": st.compressed_bytes(), "compressed_bytes_ref": int(summ["compressed_bytes"]),
    "amps_sha256": hashlib.sha256(amps.tobytes()).hexdigest(),
    "reference_wall_s": t_ref, "reference_threads": ref.max_threads(), "gpu_wall_s": t_gpu,
}))
sys.exit(0 if same_csv and same_amps else 1)
