"""Parity at BASELINE configuration sizes against the UNMODIFIED reference
(oracle/_ref/libqcsref.so, built from /root/reference by oracle/Makefile and
shipped with the repo snapshot): C1 complete (QFT-20, 2^14-amplitude strides,
240 gates) and a C2 prefix (Grover-24 gate form, H^24 + two iterations, 124
gates, 2^16-amplitude strides).  Every GateRecord field except wall time, the
final amplitudes bit for bit, and the compressed size must be identical."""
import numpy as np
import pytest

from helpers import first_diff
from paper_1811_05140_b200 import circuit as cc
from paper_1811_05140_b200 import metrics as mm

pytestmark = pytest.mark.gpu


def _gpu(prog, s, basis, ladder, stop):
    import paper_1811_05140_b200 as q
    st = q.CompressedState.basis_state(q.StateGeometry.make(prog.n_qubits, s), basis)
    m = q.apply_program_range(st, prog, 0, stop, q.ErrorBoundLadder.make(ladder), q.RatioThreshold(1.0))
    return st, mm.emit_csv(m.records, with_elapsed=False)


@pytest.mark.parametrize("cfg", ["C1", "C2-prefix"])
def test_fullsize_matches_reference(reference, cfg):
    if cfg == "C1":
        n, s, basis, eps = 20, 14, 552808, 1e-3
        prog = cc.build_qft(n)
        stop = len(prog.gates)
    else:
        n, s, basis, eps = 24, 16, 0, 1e-4
        marked = next(cc.splitmix64(7)) & ((1 << n) - 1)
        prog = cc.build_grover_gate_form(n, marked, 64)
        stop = n + 2 * (2 * n + 2)
    ladder = [cc.pow2_bound(eps, n)]
    text = cc.print_circuit(cc.CircuitProgram(n, prog.gates[:stop], prog.name))
    ref_csv, ref_amps, summ = reference.run(text, s, basis, ladder, 1.0, workers=0)
    st, csv = _gpu(prog, s, basis, ladder, stop)
    want = mm.strip_elapsed(ref_csv)
    assert csv == want, first_diff(want, csv)
    got = st.to_amplitudes()
    assert got.tobytes() == ref_amps.tobytes()
    assert st.compressed_bytes() == int(summ["compressed_bytes"])
