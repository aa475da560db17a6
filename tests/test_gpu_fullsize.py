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


def test_grid_c4_shape_matches_reference(reference):
    """C4-shaped (BASELINE configs[3], the seeded random grid family) at a size
    one GPU and the CPU reference both finish: a 4x5 grid (20 qubits), depth
    20 (CZ patterns + sqrt X / sqrt Y / T), 2^14-amplitude strides, bound
    mapped from eps = 1e-2 — every record, the amplitudes and the compressed
    size identical to the unmodified reference."""
    n, s, basis, eps = 20, 14, 0, 1e-2
    prog = cc.build_grid(4, 5, 20, 2024)
    ladder = [cc.pow2_bound(eps, n)]
    ref_csv, ref_amps, summ = reference.run(cc.print_circuit(prog), s, basis, ladder, 1.0, workers=0)
    st, csv = _gpu(prog, s, basis, ladder, len(prog.gates))
    want = mm.strip_elapsed(ref_csv)
    assert csv == want, first_diff(want, csv)
    assert st.to_amplitudes().tobytes() == ref_amps.tobytes()
    assert st.compressed_bytes() == int(summ["compressed_bytes"])


def test_sharded_qft_c5_shape_matches_reference(reference):
    """C5-shaped (BASELINE configs[4]: the top qubits index the GPU, their gates
    exchange compressed strides): QFT-20 with 2^14-amplitude strides on 4
    shards (ranks as threads sharing this GPU; the exchange moves device stride
    images), against the unmodified single-process reference bit for bit."""
    from paper_1811_05140_b200.distributed import GpuBackend, ShardGeometry, run_thread_cluster
    n, s, basis, eps = 20, 14, 552808, 1e-3
    prog = cc.build_qft(n)
    ladder = [cc.pow2_bound(eps, n)]
    ref_csv, ref_amps, _ = reference.run(cc.print_circuit(prog), s, basis, ladder, 1.0, workers=0)
    amp, recs = run_thread_cluster(prog, ShardGeometry(n, s, 2), lambda r: GpuBackend(0), basis, ladder, 1.0)
    want = mm.strip_elapsed(ref_csv)
    got = mm.emit_csv(recs, with_elapsed=False)
    assert got == want, first_diff(want, got)
    assert amp.tobytes() == ref_amps.tobytes()
