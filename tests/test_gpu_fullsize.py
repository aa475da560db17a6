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


def _vs_reference(reference, prog, s, basis, ladder, theta, stop=None):
    import paper_1811_05140_b200 as q
    n = prog.n_qubits
    stop = len(prog.gates) if stop is None else stop
    text = cc.print_circuit(cc.CircuitProgram(n, prog.gates[:stop], prog.name))
    ref_csv, ref_amps, summ = reference.run(text, s, basis, ladder, theta, workers=0)
    st = q.CompressedState.basis_state(q.StateGeometry.make(n, s), basis)
    m = q.apply_program_range(st, prog, 0, stop, q.ErrorBoundLadder.make(ladder), q.RatioThreshold(theta))
    got = mm.emit_csv(m.records, with_elapsed=False)
    want = mm.strip_elapsed(ref_csv)
    assert got == want, first_diff(want, got)
    assert st.to_amplitudes().tobytes() == ref_amps.tobytes()
    assert st.compressed_bytes() == int(summ["compressed_bytes"])


# SURVEY.md §8d's own (non-power-of-two) delta mapping eps*2^-ceil(n/2) and the
# reference's defaults (aalc.cpp:74-77 default ladder, tools/qcsim.cpp:35-36
# theta = 16), at full configuration sizes: these bounds take the serial-chain
# / event-round repair paths, which must stay bit-exact too.
def test_c1_survey_delta_matches_reference(reference):
    """C1 complete (QFT-20, 2^14-amp strides, 240 gates) at delta = 9.765625e-7."""
    n = 20
    assert cc.survey_bound(1e-3, n) == 9.765625e-7
    _vs_reference(reference, cc.build_qft(n), 14, 552808, [cc.survey_bound(1e-3, n)], 1.0)


def test_c2_prefix_survey_delta_matches_reference(reference):
    """C2 prefix (Grover-24 gate form, H^24 + two iterations, 124 gates,
    2^16-amp strides) at delta = 2.44140625e-8."""
    n = 24
    assert cc.survey_bound(1e-4, n) == 2.44140625e-8
    marked = next(cc.splitmix64(7)) & ((1 << n) - 1)
    prog = cc.build_grover_gate_form(n, marked, 64)
    _vs_reference(reference, prog, 16, 0, [cc.survey_bound(1e-4, n)], 1.0, stop=n + 2 * (2 * n + 2))


def test_qft20_default_ladder_theta16_matches_reference(reference):
    """bench_compare's configuration (bench/bench_compare.cpp: QFT-20, s = 14,
    basis 1) with the reference's default ladder 0, 1e-7 ... 1e-3 and theta 16:
    the multi-level ladder with escalation, every level a decimal bound."""
    _vs_reference(reference, cc.build_qft(20), 14, 1, [0.0, 1e-7, 1e-6, 1e-5, 1e-4, 1e-3], 16.0)


def test_grid_c4_shape_survey_delta_matches_reference(reference):
    """The 4x5 grid of test_grid_c4_shape_matches_reference at SURVEY's decimal
    mapping of eps = 1e-2 (delta = 1e-2 * 2^-10)."""
    n = 20
    _vs_reference(reference, cc.build_grid(4, 5, 20, 2024), 14, 0, [cc.survey_bound(1e-2, n)], 1.0)
