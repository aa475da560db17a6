"""Host-side logic: circuit front end, ladder/threshold validation,
GateRecord folding, parity mapping — against the reference where it runs."""
import math

import numpy as np
import pytest

from paper_1811_05140_b200 import circuit as cc
from paper_1811_05140_b200 import metrics as mm
from paper_1811_05140_b200.engine import ErrorBoundLadder, RatioThreshold, StateGeometry


def test_qft_gate_counts():
    # swaps first as 3 CX each; QFT-20 = 240 gates
    assert len(cc.build_qft(10).gates) == 70
    assert len(cc.build_qft(20).gates) == 240
    assert len(cc.build_qft(34).gates) == 646
    assert len(cc.build_qft(37).gates) == 757


def test_grover_gate_form_count_and_equivalence(oracle):
    p = cc.build_grover_gate_form(24, 5, 64)
    assert len(p.gates) == 3224
    # gate form == reference builder up to a global phase
    a = oracle.dense(6, cc.build_grover_gate_form(6, 11, 3).gates, 0)
    b = oracle.dense(6, cc.build_grover(6, 11, 3).gates, 0)
    assert abs(abs(np.vdot(a, b)) - 1.0) < 1e-12


def test_builders_match_reference_text(reference):
    assert cc.print_circuit(cc.build_qft(12)) == reference.builtin(0, 12)
    assert cc.print_circuit(cc.build_grover(9, 17, 5)) == reference.builtin(1, 9, 17, 5)


def test_parse_print_round_trip(reference):
    text = reference.builtin(2, 9, 1234, 120)
    p = cc.parse_circuit(text)
    assert cc.print_circuit(p) == text
    for a, b in zip(p.gates, cc.parse_circuit(cc.print_circuit(p)).gates):
        assert a.desc() == b.desc()


@pytest.mark.parametrize("text,line", [
    ("h 0\n", 1), ("qubits 2\nh 5\n", 2), ("qubits 2\ncx 1 1\n", 2), ("qubits 2\nfoo 1\n", 2),
    ("qubits 2\nu 0 1 0 0 0 0 0 2 0\n", 2), ("qubits 3\nh 0\nqubits 3\n", 3), ("", 1),
])
def test_parse_errors_carry_line(text, line):
    with pytest.raises(cc.ParseError) as e:
        cc.parse_circuit(text)
    assert e.value.line == line


def test_grid_circuit_is_reference_text():
    p = cc.build_grid(6, 6, 20, 1)
    text = cc.print_circuit(p)
    q = cc.parse_circuit(text)
    assert q.n_qubits == 36 and len(q.gates) == len(p.gates)
    kinds = {g.label.split()[0] for g in p.gates}
    assert kinds <= {"cz", "t", "u"}


def test_ladder_validation_and_fingerprint():
    with pytest.raises(ValueError):
        ErrorBoundLadder.make([])
    with pytest.raises(ValueError):
        ErrorBoundLadder.make([0.0, 1e-5, 1e-5])
    with pytest.raises(ValueError):
        ErrorBoundLadder.make([1e-4, 1e-5])
    with pytest.raises(ValueError):
        ErrorBoundLadder.make([-1e-5])
    ErrorBoundLadder.make([0.1])
    d = ErrorBoundLadder.default_ladder()
    assert d.bounds == (0.0, 1e-7, 1e-6, 1e-5, 1e-4, 1e-3)
    assert ErrorBoundLadder.parse("0,1e-7,1e-6").bounds == (0.0, 1e-7, 1e-6)
    with pytest.raises(ValueError):
        ErrorBoundLadder.parse("0,abc")
    with pytest.raises(ValueError):
        RatioThreshold(0.5)
    assert d.fingerprint() != ErrorBoundLadder.parse("0,1e-7,1e-6").fingerprint()
    assert d.fingerprint() == ErrorBoundLadder.default_ladder().fingerprint()


def test_geometry_validation():
    with pytest.raises(ValueError):
        StateGeometry.make(0, 0)
    with pytest.raises(ValueError):
        StateGeometry.make(60, 1)
    with pytest.raises(ValueError):
        StateGeometry.make(4, 5)
    assert StateGeometry.with_default_stride(26).stride_bits == 20


def test_pow2_bound_mapping():
    assert cc.pow2_bound(1e-3, 20) == 2.0 ** -20
    assert cc.pow2_bound(1e-4, 24) == 2.0 ** -26
    assert cc.pow2_bound(1e-3, 34) == 2.0 ** -27
    for eps, n in ((1e-3, 20), (1e-4, 24), (1e-2, 36), (1e-3, 37)):
        d = cc.pow2_bound(eps, n)
        assert d <= eps * 2.0 ** -math.ceil(n / 2) < 2 * d
        assert math.frexp(d)[0] == 0.5


def test_gate_record_fold_matches_reference(reference, oracle):
    text = reference.builtin(0, 9)
    csv_r, _, _ = reference.run(text, 4, 1, [0.0, 1e-7, 1e-6, 1e-5, 1e-4, 1e-3], 8.0)
    prog = cc.parse_circuit(text)
    st = oracle.state(9, 4, 1)
    recs = []
    for i, g in enumerate(prog.gates):
        reps, norm = st.apply_gate(g, [0.0, 1e-7, 1e-6, 1e-5, 1e-4, 1e-3], 8.0)
        recs.append(mm.gate_record(i, g.label, reps, norm)[0])
    assert mm.emit_csv(recs, with_elapsed=False) == mm.strip_elapsed(csv_r)


def test_bench_dense_checker_matches_oracle_dense(oracle):
    """bench.py's GPU dense checker (dense_apply, used for the C2 and C4s
    fidelities) equals the oracle's dense simulator (dense.cpp:30-76) on small
    circuits of every gate kind (run here on CPU tensors)."""
    import numpy as np
    import torch
    import bench
    for prog in (cc.build_grid(3, 3, 6, 5), cc.build_qft(7), cc.build_grover(6, 5, 3),
                 cc.build_grover_gate_form(6, 9, 2)):
        psi = bench.dense_state(prog, len(prog.gates), torch.device("cpu"), basis=3)
        ref = oracle.dense(prog.n_qubits, prog.gates, 3)
        assert np.array_equal(psi.numpy(), ref), prog.name
