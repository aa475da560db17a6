"""The C++ sharded driver (qcs_cluster_*, csrc/qcs_cluster.cuh) with the
loopback exchange backend: 2 and 4 ranks sharing this GPU, against the
UNMODIFIED single-process reference bit for bit (every GateRecord field
except wall time, the logical amplitudes): QFT (rank-qubit targets ->
stride-image exchanges), the Grover reference form (reflect_mean's mean and
flips folded across shards) and the seeded grid (CZ on rank qubits)."""
import pytest

from helpers import first_diff
from paper_1811_05140_b200 import circuit as cc
from paper_1811_05140_b200 import metrics as mm

pytestmark = pytest.mark.gpu


CASES = [
    ("qft", 12, 6, 1, 9, [2.0 ** -18], 1.0),
    ("qft", 12, 6, 2, 9, [2.0 ** -18], 1.0),
    ("qft", 13, 5, 2, 77, [0.0, 1e-7, 1e-6, 1e-5, 1e-4, 1e-3], 16.0),
    ("grover_ref", 11, 5, 2, 0, [0.0, 1e-6, 1e-4], 32.0),
    ("grover_gates", 12, 6, 1, 0, [2.0 ** -20], 1.0),
    ("grid", 12, 6, 2, 0, [2.0 ** -14], 1.0),
]


def _prog(kind, n):
    if kind == "qft":
        return cc.build_qft(n)
    if kind == "grover_ref":
        return cc.build_grover(n, 33, 6)
    if kind == "grover_gates":
        return cc.build_grover_gate_form(n, 1234, 2)
    return cc.build_grid(3, 4, 12, 5)


@pytest.mark.parametrize("kind,n,s,g,basis,ladder,theta", CASES)
def test_cluster_loopback_matches_reference(reference, kind, n, s, g, basis, ladder, theta):
    import paper_1811_05140_b200 as q
    prog = _prog(kind, n)
    ref_csv, ref_amps, _ = reference.run(cc.print_circuit(prog), s, basis, ladder, theta, workers=0)
    cl = q.Cluster(q.StateGeometry.make(n, s), g, basis, [0] * (1 << g), "loopback")
    cl.set_schedule(prog)
    m = cl.apply_program_range(prog, 0, len(prog.gates), q.ErrorBoundLadder.make(ladder), q.RatioThreshold(theta))
    got = mm.emit_csv(m.records, with_elapsed=False)
    want = mm.strip_elapsed(ref_csv)
    assert got == want, first_diff(want, got)
    assert cl.to_amplitudes().tobytes() == ref_amps.tobytes()
    if kind == "qft":
        assert cl.stats()["exchanges"] > 0


def test_cluster_wave_layout_shards(reference, monkeypatch):
    """Shards in the wave layout (forced, tiny arenas): suspensions and
    compactions inside the sharded run stay bit-identical."""
    import paper_1811_05140_b200 as q
    monkeypatch.setenv("QCS_FORCE_BIG", "1")
    monkeypatch.setenv("QCS_WAVE_SLOTS", "2")
    monkeypatch.setenv("QCS_ARENA_BYTES", str(3 * (16 << 10)))
    n, s, g = 12, 5, 1
    prog = cc.build_qft(n)
    ladder = [0.0]
    ref_csv, ref_amps, _ = reference.run(cc.print_circuit(prog), s, 3, ladder, 1.0, workers=0)
    cl = q.Cluster(q.StateGeometry.make(n, s), g, 3, [0, 0], "loopback")
    m = cl.apply_program_range(prog, 0, len(prog.gates), q.ErrorBoundLadder.make(ladder), q.RatioThreshold(1.0))
    got = mm.emit_csv(m.records, with_elapsed=False)
    assert got == mm.strip_elapsed(ref_csv), first_diff(mm.strip_elapsed(ref_csv), got)
    assert cl.to_amplitudes().tobytes() == ref_amps.tobytes()


def test_cluster_nccl_backend_one_rank(reference):
    """The NCCL backend (libnccl.so.2 loaded at run time, ncclCommInitAll over
    the cluster's devices) on the one GPU this box has: no rank qubits, so no
    exchange, but the communicator and the device-side folds run; results equal
    the reference."""
    import paper_1811_05140_b200 as q
    prog = cc.build_qft(10)
    ladder = [2.0 ** -16]
    ref_csv, ref_amps, _ = reference.run(cc.print_circuit(prog), 6, 5, ladder, 1.0, workers=0)
    cl = q.Cluster(q.StateGeometry.make(10, 6), 0, 5, [0], "nccl")
    m = cl.apply_program_range(prog, 0, len(prog.gates), q.ErrorBoundLadder.make(ladder), q.RatioThreshold(1.0))
    assert mm.emit_csv(m.records, with_elapsed=False) == mm.strip_elapsed(ref_csv)
    assert cl.to_amplitudes().tobytes() == ref_amps.tobytes()


def test_cluster_nccl_rejects_shared_device():
    import paper_1811_05140_b200 as q
    with pytest.raises(ValueError):
        q.Cluster(q.StateGeometry.make(10, 6), 1, 0, [0, 0], "nccl")


def test_cluster_control_on_the_only_local_stride_bit(reference):
    """n - g = s + 1: the control holding the only local stride bit is evicted
    to a rank bit for a rank-qubit target (then the rank-level skip applies)."""
    import paper_1811_05140_b200 as q
    n, s, g = 6, 4, 1
    U = cc.Unitary2x2
    prog = cc.CircuitProgram(n, [cc.GateOp.single(U.hadamard(), k, f"h {k}") for k in range(n)] +
                             [cc.GateOp.controlled(U.pauli_x(), 4, 5, "cx 4 5"),
                              cc.GateOp.controlled_phase(0.7, 5, 4, "cp 5 4"),
                              cc.GateOp.single(U.pauli_y(), 5, "y 5"),
                              cc.GateOp.controlled(U.pauli_x(), 4, 5, "cx 4 5")], "ctl-local")
    ladder = [2.0 ** -14]
    ref_csv, ref_amps, _ = reference.run(cc.print_circuit(prog), s, 3, ladder, 1.0, workers=0)
    cl = q.Cluster(q.StateGeometry.make(n, s), g, 3, [0, 0], "loopback")
    m = cl.apply_program_range(prog, 0, len(prog.gates), q.ErrorBoundLadder.make(ladder), q.RatioThreshold(1.0))
    assert mm.emit_csv(m.records, with_elapsed=False) == mm.strip_elapsed(ref_csv)
    assert cl.to_amplitudes().tobytes() == ref_amps.tobytes()
