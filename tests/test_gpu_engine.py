"""Engine parity on the GPU: per-gate records (every GateRecord field except
wall time), final amplitudes, stored blocks, scales and sums must equal the
oracle's / the reference's bit for bit."""
import os

import numpy as np
import pytest

from helpers import first_diff, golden_program, golden_runs, gpu_run, oracle_run, sha
from paper_1811_05140_b200 import circuit as cc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q():
    import paper_1811_05140_b200 as q
    return q


@pytest.mark.parametrize("name", sorted(golden_runs()))
def test_engine_matches_golden(q, name):
    e = golden_runs()[name]
    prog = golden_program(e)
    res, csv = gpu_run(prog, e["stride_bits"], e["basis"], e["ladder"], e["theta"])
    assert csv == e["csv"], first_diff(e["csv"], csv)
    assert sha(res.state.to_amplitudes()) == e["amps_sha256"]
    assert res.state.compressed_bytes() == e["compressed_bytes"]
    assert res.state.norm_sq_tracked() == e["norm_sq_tracked"]


CASES = [
    ("qft", 11, 5, 0, [0.0, 1e-7, 1e-6, 1e-5, 1e-4, 1e-3], 16.0),
    ("qft", 9, 9, 3, [2.0 ** -16], 1.0),
    ("qft", 12, 3, 1, [0.0], 1.0),
    ("qft", 13, 13, 777, [1e-3 * 2 ** -7], 1.0),       # non-power-of-two bound: serial repair path
    ("grover_gates", 11, 6, 0, [2.0 ** -20], 1.0),
    ("grover_ref", 9, 4, 0, [0.0, 1e-6, 1e-4], 32.0),
    ("grid", 9, 4, 0, [2.0 ** -14], 1.0),
]


def _prog(kind, n):
    if kind == "qft":
        return cc.build_qft(n)
    if kind == "grover_gates":
        return cc.build_grover_gate_form(n, 77, 3)
    if kind == "grover_ref":
        return cc.build_grover(n, 33, 6)
    return cc.build_grid(3, 3, 10, 3)


@pytest.mark.parametrize("kind,n,s,basis,ladder,theta", CASES)
def test_engine_matches_oracle(q, oracle, kind, n, s, basis, ladder, theta):
    prog = _prog(kind, n)
    st, want = oracle_run(oracle, prog, s, basis, ladder, theta)
    res, got = gpu_run(prog, s, basis, ladder, theta)
    assert got == want, first_diff(want, got)
    assert res.state.to_amplitudes().tobytes() == st.amplitudes().tobytes()
    for j in range(1 << (n - s)):
        blocks, scale, ssq = res.state.export_blocks(j)
        assert blocks == st.export_blocks(j), f"stride {j}"
        osc, ossq, _, _ = st.stride_info(j)
        assert (scale, ssq) == (osc, ossq), f"stride {j}"


def test_apply_gate_reports_and_norm(q, oracle):
    n, s = 8, 4
    geom = q.StateGeometry.make(n, s)
    st = q.CompressedState.basis_state(geom, 0)
    ost = oracle.state(n, s, 0)
    lad = q.ErrorBoundLadder.lossless_only()
    for k in range(8):
        g = cc.GateOp.single(cc.Unitary2x2.hadamard(), k, "h")
        r = st.apply_gate(g, lad, q.RatioThreshold(1.0))
        orr, on = ost.apply_gate(g, [0.0], 1.0)
        assert [x.as_tuple() for x in r.reports] == orr
        assert r.norm_after == on
    g = cc.GateOp.controlled(cc.Unitary2x2.phase(0.3), 7, 0, "cp 7 0")
    r = st.apply_gate(g, lad, q.RatioThreshold(1.0))
    assert len(r.reports) == geom.n_strides() // 2
    assert all(x.stride_index & (geom.n_strides() >> 1) for x in r.reports)


def test_errors_leave_state_intact(q):
    geom = q.StateGeometry.make(4, 2)
    st = q.CompressedState.basis_state(geom, 3)
    before = st.to_amplitudes().copy()
    with pytest.raises(IndexError):
        st.apply_gate(cc.GateOp.single(cc.Unitary2x2.pauli_x(), 9, "x 9"),
                      q.ErrorBoundLadder.lossless_only())
    with pytest.raises(IndexError):
        st.apply_gate(cc.GateOp.phase_flip(100), q.ErrorBoundLadder.lossless_only())
    assert st.to_amplitudes().tobytes() == before.tobytes()


def test_checkpoint_round_trip_and_resume(q, tmp_path):
    geom = q.StateGeometry.make(10, 6)
    prog = cc.build_qft(10)
    lad = q.ErrorBoundLadder.default_ladder()
    th = q.RatioThreshold(8.0)
    straight = q.run_program(prog, lad, th, geom, q.RunOptions(basis=1))
    half = q.run_program(prog, lad, th, geom, q.RunOptions(basis=1, stop_after=35))
    path = str(tmp_path / "mid.qckp")
    half.state.save(path, lad.fingerprint())
    st, fp = q.CompressedState.load(path, geom)
    assert fp == lad.fingerprint()
    resumed = q.run_program_on(st, prog, lad, th, q.RunOptions(first_gate=35))
    assert resumed.state.to_amplitudes().tobytes() == straight.state.to_amplitudes().tobytes()
    with open(path, "r+b") as f:
        f.seek(4)
        f.write(bytes([99]))
    with pytest.raises(q.CheckpointError) as e:
        q.CompressedState.load(path)
    assert e.value.kind == "version_mismatch"


def test_degenerate_wipe_stays_finite(q):
    geom = q.StateGeometry.make(8, 4)
    r = q.run_program(cc.build_qft(8), q.ErrorBoundLadder.make([0.5]), q.RatioThreshold(1.0),
                      geom, q.RunOptions(basis=1))
    a = r.state.to_amplitudes()
    assert np.all(np.isfinite(a))
    assert float(np.sum(np.abs(a) ** 2)) == 0.0


@pytest.mark.parametrize("max_rounds", [1, 2])
@pytest.mark.parametrize("kind,n,s,basis,ladder,theta", [c for c in CASES if c[0] != "grid"][:5])
def test_engine_neighbour_repair(q, oracle, monkeypatch, max_rounds, kind, n, s, basis, ladder, theta):
    """QCS_MAX_ROUNDS caps the event rounds, so every lane still inconsistent
    after them is repaired from its left neighbour's exit (parallel passes,
    then in order) — still bit-exact."""
    monkeypatch.setenv("QCS_MAX_ROUNDS", str(max_rounds))
    prog = _prog(kind, n)
    st, want = oracle_run(oracle, prog, s, basis, ladder, theta)
    res, got = gpu_run(prog, s, basis, ladder, theta)
    assert got == want, first_diff(want, got)
    assert res.state.to_amplitudes().tobytes() == st.amplitudes().tobytes()


SERIAL_CASES = [
    ("qft", 12, 8, 5, [0.0, 1e-7, 1e-6, 1e-5, 1e-4, 1e-3], 16.0),   # the reference's default ladder
    ("qft", 13, 13, 777, [1e-3 * 2 ** -7], 1.0),
    ("grover_ref", 10, 6, 0, [0.0, 1e-6, 1e-4], 32.0),                # reflect_mean + flips
    ("grid", 9, 6, 0, [0.0, 3e-6, 2.0 ** -14, 1e-3], 8.0),           # mixed decimal / power-of-two levels
]


@pytest.mark.parametrize("mode", ["0", "1", "2"])
@pytest.mark.parametrize("kind,n,s,basis,ladder,theta", SERIAL_CASES)
def test_engine_serial_chain_modes(q, oracle, monkeypatch, mode, kind, n, s, basis, ladder, theta):
    """Non-power-of-two bounds: event rounds only (QCS_SERIAL_CHAIN=0), the
    per-gate policy (1, default) and the serial chain always (2, k_serial_chain
    precomputes every plane's reference chain for all levels) are all
    bit-identical to the oracle."""
    monkeypatch.setenv("QCS_SERIAL_CHAIN", mode)
    prog = _prog(kind, n)
    st, want = oracle_run(oracle, prog, s, basis, ladder, theta)
    res, got = gpu_run(prog, s, basis, ladder, theta)
    assert got == want, first_diff(want, got)
    assert res.state.to_amplitudes().tobytes() == st.amplitudes().tobytes()


IMZ_CASES = [
    ("grover_gates", 12, 9, 0, [2.0 ** -20], 1.0),
    ("grover_gates", 11, 3, 0, [0.0, 2.0 ** -22, 1e-4], 64.0),    # 8-amplitude strides, ladder
    ("grover_ref", 10, 6, 0, [0.0, 1e-6, 1e-4], 32.0),            # reflect_mean gates stay two-plane
    ("real_random", 11, 7, 5, [0.0, 2.0 ** -18], 4.0),
    ("grover_gates", 14, 12, 0, [2.0 ** -22], 1.0),              # pair units through k_decode_gate_re
    ("real_random", 14, 13, 3, [0.0, 2.0 ** -20], 8.0),          # in-stride far (t = 12) and pairs
]


def _real_random(n, seed):
    """Random gates from a real set (H, X, Z, CX, CZ, CP(pi)), seeded."""
    import random
    rng = random.Random(seed)
    p = cc.CircuitProgram(n, [], "real-random")
    U = [cc.Unitary2x2.hadamard(), cc.Unitary2x2.pauli_x(), cc.Unitary2x2.pauli_z()]
    for _ in range(120):
        t = rng.randrange(n)
        if rng.random() < 0.4:
            c = rng.randrange(n - 1)
            c = c + 1 if c >= t else c
            p.gates.append(cc.GateOp.controlled(U[rng.randrange(1, 3)], c, t, f"c {c} {t}"))
        else:
            p.gates.append(cc.GateOp.single(U[rng.randrange(3)], t, f"u {t}"))
    return p


@pytest.mark.parametrize("imz", ["0", "1"])
@pytest.mark.parametrize("big", [False, True])
@pytest.mark.parametrize("kind,n,s,basis,ladder,theta", IMZ_CASES)
def test_engine_zero_imaginary_plane_mode(q, oracle, monkeypatch, imz, big, kind, n, s, basis, ladder, theta):
    """Real gates on strides whose im planes are zero: the CTA encodes the re
    plane with all its lanes and writes the im plane's one-token encoding
    (QCS_IMZ=1, default) — bit-identical to the two-plane path and the oracle,
    in both layouts."""
    monkeypatch.setenv("QCS_IMZ", imz)
    if big:
        monkeypatch.setenv("QCS_FORCE_BIG", "1")
        monkeypatch.setenv("QCS_WAVE_SLOTS", "3")
    prog = _real_random(n, 9) if kind == "real_random" else _prog(kind, n)
    st, want = oracle_run(oracle, prog, s, basis, ladder, theta)
    res, got = gpu_run(prog, s, basis, ladder, theta)
    assert got == want, first_diff(want, got)
    assert res.state.to_amplitudes().tobytes() == st.amplitudes().tobytes()
    for j in range(1 << (n - s)):
        assert res.state.export_blocks(j)[0] == st.export_blocks(j)
