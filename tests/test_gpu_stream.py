"""The streaming fused kernel (csrc/qcs_stream.cuh) against the oracle.

QCS_STREAM=2 sends every element-wise gate (diagonal single / controlled gates
on any target, phase flips, reflect_mean) at a power-of-two lossy level
through k_stream whatever the slot count; every GateRecord field, the
amplitudes and every stored block must equal the oracle's bit for bit, the
kernel must have encoded slots itself (counter [18]), and states it cannot
prove (escapes: a bound far below the amplitudes) must come out of the legacy
encoder unchanged (counter [17])."""
import math
import random

import pytest

from helpers import first_diff, gpu_run, oracle_run
from paper_1811_05140_b200 import circuit as cc

pytestmark = pytest.mark.gpu


def _check(oracle, prog, s, basis, ladder, theta):
    n = prog.n_qubits
    st, want = oracle_run(oracle, prog, s, basis, ladder, theta)
    res, got = gpu_run(prog, s, basis, ladder, theta)
    assert got == want, first_diff(want, got)
    assert res.state.to_amplitudes().tobytes() == st.amplitudes().tobytes()
    for j in range(1 << (n - s)):
        assert res.state.export_blocks(j)[0] == st.export_blocks(j), j
    return res.state.counters()


def _diag_program(rng, n, gates):
    U = cc.Unitary2x2
    diag = [U.t_gate(), U.s_gate(), U.pauli_z(), U.phase(0.37), U.phase(-1.1)]
    mix = [U.hadamard(), U.sqrt_x(), U.pauli_y()]
    p = cc.CircuitProgram(n, [], "stream")
    for t in range(n):  # a dense complex state first
        p.gates.append(cc.GateOp.single(U.hadamard(), t, f"h{t}"))
        p.gates.append(cc.GateOp.single(U.phase(0.1 + 0.3 * t), t, f"p{t}"))
    for _ in range(gates):
        r = rng.random()
        t = rng.randrange(n)
        if r < 0.08:
            p.gates.append(cc.GateOp.phase_flip(rng.randrange(1 << n)))
        elif r < 0.12:
            p.gates.append(cc.GateOp.reflect_mean())
        elif r < 0.2:
            p.gates.append(cc.GateOp.single(rng.choice(mix), t, f"m{t}"))
        elif r < 0.6 and n > 1:
            c = rng.randrange(n - 1)
            c = c + 1 if c >= t else c
            p.gates.append(cc.GateOp.controlled(rng.choice(diag), c, t, f"c{c}t{t}"))
        else:
            p.gates.append(cc.GateOp.single(rng.choice(diag), t, f"d{t}"))
    return p


@pytest.mark.parametrize("lanes", ["128", "256", "512"])
@pytest.mark.parametrize("n,s", [(12, 12), (13, 8), (14, 5), (11, 6)])
def test_stream_diagonal_programs(oracle, monkeypatch, lanes, n, s):
    monkeypatch.setenv("QCS_STREAM", "2")
    monkeypatch.setenv("QCS_STREAM_LANES", lanes)
    rng = random.Random(7 * n + s)
    prog = _diag_program(rng, n, 40)
    delta = 2.0 ** math.floor(math.log2(2.0 ** -(n / 2) * 1e-3))
    ctr = _check(oracle, prog, s, rng.randrange(1 << n), [delta], 1.0)
    assert ctr["stream_slots"] > 0


@pytest.mark.parametrize("n,s", [(12, 7), (13, 13)])
def test_stream_qft(oracle, monkeypatch, n, s):
    # (a single stride whose first 512 amplitudes stay zero is left to the legacy
    # encoder's sum-of-squares cases: attempted, exact, not necessarily streamed)
    monkeypatch.setenv("QCS_STREAM", "2")
    ctr = _check(oracle, cc.build_qft(n), s, 0x5a5 & ((1 << n) - 1), [cc.pow2_bound(1e-3, n)], 1.0)
    assert ctr["stream_slots"] + ctr["stream_left_slots"] > 0
    if s < n:
        assert ctr["stream_slots"] > 0


def test_stream_ladder_levels(oracle, monkeypatch):
    # a ladder of power-of-two levels with a threshold: early exits, several levels per gate
    monkeypatch.setenv("QCS_STREAM", "2")
    n, s = 12, 8
    amp = 2.0 ** -(n / 2)
    lad = [2.0 ** math.floor(math.log2(amp * 1e-6)), 2.0 ** math.floor(math.log2(amp * 1e-4)),
           2.0 ** math.floor(math.log2(amp * 1e-2))]
    ctr = _check(oracle, _diag_program(random.Random(3), n, 30), s, 77, lad, 6.0)
    assert ctr["stream_slots"] > 0


def test_stream_leaves_escapes_to_the_legacy_encoder(oracle, monkeypatch):
    # a bound 2^-45 under amplitudes of 2^-6: every code overflows 2^15 bins, the reference
    # escapes, the streaming kernel must give those slots up
    monkeypatch.setenv("QCS_STREAM", "2")
    n, s = 12, 8
    ctr = _check(oracle, _diag_program(random.Random(5), n, 20), s, 9, [2.0 ** -45], 1.0)
    assert ctr["stream_left_slots"] > 0


def test_stream_wave_layout(oracle, monkeypatch):
    monkeypatch.setenv("QCS_STREAM", "2")
    monkeypatch.setenv("QCS_FORCE_BIG", "1")
    n, s = 13, 7
    ctr = _check(oracle, _diag_program(random.Random(11), n, 30), s, 1234, [cc.pow2_bound(1e-3, n)], 1.0)
    assert ctr["stream_slots"] > 0


def test_stream_default_threshold_of_slots(oracle, monkeypatch):
    # default mode: the streaming kernel from one slot per SM on (256 strides here)
    monkeypatch.delenv("QCS_STREAM", raising=False)
    n, s = 14, 6
    ctr = _check(oracle, _diag_program(random.Random(13), n, 24), s, 99, [cc.pow2_bound(1e-3, n)], 1.0)
    assert ctr["stream_slots"] > 0


def test_stream_persistent_kernel_suspends_and_resumes(oracle, monkeypatch):
    # wave layout, single-level ladder: the persistent kernel installs the strides itself; an arena
    # of about 1.5x the dense compressed state fills inside gates, which suspend, compact and resume
    # with the slots not installed yet
    monkeypatch.setenv("QCS_STREAM_PERSIST", "1")
    monkeypatch.setenv("QCS_FORCE_BIG", "1")
    monkeypatch.setenv("QCS_WAVE_SLOTS", "8")
    monkeypatch.setenv("QCS_INPLACE", "0")  # (no in-place rewrite: the arena fills inside gates)
    n, s = 13, 7
    monkeypatch.setenv("QCS_ARENA_BYTES", str(int(1.5 * 4.5 * (1 << n))))
    ctr = _check(oracle, _diag_program(random.Random(17), n, 30), s, 321, [cc.pow2_bound(1e-3, n)], 1.0)
    assert ctr["stream_slots"] > 0
    assert ctr["compactions"] > 0


def test_stream_persistent_kernel_reports_nomem(oracle, monkeypatch):
    monkeypatch.setenv("QCS_STREAM_PERSIST", "1")
    import paper_1811_05140_b200 as q
    monkeypatch.setenv("QCS_FORCE_BIG", "1")
    monkeypatch.setenv("QCS_WAVE_SLOTS", "8")
    n, s = 13, 7
    monkeypatch.setenv("QCS_ARENA_BYTES", str(3 * (1 << n)))  # less than the dense state at ~4.5 B per amplitude
    with pytest.raises(RuntimeError) as ei:
        gpu_run(_diag_program(random.Random(17), n, 30), s, 321, [cc.pow2_bound(1e-3, n)], 1.0)
    assert "block arena exhausted" in str(ei.value)


def test_stream_persistent_kernel_behind_a_precheck_suspension(oracle, monkeypatch):
    # an arena large enough for the pre-gate check to act (it keeps 1 MiB of slack): gates queued in
    # one pass suspend at unit 0 before the persistent kernel starts, compact and start over — the
    # installed flags of the gate before must not leak into the restarted one
    monkeypatch.setenv("QCS_STREAM_PERSIST", "1")
    monkeypatch.setenv("QCS_FORCE_BIG", "1")
    monkeypatch.setenv("QCS_WAVE_SLOTS", "64")
    monkeypatch.setenv("QCS_INPLACE", "0")  # (every gate leaves its old blocks behind: the arena does fill)
    n, s = 17, 8
    monkeypatch.setenv("QCS_ARENA_BYTES", str(int(2.5 * (1 << 20))))
    ctr = _check(oracle, _diag_program(random.Random(23), n, 16), s, 4321, [cc.pow2_bound(1e-3, n)], 1.0)
    assert ctr["stream_slots"] > 0
    assert ctr["compactions"] > 0


def test_stream_persistent_kernel_reuses_blocks_in_place(oracle, monkeypatch):
    # wave layout: a block the persistent kernel placed has a little slack, and the stride's next
    # encoding goes over it in place — a run of diagonal gates on a dense state must not grow the
    # arena (no compaction), where each gate used to leave the whole state behind as garbage
    monkeypatch.setenv("QCS_STREAM_PERSIST", "1")
    import paper_1811_05140_b200 as q
    from paper_1811_05140_b200 import metrics as mm
    monkeypatch.setenv("QCS_FORCE_BIG", "1")
    monkeypatch.setenv("QCS_INPLACE", "1")
    monkeypatch.setenv("QCS_WAVE_SLOTS", "16")
    n, s = 16, 7  # (512 strides: pair-unit targets take the fused path also under a stride-bit control)
    monkeypatch.setenv("QCS_ARENA_BYTES", str(int(3.2 * 4.5 * (1 << n))))
    rng = random.Random(29)
    U = cc.Unitary2x2
    prog = cc.CircuitProgram(n, [], "reuse")
    for t in range(n):
        prog.gates.append(cc.GateOp.single(U.hadamard(), t, f"h{t}"))
        prog.gates.append(cc.GateOp.single(U.phase(0.1 + 0.3 * t), t, f"p{t}"))
    n_prep = len(prog.gates)
    diag = [U.t_gate(), U.s_gate(), U.pauli_z(), U.phase(0.37)]
    for _ in range(40):
        t = rng.randrange(n)
        c = rng.randrange(n - 1)
        c = c + 1 if c >= t else c
        prog.gates.append(cc.GateOp.controlled(rng.choice(diag), c, t, f"c{c}t{t}") if rng.random() < 0.5
                          else cc.GateOp.single(rng.choice(diag), t, f"d{t}"))
    delta = cc.pow2_bound(1e-3, n)
    st, want = oracle_run(oracle, prog, s, 77, [delta], 1.0)
    lad, th = q.ErrorBoundLadder.make([delta]), q.RatioThreshold(1.0)
    gst = q.CompressedState.basis_state(q.StateGeometry.make(n, s), 77)
    m1 = q.apply_program_range(gst, prog, 0, n_prep + 2, lad, th)   # (two diagonal gates place the slack blocks)
    c1 = gst.counters()["compactions"]
    m2 = q.apply_program_range(gst, prog, n_prep + 2, len(prog.gates), lad, th)
    assert gst.counters()["compactions"] == c1
    got = mm.emit_csv(list(m1.records) + list(m2.records), with_elapsed=False)
    assert got == want, first_diff(want, got)
    assert gst.to_amplitudes().tobytes() == st.amplitudes().tobytes()
    for j in range(1 << (n - s)):
        assert gst.export_blocks(j)[0] == st.export_blocks(j), j
