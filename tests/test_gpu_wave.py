"""Wave layout for states too large for whole-gate staging:
one arena with in-place compaction, per-wave staging buffers, per-wave commit.
Forced on small states (QCS_FORCE_BIG, tiny waves, tiny arenas) so every
code path runs against the oracle bit for bit."""
import numpy as np
import pytest

from helpers import first_diff, golden_program, golden_runs, gpu_run, oracle_run, sha
from paper_1811_05140_b200 import circuit as cc

pytestmark = pytest.mark.gpu


@pytest.fixture
def wave_env(monkeypatch):
    def set_(wave, arena, inplace="0"):
        # (inplace 0: every rewritten stride gets a new block, so these small arenas fill, suspend
        # and compact as they are meant to; test_wave_layout_in_place runs the same cases with the
        # default in-place rewrite)
        monkeypatch.setenv("QCS_FORCE_BIG", "1")
        monkeypatch.setenv("QCS_WAVE_SLOTS", str(wave))
        monkeypatch.setenv("QCS_ARENA_BYTES", str(arena))
        monkeypatch.setenv("QCS_INPLACE", inplace)
    return set_


CASES = [
    # kind, n, s, basis, ladder, theta, wave slots, arena bytes
    ("qft", 11, 5, 0, [0.0, 1e-7, 1e-6, 1e-5, 1e-4, 1e-3], 16.0, 4, 3 * (16 << 11)),
    ("qft", 12, 6, 9, [2.0 ** -18], 1.0, 6, 2 * (16 << 12)),
    ("qft", 12, 3, 1, [0.0], 1.0, 8, 3 * (16 << 12)),
    ("grover_gates", 12, 8, 0, [2.0 ** -20], 1.0, 2, 1 << 16),
    ("grover_ref", 10, 4, 0, [0.0, 1e-6, 1e-4], 32.0, 4, 3 * (16 << 10)),
    ("grid", 9, 4, 0, [2.0 ** -14], 1.0, 2, 3 * (16 << 9)),
    ("qft", 14, 13, 5, [2.0 ** -19], 1.0, 1, 3 * (16 << 14)),
]


def _prog(kind, n):
    if kind == "qft":
        return cc.build_qft(n)
    if kind == "grover_gates":
        return cc.build_grover_gate_form(n, 77, 3)
    if kind == "grover_ref":
        return cc.build_grover(n, 33, 6)
    return cc.build_grid(3, 3, 10, 3)


@pytest.mark.parametrize("kind,n,s,basis,ladder,theta,wave,arena", CASES)
def test_wave_layout_matches_oracle(oracle, wave_env, kind, n, s, basis, ladder, theta, wave, arena):
    wave_env(wave, arena)
    prog = _prog(kind, n)
    st, want = oracle_run(oracle, prog, s, basis, ladder, theta)
    res, got = gpu_run(prog, s, basis, ladder, theta)
    assert got == want, first_diff(want, got)
    assert res.state.to_amplitudes().tobytes() == st.amplitudes().tobytes()
    c = res.state.counters()
    w = max(min(wave, 1 << (n - s)), min(1 << (n - s), 2))
    assert c["wave_slots"] == (w - 1 if w > 1 and w & 1 else w)
    for j in range(1 << (n - s)):
        assert res.state.export_blocks(j)[0] == st.export_blocks(j)


@pytest.mark.parametrize("kind,n,s,basis,ladder,theta,wave,arena", CASES)
def test_wave_layout_in_place(oracle, wave_env, kind, n, s, basis, ladder, theta, wave, arena):
    # blocks rewritten in place when they fit (the default): same results, every path
    wave_env(wave, arena, inplace="1")
    prog = _prog(kind, n)
    st, want = oracle_run(oracle, prog, s, basis, ladder, theta)
    res, got = gpu_run(prog, s, basis, ladder, theta)
    assert got == want, first_diff(want, got)
    assert res.state.to_amplitudes().tobytes() == st.amplitudes().tobytes()
    for j in range(1 << (n - s)):
        assert res.state.export_blocks(j)[0] == st.export_blocks(j)


@pytest.mark.parametrize("name", ["qft12_s8_pow2", "grover10_ref", "random10_ladder", "grid3x3_pow2"])
def test_wave_layout_matches_golden(wave_env, name):
    e = golden_runs()[name]
    prog = golden_program(e)
    wave_env(2, (16 << prog.n_qubits) + (1 << 16))
    res, csv = gpu_run(prog, e["stride_bits"], e["basis"], e["ladder"], e["theta"])
    assert csv == e["csv"], first_diff(e["csv"], csv)
    assert sha(res.state.to_amplitudes()) == e["amps_sha256"]
    if name != "grover10_ref":  # Grover blocks are tiny: the arena never fills
        assert res.state.counters()["compactions"] > 0


def test_wave_layout_compacts_and_reports_nomem(oracle, wave_env):
    import paper_1811_05140_b200 as q
    prog = cc.build_qft(10)
    lad = [0.0]
    wave_env(2, 2 * (16 << 10))
    st, want = oracle_run(oracle, prog, 4, 3, lad, 1.0)
    res, got = gpu_run(prog, 4, 3, lad, 1.0)
    assert got == want
    assert res.state.counters()["compactions"] > 0
    # an arena that cannot hold the lossless state at all
    wave_env(2, 4096)
    with pytest.raises(RuntimeError) as ei:
        gpu_run(prog, 4, 3, lad, 1.0)
    assert "block arena exhausted" in str(ei.value)


def test_wave_layout_hot_block_beyond_16_bytes(oracle, wave_env):
    """Basis state whose hot block is longer than 16 bytes (stride bits 22,
    in-stride offset 2^21: two 4-byte varints around the word) in a stride of
    a later wave: the first wave's blocks must be placed after it."""
    n, s = 24, 22
    basis = 3 * (1 << s) + (1 << 21)
    prog = cc.CircuitProgram(n, [cc.GateOp.single(cc.Unitary2x2.hadamard(), 0, "h 0"),
                                 cc.GateOp.single(cc.Unitary2x2.hadamard(), 23, "h 23")], "hot")
    wave_env(2, 1 << 28)
    st, want = oracle_run(oracle, prog, s, basis, [2.0 ** -20], 1.0)
    res, got = gpu_run(prog, s, basis, [2.0 ** -20], 1.0)
    assert got == want, first_diff(want, got)
    assert res.state.to_amplitudes().tobytes() == st.amplitudes().tobytes()
