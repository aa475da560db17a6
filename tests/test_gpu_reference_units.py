"""The reference's own unit-test assertions (proj/tests/test_codec.cpp and
test_aalc.cpp, doctest suites that cannot be built here: vendor/ is absent),
restated against the B200 engine.  Data are seeded numpy draws instead of
std::mt19937_64 streams — every assertion is a property of the codec or the
engine, not of particular values; bit-for-bit agreement with the reference
is pinned elsewhere (golden runs, oracle fuzz, full-size runs)."""
import math
import os
import tempfile

import numpy as np
import pytest

from helpers import gpu_run
from paper_1811_05140_b200 import circuit as cc

pytestmark = pytest.mark.gpu

HEADER = 29


@pytest.fixture(scope="module")
def q():
    import paper_1811_05140_b200 as q
    return q


def _ratio(blk: bytes, n: int) -> float:
    return 8.0 * n / len(blk)  # CompressedBlock::ratio (codec.hpp:66-70): header included


# ---- test_codec.cpp ---------------------------------------------------------------

def test_lossless_single_spike_in_a_megaword(q):  # test_codec.cpp:39-48
    x = np.zeros(1 << 20)
    x[123456] = 1.0
    blk = q.compress(x, 0.0)
    assert len(blk) <= 64
    assert _ratio(blk, x.size) >= 131072.0
    assert q.decompress(blk, x.size).tobytes() == x.tobytes()


def test_lossless_random_doubles_expand_at_most_5_percent(q):  # :50-60
    x = np.random.default_rng(11).uniform(-1e6, 1e6, 4096)
    blk = q.compress(x, 0.0)
    assert _ratio(blk, x.size) >= 0.95
    assert q.decompress(blk, x.size).tobytes() == x.tobytes()


def test_lossless_empty_input(q):  # :62-69
    blk = q.compress(np.zeros(0), 0.0)
    assert len(blk) == HEADER
    assert q.decompress(blk, 0).size == 0


def test_lossless_bit_patterns_survive(q):  # :71-92
    rng = np.random.default_rng(13)
    specials = np.array([-0.0, 0.0, 5e-324, -5e-324, 1e-310, np.finfo(float).max, -np.finfo(float).tiny])
    w = rng.integers(0, 2 ** 63, 4000, dtype=np.uint64) * 2 + rng.integers(0, 2, 4000, dtype=np.uint64)
    r = w.view(np.float64).copy()
    r[~np.isfinite(r)] = 0.0
    x = np.concatenate([specials, r])
    x = np.insert(x, np.arange(7, x.size, 5), 0.0)
    blk = q.compress(x, 0.0)
    assert q.decompress(blk, x.size).tobytes() == x.tobytes()


def test_codecs_reject_nan_and_inf(q):  # :94-102, :176-184
    for bad in (np.array([1.0, np.nan]), np.array([np.inf])):
        for d in (0.0, 1e-4):
            with pytest.raises(q.CodecError):
                q.compress(bad, d)
    with pytest.raises(ValueError):
        q.compress(np.ones(1), -1.0)


def test_lossy_constant_plane_collapses(q):  # :104-114
    x = np.full(1000, 0.25)
    blk = q.compress(x, 1e-4)
    assert np.max(np.abs(q.decompress(blk, x.size) - x)) <= 1e-4
    assert _ratio(blk, x.size) >= 100.0


@pytest.mark.parametrize("delta", [1e-7, 1e-6, 1e-5, 1e-4, 1e-3, 1e-2])
def test_lossy_bound_holds_across_distributions(q, delta):  # :116-139
    rng = np.random.default_rng(17)
    x = np.concatenate([rng.uniform(-1, 1, 10000), rng.normal(0, delta, 10000), rng.normal(0, 1e8, 10000),
                        [0.0, -0.0, 1e300, -1e300]])
    y = q.decompress(q.compress(x, delta), x.size)
    assert np.max(np.abs(y - x)) <= delta


def test_lossy_escapes_store_extremes_exactly(q):  # :141-149
    x = np.array([1e308, -1e308, 0.0, 1e-12, 2.0, 2.0 + 1e-13])
    y = q.decompress(q.compress(x, 1e-7), x.size)
    assert np.max(np.abs(y - x)) <= 1e-7
    assert y[0] == 1e308 and y[1] == -1e308


@pytest.mark.parametrize("delta", [1e-6, 1e-3])
def test_lossy_recompression_is_stable(q, delta):  # :151-165
    x = np.random.default_rng(19).uniform(-2, 2, 5000)
    r1 = q.decompress(q.compress(x, delta), x.size)
    r2 = q.decompress(q.compress(r1, delta), x.size)
    assert r1.tobytes() == r2.tobytes()


def test_lossy_uniform_amplitude_plane(q):  # :167-174
    x = np.full(1 << 20, 1.0 / math.sqrt(1 << 20))
    blk = q.compress(x, 1e-7)
    assert _ratio(blk, x.size) >= 100000.0
    assert np.max(np.abs(q.decompress(blk, x.size) - x)) <= 1e-7


def test_decompression_is_deterministic(q):  # :186-197
    x = np.random.default_rng(23).uniform(-1, 1, 3000)
    blk = q.compress(x, 1e-5)
    assert q.decompress(blk, x.size).tobytes() == q.decompress(blk, x.size).tobytes()


def test_block_container_rejects_corruption(q):  # :199-271
    blk = bytearray(q.compress(np.array([1.5, 0.0, -2.25, 1e-9]), 1e-6))
    cases = [(bytes(b"X") + bytes(blk[1:]), "bad_magic"), (bytes(blk[:-1]), "truncated"),
             (bytes(blk[:4]) + b"\x09" + bytes(blk[5:]), "unknown_codec")]
    for data, kind in cases:
        with pytest.raises(q.CodecError) as e:
            q.decompress(data, 4)
        assert e.value.kind == kind


def test_compress_dispatch_on_the_bound(q):  # :273-278
    x = np.full(64, 0.125)
    assert q.compress(x, 0.0)[4] == 0   # kCodecLossless
    assert q.compress(x, 1e-5)[4] == 1  # kCodecLossy


# ---- test_aalc.cpp ------------------------------------------------------------------

def _adaptive_stride(q, re, im, ladder, theta):
    """compress_stride_adaptive (aalc.cpp:117-138) through the engine: a one-
    stride state holding (re, im), one identity gate, the stride's report."""
    n = int(math.log2(re.size))
    st = q.CompressedState.basis_state(q.StateGeometry.make(n, n), 0)
    blob = q.compress(re, 0.0) + q.compress(im, 0.0)
    q.engine._check(q.engine.lib().qcs_import_blocks(st._h, 0, blob, len(blob), 1.0,
                                                      float(np.sum(re * re + im * im))))
    g = cc.GateOp.single(cc.Unitary2x2.identity(), 0, "id")
    res = st.apply_gate(g, q.ErrorBoundLadder.make(ladder), q.RatioThreshold(theta))
    return res.reports[0]


def test_adaptive_all_zero_stride_clears_any_threshold(q):  # test_aalc.cpp:126-139
    L = 1 << 12
    rep = _adaptive_stride(q, np.zeros(L), np.zeros(L), list(q.ErrorBoundLadder.default_ladder().bounds), 16.0)
    assert rep.chosen_delta == 0.0 and rep.ratio >= 16.0 and rep.threshold_met
    assert rep.bytes_in == L * 16


def test_adaptive_single_level_cannot_escalate(q):  # :141-153
    rng = np.random.default_rng(31)
    L = 1 << 12
    rep = _adaptive_stride(q, rng.uniform(-1, 1, L), rng.uniform(-1, 1, L), [0.0], 16.0)
    assert rep.chosen_delta == 0.0 and not rep.threshold_met and rep.ratio < 16.0


def test_adaptive_escalation_picks_the_smallest_workable_bound(q):  # :155-183
    L = 1 << 12
    i = np.arange(L)
    c = 1.0 / math.sqrt(L)
    re, im = c * np.cos(2 * math.pi * i / L), c * np.sin(2 * math.pi * i / L)
    ladder = list(q.ErrorBoundLadder.default_ladder().bounds)
    rep = _adaptive_stride(q, re, im, ladder, 16.0)
    assert rep.threshold_met and rep.ratio >= 16.0 and rep.chosen_delta > 0.0
    for smaller in ladder:
        if smaller >= rep.chosen_delta:
            break
        assert _adaptive_stride(q, re, im, [smaller], 16.0).ratio < 16.0


def test_hadamard_on_zero_through_the_compressed_path(q):  # :185-198
    st = q.CompressedState.basis_state(q.StateGeometry.make(1, 1), 0)
    res = st.apply_gate(cc.GateOp.single(cc.Unitary2x2.hadamard(), 0, "h 0"),
                        q.ErrorBoundLadder.lossless_only(), q.RatioThreshold(1.0))
    a = st.to_amplitudes()
    h = 1.0 / math.sqrt(2.0)
    assert abs(a[0] - h) < 1e-15 and abs(a[1] - h) < 1e-15
    assert abs(res.norm_after - 1.0) <= 1e-12


def _random_program(n, count, seed):
    rng = np.random.default_rng(seed)
    U = cc.Unitary2x2
    pool = [U.hadamard(), U.pauli_x(), U.t_gate(), U.s_gate(), U.sqrt_x(), U.phase(0.77)]
    p = cc.CircuitProgram(n, [], "random")
    for _ in range(count):
        t = int(rng.integers(n))
        if n > 1 and rng.random() < 0.3:
            c = int(rng.integers(n - 1))
            c = c + 1 if c >= t else c
            p.gates.append(cc.GateOp.controlled(pool[int(rng.integers(len(pool)))], c, t, "c"))
        else:
            p.gates.append(cc.GateOp.single(pool[int(rng.integers(len(pool)))], t, "u"))
    return p


def test_lossless_ladder_is_semantically_transparent(q, oracle):  # :200-214
    for n in (1, 2, 3, 5, 8, 12):
        for s in sorted({0, n // 2, n}):
            p = _random_program(n, 60, 37 + n * 13 + s)
            res, _ = gpu_run(p, s, 0, [0.0], 1.0)
            ref = oracle.dense(n, p.gates, 0)
            assert np.max(np.abs(res.state.to_amplitudes() - ref)) < 1e-12, (n, s)


def test_runs_stay_normalized_after_every_gate(q):  # :216-234
    for p in (cc.build_qft(10), cc.build_grover(10, 5, 8), _random_program(10, 80, 99)):
        res, _ = gpu_run(p, 6, 1, list(q.ErrorBoundLadder.default_ladder().bounds), 16.0)
        for r in res.metrics.records:
            assert abs(r.norm_after - 1.0) <= 1e-9
        a = res.state.to_amplitudes()
        assert abs(float(np.sum(np.abs(a) ** 2)) - 1.0) <= 1e-9


def test_threshold_contract(q):  # :236-257
    p = cc.build_qft(10)
    res, _ = gpu_run(p, 10, 1, list(q.ErrorBoundLadder.default_ladder().bounds), 16.0)
    assert res.metrics.threshold_violations == 0
    for r in res.metrics.records:
        assert r.min_ratio >= 16.0 and r.min_ratio <= r.mean_ratio + 1e-12 and r.bytes_after > 0
    flagged, _ = gpu_run(p, 10, 1, [0.0], 16.0)
    assert flagged.metrics.threshold_violations > 0


def test_controlled_gates_skip_strides_with_clear_control(q, oracle):  # :259-287
    geom = q.StateGeometry.make(8, 4)
    st = q.CompressedState.basis_state(geom, 0)
    lad, th = q.ErrorBoundLadder.lossless_only(), q.RatioThreshold(1.0)
    gates = [cc.GateOp.single(cc.Unitary2x2.hadamard(), k, "h") for k in range(8)]
    for g in gates:
        st.apply_gate(g, lad, th)
    cp = cc.GateOp.controlled(cc.Unitary2x2.phase(0.3), 7, 0, "cp 7 0")
    res = st.apply_gate(cp, lad, th)
    assert len(res.reports) == geom.n_strides() // 2
    assert all(r.stride_index & (geom.n_strides() >> 1) for r in res.reports)
    ref = oracle.dense(8, gates + [cp], 0)
    assert np.max(np.abs(st.to_amplitudes() - ref)) < 1e-12


def test_lossy_drift_is_repaired_across_skipped_strides(q, oracle):  # :289-315
    p = cc.CircuitProgram(8, [], "drift")
    p.gates += [cc.GateOp.single(cc.Unitary2x2.hadamard(), k, "h") for k in range(8)]
    for rep in range(6):
        p.gates.append(cc.GateOp.controlled(cc.Unitary2x2.phase(0.7), 7, 2, "cp"))
        p.gates.append(cc.GateOp.controlled(cc.Unitary2x2.phase(0.3), 6, 1, "cp"))
        p.gates.append(cc.GateOp.single(cc.Unitary2x2.t_gate(), rep % 8, "t"))
    res, _ = gpu_run(p, 3, 0, [0.0, 1e-6, 1e-5], 4.0)
    a = res.state.to_amplitudes()
    assert oracle.fidelity(oracle.dense(8, p.gates, 0), a) > 0.999
    assert abs(float(np.sum(np.abs(a) ** 2)) - 1.0) < 1e-9


def test_invalid_gates_leave_the_state_intact(q):  # :317-332
    st = q.CompressedState.basis_state(q.StateGeometry.make(4, 2), 3)
    before = st.to_amplitudes().tobytes()
    lad, th = q.ErrorBoundLadder.lossless_only(), q.RatioThreshold(1.0)
    with pytest.raises(IndexError):
        st.apply_gate(cc.GateOp.single(cc.Unitary2x2.pauli_x(), 9, "x 9"), lad, th)
    with pytest.raises(IndexError):
        st.apply_gate(cc.GateOp.phase_flip(100), lad, th)
    assert st.to_amplitudes().tobytes() == before


def test_empty_program_returns_the_initial_state(q):  # :334-346
    p = cc.CircuitProgram(12, [], "empty")
    res, _ = gpu_run(p, 12, 0, list(q.ErrorBoundLadder.default_ladder().bounds), 16.0)
    assert not res.metrics.records
    assert res.metrics.init_min_ratio > 16.0
    assert res.state.to_amplitudes()[0] == 1.0 + 0j


def test_checkpoint_restores_amplitudes_and_scales(q):  # :376-395
    geom = q.StateGeometry.make(8, 4)
    lad = q.ErrorBoundLadder.default_ladder()
    res, _ = gpu_run(cc.build_qft(8), 4, 1, list(lad.bounds), 8.0)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "roundtrip.qckp")
        res.state.save(path, lad.fingerprint())
        st, fp = q.CompressedState.load(path)
    assert fp == lad.fingerprint()
    assert st.to_amplitudes().tobytes() == res.state.to_amplitudes().tobytes()
    for j in range(geom.n_strides()):
        assert st.stride_scale(j) == res.state.stride_scale(j)


# ---- test_circuit.cpp ---------------------------------------------------------------

@pytest.mark.parametrize("n", [1, 2, 3, 5, 7])
def test_qft_equals_the_dft_row_for_every_input(q, n):  # test_circuit.cpp:18-30, :199-209
    """Through the engine (lossless ladder, s = n // 2): QFT|x> is the DFT row
    a_y = e^{2 pi i x y / 2^n} / 2^{n/2} for every basis input x."""
    prog = cc.build_qft(n)
    y = np.arange(1 << n)
    for x in range(1 << n):
        res, _ = gpu_run(prog, n // 2, x, [0.0], 1.0)
        want = np.exp(2j * math.pi * ((x * y) % (1 << n)) / (1 << n)) / math.sqrt(1 << n)
        assert np.max(np.abs(res.state.to_amplitudes() - want)) < 1e-12, (n, x)
