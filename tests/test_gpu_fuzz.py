"""Randomised engine parity on the GPU: seeded random circuits (real and
complex single / controlled gates, phase flips, reflect_mean), random
geometries (including strides shorter than one 32-element sub-chunk), random
ladders (lossless, power-of-two and decimal bounds) and thresholds — every
GateRecord field except wall time, the amplitudes and every stored block must
equal the oracle's.  Exercises every encoder mode together (in-chunk and
split paths, the zero-imaginary-plane mode while the state is real, the
serial-chain policy for decimal bounds)."""
import math
import random

import pytest

from helpers import first_diff, gpu_run, oracle_run
from paper_1811_05140_b200 import circuit as cc

pytestmark = pytest.mark.gpu


def _random_program(rng, n):
    U = cc.Unitary2x2
    real = [U.hadamard(), U.pauli_x(), U.pauli_z()]
    cplx = [U.t_gate(), U.s_gate(), U.sqrt_x(), U.sqrt_y(), U.phase(0.37), U.pauli_y()]
    p = cc.CircuitProgram(n, [], "fuzz")
    real_phase = rng.random() < 0.5  # start with real gates only (zero-imaginary-plane mode)
    for i in range(rng.randrange(20, 70)):
        if real_phase and i > 25:
            real_phase = False
        r = rng.random()
        pool = real if real_phase else real + cplx
        t = rng.randrange(n)
        if r < 0.06:
            p.gates.append(cc.GateOp.phase_flip(rng.randrange(1 << n)))
        elif r < 0.09:
            p.gates.append(cc.GateOp.reflect_mean())
        elif r < 0.4 and n > 1:
            c = rng.randrange(n - 1)
            c = c + 1 if c >= t else c
            p.gates.append(cc.GateOp.controlled(rng.choice(pool), c, t, f"c{c}t{t}"))
        else:
            p.gates.append(cc.GateOp.single(rng.choice(pool), t, f"u{t}"))
    return p


def _random_ladder(rng, n):
    amp = 2.0 ** -(n / 2)
    kind = rng.randrange(4)
    if kind == 0:
        return [0.0], 1.0
    if kind == 1:
        return [2.0 ** math.floor(math.log2(amp * 1e-3))], 1.0
    if kind == 2:
        return [0.0, amp * 3e-5, amp * 1e-3], rng.choice([2.0, 8.0])
    return [2.0 ** math.floor(math.log2(amp * 1e-5)), amp * 7e-4], 4.0


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("QCS_FUZZ_CASES", "60"))))
def test_engine_fuzz_vs_oracle(oracle, seed):
    rng = random.Random(1000 + seed)
    n = rng.randrange(3, 14)
    s = rng.randrange(0, n + 1)
    prog = _random_program(rng, n)
    ladder, theta = _random_ladder(rng, n)
    basis = rng.randrange(1 << n)
    st, want = oracle_run(oracle, prog, s, basis, ladder, theta)
    res, got = gpu_run(prog, s, basis, ladder, theta)
    assert got == want, f"seed {seed} n={n} s={s} ladder={ladder}: " + first_diff(want, got)
    assert res.state.to_amplitudes().tobytes() == st.amplitudes().tobytes()
    for j in range(1 << (n - s)):
        assert res.state.export_blocks(j)[0] == st.export_blocks(j), (seed, j)
