"""The closed-form QFT stage state (circuit.qft_stage / stage_tables) that the
headline bench starts from, against the dense oracle (dense.cpp:30-76
restated in oracle/qcs_oracle.c) for every gate boundary of small QFTs, and
the reference arm's generator + compress_stride_adaptive + QCKP + load
(oracle/ref_capi.cpp) against it within the codec's point-wise bound."""
import numpy as np
import pytest

from paper_1811_05140_b200 import circuit as cc


def closed_form(n, x, g):
    m, r, zm, zv = cc.qft_stage(n, x, g)
    y = np.arange(1 << n, dtype=np.int64)
    R = np.zeros(1 << n, dtype=np.int64)
    for k in range(n):
        R = (R + ((y >> k) & 1) * r[k]) % (1 << n)
    return 2.0 ** (-m / 2) * np.exp(2j * np.pi * R / 2 ** n) * ((y & zm) == zv)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 7])
def test_qft_stage_matches_dense_every_gate(oracle, n):
    prog = cc.build_qft(n)
    for x in sorted({0, 1, (1 << n) - 1, 0x2B % (1 << n)}):
        for g in range(len(prog.gates) + 1):
            d = oracle.dense(n, prog.gates[:g], x)
            assert np.abs(closed_form(n, x, g) - d).max() < 1e-14, (x, g)


def test_stage_tables_factorisation():
    n, s, x = 9, 4, 301
    prog = cc.build_qft(n)
    for g in (0, len(prog.gates) - n, len(prog.gates) - 3, len(prog.gates)):
        t = cc.stage_tables(n, s, *cc.qft_stage(n, x, g))
        y = np.arange(1 << n)
        lo = t["lo_re"][y & 15] + 1j * t["lo_im"][y & 15]
        hi = t["hi_re"][y >> 4] + 1j * t["hi_im"][y >> 4]
        a = t["amp"] * lo * hi * ((y & t["zmask"]) == t["zval"])
        assert np.abs(a - closed_form(n, x, g)).max() < 1e-14


def test_reference_stage_state_within_bound(reference, oracle, tmp_path):
    n, s = 12, 8
    prog = cc.build_qft(n)
    x = next(cc.splitmix64(n)) & ((1 << n) - 1)
    g0 = len(prog.gates) - n
    delta = cc.pow2_bound(1e-3, n)
    st = reference.state_from_tables(cc.print_circuit(prog), s, cc.stage_tables(n, s, *cc.qft_stage(n, x, g0)),
                                     [delta], 1.0, str(tmp_path / "s.qckp"))
    a = st.amplitudes(n)
    e = closed_form(n, x, g0)
    assert np.abs(a.real - e.real).max() <= delta and np.abs(a.imag - e.imag).max() <= delta
    assert abs(st.stats()["norm_sq"] - 1.0) < 1e-3
