"""Codec plugin on the GPU (qcs_codec_compress / qcs_codec_decompress) vs the
oracle and the reference's golden blocks: block bytes must be identical."""
import numpy as np
import pytest

from helpers import golden_codec

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q():
    import paper_1811_05140_b200 as q
    return q


@pytest.mark.parametrize("case", [c[0] for c in golden_codec()])
def test_codec_golden_bytes(q, case):
    name, x, d, blk = next(c for c in golden_codec() if c[0] == case)
    got = q.compress(x, d)
    assert got == blk, f"{name}: {len(got)} vs {len(blk)} bytes"
    y = q.decompress(blk, x.size)
    if d == 0.0:
        assert y.tobytes() == x.tobytes()
    else:
        assert np.all(np.abs(y - x) <= d)


def _planes(rng, n):
    yield rng.normal(0, 1e-3, n)
    yield np.cumsum(rng.normal(0, 1e-5, n))
    yield rng.choice([0.0, 1.0, -0.5, 1e-301, 3.0e5, -0.0], n)
    yield rng.uniform(-1, 1, n) * (rng.uniform(0, 1, n) < 0.3)
    i = np.arange(n)
    yield np.cos(2 * np.pi * 0.013 * i) / 1024.0
    yield np.where(i % 97 == 0, 0.7, 1.0 / 4096.0)


@pytest.mark.parametrize("n", [1, 31, 32, 33, 1000, 4095, 4096, 4097, 8192 + 77, 50000])
def test_codec_fuzz_vs_oracle(q, oracle, n):
    rng = np.random.default_rng(n)
    for x in _planes(rng, n):
        for d in (0.0, 1e-6, 2.0 ** -20, 2.0 ** -12, 0.37):
            want = oracle.compress(x, d)
            got = q.compress(x, d)
            assert got == want, f"n={n} d={d} kind={x[:3]}: len {len(got)} vs {len(want)}, first diff at byte " + str(
                next((i for i, (a, b) in enumerate(zip(got, want)) if a != b), min(len(got), len(want))))
            y = q.decompress(got, n)
            assert y.tobytes() == oracle.decompress(want, n).tobytes()


def test_codec_long_runs(q, oracle):
    """Escape/literal runs and zero runs spanning CTA iterations (4096)."""
    n = 3 * 4096 + 100
    x = np.zeros(n)
    x[1000:9000] = np.random.default_rng(1).uniform(-1e6, 1e6, 8000)   # long escape run
    x[9500:9600] = 1e-4
    for d in (0.0, 1e-7, 2.0 ** -30):
        assert q.compress(x, d) == oracle.compress(x, d)
    y = np.random.default_rng(2).uniform(-1, 1, n)
    assert q.compress(y, 0.0) == oracle.compress(y, 0.0)   # full-plane literal run
    z = y.copy()
    z[5000:] = 0.0                                          # literal run closing early
    assert q.compress(z, 0.0) == oracle.compress(z, 0.0)


def test_codec_errors(q):
    with pytest.raises(q.CodecError) as e:
        q.compress(np.array([1.0, np.inf]), 1e-3)
    assert e.value.kind == "bad_value"
    with pytest.raises(ValueError):
        q.compress(np.zeros(4), -1.0)
    blk = q.compress(np.linspace(0, 1, 100), 1e-3)
    with pytest.raises(q.CodecError) as e:
        q.decompress(b"XXXX" + blk[4:], 100)
    assert e.value.kind == "bad_magic"
    with pytest.raises(q.CodecError) as e:
        q.decompress(blk[:-3], 100)
    assert e.value.kind == "truncated"
    with pytest.raises(q.CodecError) as e:
        q.decompress(blk[:4] + bytes([9]) + blk[5:], 100)
    assert e.value.kind == "unknown_codec"
    bad = bytearray(blk)
    bad[29] = 0x03  # tag 3: unknown payload token
    with pytest.raises(q.CodecError) as e:
        q.decompress(bytes(bad), 100)
    assert e.value.kind == "bad_value"


@pytest.mark.parametrize("max_rounds", [1, 2])
def test_codec_fuzz_neighbour_repair(q, oracle, monkeypatch, max_rounds):
    """The codec with the event rounds capped (QCS_MAX_ROUNDS): misses go to
    the neighbour-exit repair right away; bytes must not change."""
    monkeypatch.setenv("QCS_MAX_ROUNDS", str(max_rounds))
    for n in (33, 4097, 50000):
        rng = np.random.default_rng(1000 + n)
        for x in _planes(rng, n):
            for d in (2.0 ** -20, 2.0 ** -12):
                assert q.compress(x, d) == oracle.compress(x, d), (n, d)


@pytest.mark.parametrize("mode", ["0", "1"])
def test_codec_serial_chain_vs_oracle(q, oracle, monkeypatch, mode):
    """Codec plugin with decimal bounds: serial-chain precompute (1) and the
    event rounds (0) both reproduce the oracle's blocks."""
    monkeypatch.setenv("QCS_SERIAL_CHAIN", mode)
    rng = np.random.default_rng(5)
    for n in (1, 7, 33, 4096, 20000):
        for x in _planes(rng, n):
            for d in (1e-7, 1e-5, 3e-3):
                assert q.compress(x, d) == oracle.compress(x, d), (n, d)
