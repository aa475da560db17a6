"""Crafted states for the streaming kernel's rare paths, against the UNMODIFIED
reference (oracle/_ref): both engines compress the same product-form amplitude
tables (oracle/ref_capi.cpp ref_state_from_tables; qcs_load_strides_device) and
run the same program of diagonal gates; the loaded amplitudes, every GateRecord
field and the final amplitudes must be identical.

The tables put, on the 2*delta lattice of the bound: exact half-lattice points
and their neighbours one ulp away (the reference's llround against the
kernel's round-to-even: the unproven-step path), zero runs of every length
across sub-chunk, lane and iteration boundaries, stretches whose codes are all
zero while the values are not, dense noise, spikes that escape (the slot must
come out of the legacy encoder), and a state of huge norm whose squares do not
fit the running sum exactly (rounding, ties and binade crossings of the stored
sum of squares; its gates act on the stride-index qubits only, so the planes
stay smooth and nothing escapes)."""
import numpy as np
import pytest

from helpers import first_diff
from paper_1811_05140_b200 import circuit as cc
from paper_1811_05140_b200 import metrics as mm

pytestmark = pytest.mark.gpu

DELTA = 2.0 ** -20
TD = 2.0 * DELTA


def _lo_tables(kind, L, rng):
    m = rng.integers(-900, 900, size=L).astype(np.float64)
    re = m * TD
    im = rng.integers(-900, 900, size=L).astype(np.float64) * TD
    if kind in ("halves", "spikes", "huge"):
        a = slice(0, L // 8)                       # exact halves
        re[a] = (m[a] + 0.5) * TD
        b = slice(L // 8, L // 4)                  # one ulp either side of a half
        h = (m[b] + 0.5) * TD
        re[b] = np.where(rng.integers(0, 2, size=h.size) == 1, np.nextafter(h, np.inf), np.nextafter(h, -np.inf))
        im[b] = (rng.integers(-900, 900, size=h.size) + 0.5) * TD
    if kind in ("runs", "halves", "spikes"):
        z = np.zeros(L, dtype=bool)                # zero runs of many lengths and alignments
        pos = L // 4
        for ln in (1, 2, 31, 32, 33, 63, 64, 65, 127, 129, 1000, 4097):
            if pos + ln + 7 >= L:
                break
            z[pos:pos + ln] = True
            pos += ln + int(rng.integers(1, 40))
        re[z] = 0.0
        im[z & (rng.random(L) < 0.7)] = 0.0
        c = slice(L - L // 8, L - L // 16)         # codes all zero, values not: a slow ramp below delta
        re[c] = 17 * TD + np.arange(L // 16) * (TD * 2.0 ** -12)
        im[c] = -5 * TD
    if kind == "spikes":
        for k in rng.integers(0, L, size=6):       # jumps of more than 2^15 bins: the reference escapes
            re[k] = 0.9
    if kind == "huge":
        # lattice indices climbing (in steps the codes can hold) to 2^24: the squares, multiples of
        # (2 delta)^2 up to 2^48 of them, no longer fit the running sum exactly
        k = np.arange(L, dtype=np.float64)
        re = (np.minimum(30000.0 * k, 2.0 ** 24) + m) * TD
        im = (np.minimum(20000.0 * k, 2.0 ** 23) + rng.integers(-900, 900, size=L)) * TD
    return re, im


def _program(n, rng, gates=14, qmin=0):
    """Diagonal gates in the reference's text format; both engines parse the same text.
    qmin > 0: only qubits from qmin on (whole strides change phase: smooth planes stay smooth)."""
    lines = [f"qubits {n}", f"z {int(rng.integers(qmin, n))}"]  # first gate: values unchanged up to sign
    for _ in range(gates):
        t = int(rng.integers(qmin, n))
        r = rng.random()
        if r < 0.5 and n - qmin > 1:
            c = int(rng.integers(qmin, n - 1))
            c = c + 1 if c >= t else c
            lines.append(f"cz {c} {t}" if r < 0.2 else f"cp {c} {t} {0.3 + 0.1 * t!r}")
        elif r < 0.6 and qmin == 0:
            lines.append(f"flip {int(rng.integers(0, 1 << n))}")
        else:
            lines.append(f"{'zst'[int(rng.integers(0, 3))]} {t}")
    return cc.parse_circuit("\n".join(lines) + "\n")


def _load_gpu(q, n, s, tables, lad, th):
    import torch
    from paper_1811_05140_b200.stage import StageGen
    geom = q.StateGeometry.make(n, s)
    st = q.CompressedState.basis_state(geom, 0, device=0)
    gen = StageGen(tables, n, s, 0)
    NS, L = geom.n_strides(), geom.stride_len()
    buf = torch.empty(NS * 2 * L, dtype=torch.float64, device=0)
    gen.fill(buf.view(NS, 2, L), 0, NS)
    torch.cuda.synchronize()
    st.load_strides_device(0, NS, buf.data_ptr(), lad, th)
    return st


@pytest.mark.parametrize("lanes", ["128", "512"])
@pytest.mark.parametrize("kind", ["dense", "runs", "halves", "spikes", "huge"])
def test_crafted_state_matches_reference(reference, tmp_path, monkeypatch, kind, lanes):
    import paper_1811_05140_b200 as q
    monkeypatch.setenv("QCS_STREAM_LANES", lanes)
    # (huge: 256 strides, so that its pair units on the stride-index qubits take the fused path)
    n, s = (21, 13) if kind == "huge" else (15, 13)
    L, NS = 1 << s, 1 << (n - s)
    rng = np.random.default_rng(sum(map(ord, kind)) * 1000 + int(lanes))
    lo_re, lo_im = _lo_tables(kind, L, rng)
    hi_re = np.array([1.0, 0.5, 1.0, 0.25] * (NS // 4))
    tables = dict(lo_re=lo_re, lo_im=lo_im, hi_re=hi_re, hi_im=np.zeros(NS), amp=1.0, zmask=0, zval=0)
    prog = _program(n, rng, qmin=s if kind == "huge" else 0)
    rst = reference.state_from_tables(cc.print_circuit(prog), s, tables, [DELTA], 1.0, str(tmp_path / "crafted.qckp"))
    lad, th = q.ErrorBoundLadder.make([DELTA]), q.RatioThreshold(1.0)
    gst = _load_gpu(q, n, s, tables, lad, th)
    assert gst.to_amplitudes().tobytes() == rst.amplitudes(n).tobytes(), "loaded states differ"
    want = mm.strip_elapsed(rst.apply_csv(0, len(prog.gates), [DELTA], 1.0))
    m = q.apply_program_range(gst, prog, 0, len(prog.gates), lad, th)
    got = mm.emit_csv(m.records, with_elapsed=False)
    assert got == want, first_diff(want, got)
    assert gst.to_amplitudes().tobytes() == rst.amplitudes(n).tobytes()
    ctr = gst.counters()
    assert ctr["stream_slots"] + ctr["stream_left_slots"] > 0
    if kind == "spikes":
        assert ctr["stream_left_slots"] > 0
    if kind in ("dense", "halves", "huge"):
        assert ctr["stream_slots"] > 0
