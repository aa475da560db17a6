"""C3-shaped parity (BASELINE configs[2]: QFT, 2^20-amplitude strides) against
the UNMODIFIED reference, on the state bench.py's headline times: the exact
closed-form state at the start of QFT-n's last stage (circuit.qft_stage),
compressed by each engine from bit-identical amplitudes -- the reference
through compress_stride_adaptive + a QCKP checkpoint + CompressedState::load
(aalc.cpp:117-138, 466-586; oracle/ref_capi.cpp), the GPU through
qcs_load_strides_device -- then the whole last stage (CP(k, n-1) for every
k, H(n-1)).  The loaded amplitudes, every GateRecord field except wall time
and the final amplitudes must be identical, at the power-of-two bound the
bench uses and at SURVEY.md's own decimal mapping eps*2^-ceil(n/2)."""
import numpy as np
import pytest

from helpers import first_diff
from paper_1811_05140_b200 import circuit as cc
from paper_1811_05140_b200 import metrics as mm

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mapping", ["pow2", "survey"])
def test_qft_last_stage_s20_matches_reference(reference, tmp_path, mapping):
    import paper_1811_05140_b200 as q
    from paper_1811_05140_b200.stage import load_stage_state
    n, s, eps = 24, 20, 1e-3
    prog = cc.build_qft(n)
    x = next(cc.splitmix64(n)) & ((1 << n) - 1)
    g0 = len(prog.gates) - n
    delta = cc.pow2_bound(eps, n) if mapping == "pow2" else cc.survey_bound(eps, n)
    tables = cc.stage_tables(n, s, *cc.qft_stage(n, x, g0))
    rst = reference.state_from_tables(cc.print_circuit(prog), s, tables, [delta], 1.0,
                                      str(tmp_path / "stage.qckp"))
    lad, th = q.ErrorBoundLadder.make([delta]), q.RatioThreshold(1.0)
    gst = load_stage_state(q, n, s, x, g0, lad, th, 0)
    a_ref, a_gpu = rst.amplitudes(n), gst.to_amplitudes()
    assert a_gpu.tobytes() == a_ref.tobytes(), "loaded states differ"
    assert gst.compressed_bytes() == int(rst.stats()["compressed_bytes"])
    want = mm.strip_elapsed(rst.apply_csv(g0, len(prog.gates), [delta], 1.0))
    m = q.apply_program_range(gst, prog, g0, len(prog.gates), lad, th)
    got = mm.emit_csv(m.records, with_elapsed=False)
    assert got == want, first_diff(want, got)
    assert gst.to_amplitudes().tobytes() == rst.amplitudes(n).tobytes()
    # the closed form is the exact QFT output (the DFT row) after the last gate
    amps = gst.to_amplitudes()
    y = np.arange(1 << n, dtype=np.uint64)
    ph = ((np.uint64(x) * y) & np.uint64((1 << n) - 1)).astype(np.float64) * (2 * np.pi / (1 << n))
    e = np.exp(1j * ph) / np.sqrt(float(1 << n))
    fid = abs(np.vdot(e, amps)) / (np.linalg.norm(e) * np.linalg.norm(amps))
    assert fid > 1 - 1e-6
