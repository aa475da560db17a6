"""Generate tests/golden/ from the UNMODIFIED reference (oracle/_ref/libqcsref.so).

TEST INFRASTRUCTURE ONLY.  Run in the build container (where /root/reference
exists):  python oracle/make_golden.py
The reference stores no golden vectors of its own, so these
are produced by running it here; the fixtures pin both our C restatement
(oracle/qcs_oracle.c) and the CUDA path.

Outputs (small, committed):
  tests/golden/codec.npz        inputs and QCS1 blocks (reference compress)
  tests/golden/circuits/*.txt   reference-built circuits (build_random, ...)
  tests/golden/runs.json        per-run CSV (elapsed column zeroed), sha256 of
                                the final amplitudes, final stats
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from oracle import Reference  # noqa: E402
from paper_1811_05140_b200 import circuit as cc  # noqa: E402
from paper_1811_05140_b200 import metrics as mm  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
DEFAULT_LADDER = [0.0, 1e-7, 1e-6, 1e-5, 1e-4, 1e-3]


def codec_inputs():
    """Seeded inputs shaped like the reference's codec tests
    (test_codec.cpp:39-197) plus state-shaped planes; numpy PCG64 seeds."""
    rng = np.random.default_rng(20260101)
    cases = []
    spike = np.zeros(1 << 16)
    spike[12345] = 1.0
    cases.append(("lossless_spike", spike, 0.0))
    cases.append(("lossless_random", rng.uniform(-1e6, 1e6, 4096), 0.0))
    bits = rng.integers(0, 2**63, 3000, dtype=np.uint64).view(np.float64).copy()
    bits[~np.isfinite(bits)] = 0.0
    bits[::5] = 0.0
    special = np.array([-0.0, 0.0, 5e-324, -5e-324, 1e-310, np.finfo(float).max, -np.finfo(float).tiny])
    cases.append(("lossless_bits", np.concatenate([special, bits]), 0.0))
    cases.append(("lossless_empty", np.zeros(0), 0.0))
    cases.append(("lossy_constant", np.full(1000, 0.25), 1e-4))
    for d in (1e-7, 1e-5, 1e-3, 1e-2):
        mix = np.concatenate([rng.uniform(-1, 1, 3000), rng.normal(0, d, 3000),
                              rng.normal(0, 1e8, 3000), [0.0, -0.0, 1e300, -1e300]])
        cases.append((f"lossy_mix_{d:g}", mix, d))
    cases.append(("lossy_escapes", np.array([1e308, -1e308, 0.0, 1e-12, 2.0, 2.0 + 1e-13]), 1e-7))
    cases.append(("lossy_uniform", np.full(1 << 16, 1.0 / np.sqrt(1 << 16)), 1e-7))
    i = np.arange(1 << 15)
    wave = np.cos(2 * np.pi * 37 * i / (1 << 15)) / 256.0
    cases.append(("lossy_wave_pow2", wave, 2.0 ** -22))
    cases.append(("lossy_wave_dec", wave, 9.765625e-7))
    cases.append(("lossy_odd_len", rng.uniform(-0.01, 0.01, 4097 * 3 + 17), 2.0 ** -20))
    return cases


def run_cases():
    """(name, circuit text, stride_bits, basis, ladder, theta)."""
    R = Reference()
    out = []
    out.append(("qft10_s6_default", cc.print_circuit(cc.build_qft(10)), 6, 1, DEFAULT_LADDER, 16.0))
    out.append(("qft10_s0_default", cc.print_circuit(cc.build_qft(10)), 0, 1, DEFAULT_LADDER, 8.0))
    out.append(("qft12_s8_pow2", cc.print_circuit(cc.build_qft(12)), 8, 77,
                [cc.pow2_bound(1e-3, 12)], 1.0))
    out.append(("qft12_s12_c1map", cc.print_circuit(cc.build_qft(12)), 12, 1234,
                [1e-3 * 2.0 ** -6], 1.0))
    out.append(("grover10_ref", R.builtin(1, 10, 5, 8), 6, 0, DEFAULT_LADDER, 16.0))
    out.append(("grover12_gates_pow2", cc.print_circuit(cc.build_grover_gate_form(12, 3001, 4)),
                8, 0, [cc.pow2_bound(1e-4, 12)], 1.0))
    out.append(("grid3x3_pow2", cc.print_circuit(cc.build_grid(3, 3, 8, 5)), 5, 0,
                [cc.pow2_bound(1e-2, 9)], 1.0))
    for n, seed in ((8, 99), (10, 808)):
        txt = R.builtin(2, n, seed, 80)
        out.append((f"random{n}_lossless", txt, n // 2, 0, [0.0], 1.0))
        out.append((f"random{n}_ladder", txt, n // 2, 3, [0.0, 1e-6, 1e-5], 4.0))
    out.append(("qft14_s14_pow2", cc.print_circuit(cc.build_qft(14)), 14, 4321,
                [cc.pow2_bound(1e-3, 14)], 1.0))
    out.append(("qft14_s13_lossless", cc.print_circuit(cc.build_qft(14)), 13, 9, [0.0], 16.0))
    return out


def main():
    R = Reference()
    os.makedirs(os.path.join(GOLD, "circuits"), exist_ok=True)
    arrays = {}
    names = []
    for name, x, d in codec_inputs():
        blk = R.compress(x, d)
        arrays[f"{name}__x"] = x
        arrays[f"{name}__blk"] = np.frombuffer(blk, dtype=np.uint8)
        arrays[f"{name}__delta"] = np.array([d])
        names.append(name)
    np.savez_compressed(os.path.join(GOLD, "codec.npz"), names=np.array(names), **arrays)

    runs = {}
    for name, text, s, basis, ladder, theta in run_cases():
        path = os.path.join(GOLD, "circuits", name + ".txt")
        with open(path, "w") as f:
            f.write(text)
        csv, amps, summ = R.run(text, s, basis, ladder, theta, workers=0)
        n = int(text.split()[1])
        dense = R.dense(text, basis, n)
        fid = abs(np.vdot(dense, amps)) / (np.linalg.norm(dense) * np.linalg.norm(amps))
        runs[name] = dict(circuit=f"circuits/{name}.txt", stride_bits=s, basis=basis,
                          ladder=ladder, theta=theta, csv=mm.strip_elapsed(csv),
                          amps_sha256=hashlib.sha256(amps.tobytes()).hexdigest(),
                          compressed_bytes=int(summ["compressed_bytes"]),
                          norm_sq_tracked=summ["norm_sq_tracked"],
                          overall_min_ratio=summ["overall_min_ratio"], fidelity=fid)
        print(f"{name}: {int(summ['n_records'])} gates, fid {fid:.12f}")
    with open(os.path.join(GOLD, "runs.json"), "w") as f:
        json.dump(runs, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
