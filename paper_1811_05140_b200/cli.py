"""Command-line front end on the B200 engine, after the reference's qcsim
(tools/qcsim.cpp): the subcommands simulate / compare / bench / codec with
the same flags, defaults (theta 16, ladder 0,1e-7,1e-6,1e-5,1e-4,1e-3, stride
bits min(n, 20)), printed summary, CSV / JSON artifacts and exit codes
(0 success; 1 runtime failure; 2 usage or configuration error: a bad flag,
std::invalid_argument, std::out_of_range, ParseError; qcsim.cpp:393-398,
441-468).  Usage: python -m paper_1811_05140_b200 <subcommand> ...
"""
from __future__ import annotations

import argparse
import math
import os
import sys
import time

from . import circuit as cc
from . import metrics as mm

DEFAULT_LADDER = "0,1e-7,1e-6,1e-5,1e-4,1e-3"


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage errors exit 2 (CLI11's ParseError)
        self.print_usage(sys.stderr)
        print(f"error: {message}", file=sys.stderr)
        raise SystemExit(2)


def _add_circuit(p):
    p.add_argument("--circuit", required=True,
                   help="circuit file path, or builtin:qft | builtin:grover | builtin:random")
    p.add_argument("--qubits", type=int, default=0, help="qubit count for builtin circuits")
    p.add_argument("--basis", type=int, default=0, help="initial computational basis index")
    p.add_argument("--marked", type=int, default=0, help="marked basis index (grover)")
    p.add_argument("--iterations", type=int, default=-1, help="grover iterations, -1 = optimal")
    p.add_argument("--gates", type=int, default=100, help="gate count (random builtin)")
    p.add_argument("--seed", type=int, default=1, help="seed for builtin:random; qft/grover ignore it")


def _add_pipeline(p):
    p.add_argument("--theta", type=float, default=16.0, help="compression ratio threshold")
    p.add_argument("--ladder", default=DEFAULT_LADDER, help="comma-separated error bounds, 0 = lossless level")
    p.add_argument("--stride-bits", type=int, default=-1, help="log2 amplitudes per stride, -1 = min(qubits, 20)")
    p.add_argument("--workers", type=int, default=0,
                   help="accepted for compatibility; results never depend on it (one GPU)")
    p.add_argument("--device", type=int, default=0, help="CUDA device")
    p.add_argument("--out-csv", default="", help="write per-gate records here")
    p.add_argument("--out-json", default="", help="write the run summary here")


def build_circuit(a) -> cc.CircuitProgram:
    """qcsim.cpp:72-114."""
    if a.circuit == "builtin:qft":
        if a.qubits < 1:
            raise ValueError("builtin:qft needs --qubits")
        return cc.build_qft(a.qubits)
    if a.circuit == "builtin:grover":
        if a.qubits < 1:
            raise ValueError("builtin:grover needs --qubits")
        return cc.build_grover(a.qubits, a.marked, a.iterations)
    if a.circuit == "builtin:random":
        if a.qubits < 1:
            raise ValueError("builtin:random needs --qubits")
        return cc.build_random(a.qubits, a.gates, a.seed)
    if a.circuit.startswith("builtin:"):
        raise ValueError(f"unknown builtin circuit '{a.circuit}'")
    try:
        with open(a.circuit) as f:
            text = f.read()
    except OSError:
        raise ValueError(f"cannot open circuit file '{a.circuit}'") from None
    prog = cc.parse_circuit(text, os.path.basename(a.circuit))
    if a.qubits > 0 and a.qubits != prog.n_qubits:
        raise ValueError(f"--qubits disagrees with circuit file ({prog.n_qubits})")
    return prog


def _geometry(q, prog, a):
    if a.stride_bits < 0:
        return q.StateGeometry.with_default_stride(prog.n_qubits)
    return q.StateGeometry.make(prog.n_qubits, a.stride_bits)


def _write(path, text):
    try:
        with open(path, "w") as f:
            f.write(text)
    except OSError as e:
        raise RuntimeError(f"cannot open '{path}' for writing") from e


def print_summary(prog, geom, theta, s: mm.RunSummary, final_bytes: int):
    """qcsim.cpp:137-164."""
    print(f"circuit:              {prog.name} ({len(prog.gates)} gates, {prog.n_qubits} qubits)")
    print(f"raw state bytes:      {16 << geom.n_qubits}")
    print(f"strides:              {geom.n_strides()} x {geom.stride_len()} amplitudes")
    print(f"theta:                {theta:g}")
    print(f"overall min ratio:    {s.overall_min_ratio:.6g}")
    print(f"qubit gain:           {s.qubit_gain}")
    print(f"threshold violations: {s.threshold_violations}")
    print(f"final state bytes:    {final_bytes}")
    print(f"total time:           {s.total_elapsed_ns * 1e-9:.3f} s")
    if s.fidelity is not None:
        print(f"fidelity:             {s.fidelity:.8f}")
    if s.overhead_factor is not None:
        print(f"overhead factor:      {s.overhead_factor:.2f}x")


def run_simulate(a) -> int:
    """qcsim.cpp:175-219."""
    import paper_1811_05140_b200 as q
    prog = build_circuit(a)
    geom = _geometry(q, prog, a)
    ladder = q.ErrorBoundLadder.parse(a.ladder)
    theta = q.RatioThreshold(a.theta)
    opts = q.RunOptions(basis=a.basis, workers=a.workers, first_gate=a.start_gate,
                        stop_after=None if a.stop_after < 0 else a.stop_after, device=a.device)
    if a.load_state:
        st, fp = q.CompressedState.load(a.load_state, geom, a.device)
        if fp != ladder.fingerprint():
            print("warning: checkpoint was written with a different error-bound ladder", file=sys.stderr)
        res = q.run_program_on(st, prog, ladder, theta, opts)
    else:
        res = q.run_program(prog, ladder, theta, geom, opts)
    if a.save_state:
        res.state.save(a.save_state, ladder.fingerprint())
    s = mm.summarize_run(res.metrics)
    if a.out_csv:
        _write(a.out_csv, mm.emit_csv(res.metrics.records))
    if a.out_json:
        _write(a.out_json, mm.emit_summary_json(s))
    print_summary(prog, geom, theta.theta, s, res.state.compressed_bytes())
    return 0


def _compressed_vs_dense(q, prog, a, geom, ladder, theta, guard):
    import torch
    from . import dense
    if prog.n_qubits > guard:
        raise ValueError(f"dense reference guard exceeded: {prog.n_qubits} qubits > {guard} (raise --max-dense)")
    torch.cuda.synchronize(a.device)
    t0 = time.perf_counter_ns()
    ref = dense.run_dense(prog, a.basis, guard, a.device)
    torch.cuda.synchronize(a.device)
    ref_ns = time.perf_counter_ns() - t0
    res = q.run_program(prog, ladder, theta, geom, q.RunOptions(basis=a.basis, workers=a.workers, device=a.device))
    comp = torch.from_numpy(res.state.to_amplitudes()).to(a.device)
    return ref, ref_ns, res, comp, dense.fidelity(ref, comp)


def run_compare(a) -> int:
    """qcsim.cpp:227-277."""
    import paper_1811_05140_b200 as q
    import torch
    prog = build_circuit(a)
    geom = _geometry(q, prog, a)
    ladder = q.ErrorBoundLadder.parse(a.ladder)
    theta = q.RatioThreshold(a.theta)
    ref, ref_ns, res, comp, fid = _compressed_vs_dense(q, prog, a, geom, ladder, theta, a.max_dense)
    s = mm.summarize_run(res.metrics, fid, ref_ns)
    if a.out_csv:
        _write(a.out_csv, mm.emit_csv(res.metrics.records))
    if a.out_json:
        _write(a.out_json, mm.emit_summary_json(s))
    print_summary(prog, geom, theta.theta, s, res.state.compressed_bytes())
    print(f"reference time:       {ref_ns * 1e-9:.3f} s")
    print(f"reference norm:       {float(torch.linalg.vector_norm(ref)):.12f}")
    print(f"compressed norm:      {float(torch.linalg.vector_norm(comp)):.12f}")
    return 0


def run_bench(a) -> int:
    """qcsim.cpp:286-343: one CSV row per theta."""
    import paper_1811_05140_b200 as q
    from . import dense
    thetas = [float(x) for x in a.thetas.split(",") if x]
    if not thetas:
        raise ValueError("--thetas must list at least one threshold")
    prog = build_circuit(a)
    if prog.n_qubits > a.max_dense:
        raise ValueError("dense reference guard exceeded")
    geom = _geometry(q, prog, a)
    ladder = q.ErrorBoundLadder.parse(a.ladder)
    import torch
    ref = dense.run_dense(prog, a.basis, a.max_dense, a.device)
    csv = "theta,min_ratio,fidelity,time_ns\n"
    print(f"{'theta':>10} {'min_ratio':>14} {'fidelity':>12} {'time_s':>12}")
    for th in thetas:
        res = q.run_program(prog, ladder, q.RatioThreshold(th), geom,
                            q.RunOptions(basis=a.basis, workers=a.workers, device=a.device))
        comp = torch.from_numpy(res.state.to_amplitudes()).to(a.device)
        fid = dense.fidelity(ref, comp)
        mr = res.metrics.overall_min_ratio()
        csv += f"{th:.17g},{mr:.17g},{fid:.17g},{res.metrics.total_elapsed_ns}\n"
        print(f"{th:10g} {mr:14.5g} {fid:12.8f} {res.metrics.total_elapsed_ns * 1e-9:12.3f}")
    if a.out_csv:
        _write(a.out_csv, csv)
    return 0


def run_codec(a) -> int:
    """qcsim.cpp:351-391: compress (codec plugin on the GPU) and decompress a
    raw little-endian double file."""
    import numpy as np
    import paper_1811_05140_b200 as q
    try:
        with open(a.input, "rb") as f:
            raw = f.read()
    except OSError:
        raise ValueError(f"cannot open input file '{a.input}'") from None
    if len(raw) % 8:
        raise ValueError("input length is not a multiple of 8 bytes")
    x = np.frombuffer(raw, dtype="<f8").copy()
    blk = q.compress(x, a.delta)
    back = q.decompress(blk, x.size)
    err = float(np.max(np.abs(back - x))) if x.size else 0.0
    print(f"scalars:          {x.size}")
    print(f"input bytes:      {len(raw)}")
    print(f"compressed bytes: {len(blk)}")
    print(f"ratio:            {len(raw) / len(blk):.6g}")
    print(f"max error:        {err:.17g}")
    if a.output:
        try:
            with open(a.output, "wb") as f:
                f.write(back.astype("<f8").tobytes())
        except OSError as e:
            raise RuntimeError(f"cannot open '{a.output}' for writing") from e
    return 0


def main(argv=None) -> int:
    ap = _Parser(prog="qcsim-b200", description="state-vector quantum circuit simulation on a compressed "
                                                "amplitude vector (B200 engine)")
    ap.add_argument("--version", action="version", version="qcsim-b200 0.2.0")
    sub = ap.add_subparsers(dest="cmd", parser_class=_Parser)
    sp = sub.add_parser("simulate", help="run the adaptive-compression pipeline")
    _add_circuit(sp)
    _add_pipeline(sp)
    sp.add_argument("--load-state", default="", help="resume from a saved state")
    sp.add_argument("--save-state", default="", help="save the final state here")
    sp.add_argument("--stop-after", type=int, default=-1, help="apply only the first N gates")
    sp.add_argument("--start-gate", type=int, default=0, help="skip gates before this index (resume)")
    cp = sub.add_parser("compare", help="run compressed and dense pipelines, report fidelity")
    _add_circuit(cp)
    _add_pipeline(cp)
    cp.add_argument("--max-dense", type=int, default=26, help="dense reference qubit guard")
    bp = sub.add_parser("bench", help="sweep ratio thresholds, one CSV row per theta")
    _add_circuit(bp)
    _add_pipeline(bp)
    bp.add_argument("--thetas", required=True, help="comma-separated thresholds")
    bp.add_argument("--max-dense", type=int, default=26, help="dense reference qubit guard")
    xp = sub.add_parser("codec", help="round-trip a raw little-endian double file")
    xp.add_argument("--input", required=True, help="raw double file")
    xp.add_argument("--output", default="", help="write round-tripped doubles here")
    xp.add_argument("--delta", type=float, default=0.0, help="error bound, 0 = lossless")
    a = ap.parse_args(argv)
    if a.cmd is None:
        ap.error("a subcommand is required")
    fn = {"simulate": run_simulate, "compare": run_compare, "bench": run_bench, "codec": run_codec}[a.cmd]
    try:
        return fn(a)
    except (ValueError, IndexError) as e:  # invalid_argument / out_of_range / ParseError
        print(f"error: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # noqa: BLE001 - runtime failures exit 1 (qcsim.cpp:465-468)
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
