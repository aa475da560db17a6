"""B200-native compressed-state gate engine (arXiv 1811.05140 hot path).

The product is libqcs_b200.so (sm_100a CUDA + C++ host code behind the C-ABI
in include/qcs_b200.h).  This package is its host-side mirror of the
reference API: circuit front end (circuit.py), engine/codec bindings
(engine.py), per-gate metrics (metrics.py) and the qcsim-style command line
(cli.py, `python -m paper_1811_05140_b200`).
"""
from .circuit import (CircuitProgram, GateOp, ParseError, Unitary2x2, build_grid, build_grover,
                      build_grover_gate_form, build_qft, build_random, parse_circuit, pow2_bound,
                      print_circuit, survey_bound)
from .metrics import (GateRecord, RunMetrics, RunSummary, emit_csv, emit_summary_json, gate_record,
                      qubit_gain, summarize_run)
from .engine import (CheckpointError, Cluster, CodecError, CompressedState, DeviceError, ErrorBoundLadder,
                     GateResult, RatioThreshold, RunOptions, RunResult, StateGeometry,
                     apply_program_range, compress, decompress, run_program, run_program_on)

__all__ = [n for n in dir() if not n.startswith("_")]
