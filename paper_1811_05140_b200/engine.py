"""Host-side mirror of the reference engine API over the C-ABI.

Mirrors /root/reference/proj/include/qcs/aalc.hpp and codec.hpp: same names,
argument meaning and error behaviour (C++ exceptions map to Python ones:
std::invalid_argument -> ValueError, std::out_of_range -> IndexError,
CodecError / CheckpointError keep their ``kind``).  Every computation runs
in libqcs_b200.so on the GPU; this module only marshals arguments.  There is
no CPU path: if the CUDA library or a device is missing, calls raise.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import struct
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from .circuit import CircuitProgram, GateOp, pack_gates
from .metrics import GateRecord, RunMetrics

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libqcs_b200.so")

HEADER_BYTES = 29  # codec.hpp:54


class CodecError(RuntimeError):
    """codec.hpp:34-52."""
    KINDS = {10: "bad_magic", 11: "truncated", 12: "unknown_codec", 13: "bad_value"}

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.kind = self.KINDS.get(code, "bad_value")


class CheckpointError(RuntimeError):
    """aalc.hpp:71-90."""

    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind


class DeviceError(RuntimeError):
    pass


_lib_handle = None


def lib() -> C.CDLL:
    global _lib_handle
    if _lib_handle is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(f"{LIB_PATH} is not built (run __graft_entry__.build()); "
                              "the engine has no CPU fallback")
        L = C.CDLL(LIB_PATH)
        L.qcs_last_error.restype = C.c_char_p
        L.qcs_state_launches.restype = C.c_uint64
        L.qcs_state_create.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, C.POINTER(C.c_void_p)]
        L.qcs_state_destroy.argtypes = [C.c_void_p]
        L.qcs_apply_gate_ex.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_double), C.c_int,
                                        C.c_double, C.c_int, C.POINTER(C.c_double), C.c_void_p,
                                        C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
        L.qcs_stride_norms.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.qcs_stride_sums.argtypes = [C.c_void_p, C.c_void_p]
        L.qcs_scale_all.argtypes = [C.c_void_p, C.c_double]
        L.qcs_pack_strides.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_uint64,
                                       C.POINTER(C.c_uint64)]
        L.qcs_pack_strides_range.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_uint64,
                                             C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]
        L.qcs_unpack_strides.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64]
        L.qcs_apply_gate.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_double), C.c_int,
                                     C.c_double, C.c_void_p, C.POINTER(C.c_uint64),
                                     C.POINTER(C.c_double)]
        L.qcs_run_program.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                      C.POINTER(C.c_double), C.c_int, C.c_double, C.c_void_p,
                                      C.POINTER(C.c_uint64)]
        L.qcs_read_stride.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p]
        L.qcs_read_strides_device.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_int, C.c_void_p]
        L.qcs_to_amplitudes.argtypes = [C.c_void_p, C.c_void_p]
        L.qcs_load_strides_device.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p,
                                              C.POINTER(C.c_double), C.c_int, C.c_double]
        L.qcs_state_stats.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_double),
                                      C.POINTER(C.c_double)]
        L.qcs_stride_info.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_double),
                                      C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                                      C.POINTER(C.c_uint64)]
        L.qcs_export_blocks.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64,
                                        C.POINTER(C.c_uint64), C.POINTER(C.c_double),
                                        C.POINTER(C.c_double)]
        L.qcs_import_blocks.argtypes = [C.c_void_p, C.c_uint64, C.c_char_p, C.c_uint64,
                                        C.c_double, C.c_double]
        L.qcs_state_memory.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                       C.POINTER(C.c_uint64)]
        L.qcs_state_launches.argtypes = [C.c_void_p]
        L.qcs_state_counters.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
        L.qcs_state_profile.argtypes = [C.c_void_p, C.c_int]
        L.qcs_state_kernel_time.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_double),
                                            C.POINTER(C.c_uint64)]
        L.qcs_codec_compress.argtypes = [C.c_void_p, C.c_uint64, C.c_double, C.c_void_p,
                                         C.c_uint64, C.POINTER(C.c_uint64)]
        L.qcs_codec_decompress.argtypes = [C.c_char_p, C.c_uint64, C.c_void_p, C.c_uint64]
        _lib_handle = L
    return _lib_handle


def _raise(rc: int):
    msg = lib().qcs_last_error().decode()
    if rc == 2:
        raise ValueError(msg)
    if rc == 3:
        raise IndexError(msg)
    if rc in CodecError.KINDS:
        raise CodecError(rc, msg)
    if rc in (5, 6):
        raise DeviceError(msg)
    raise RuntimeError(msg)


def _check(rc: int):
    if rc:
        _raise(rc)


class Report(C.Structure):
    _fields_ = [("stride_index", C.c_uint64), ("bytes_in", C.c_uint64), ("bytes_out", C.c_uint64),
                ("chosen_delta", C.c_double), ("ratio", C.c_double),
                ("threshold_met", C.c_int32), ("pad_", C.c_int32)]


class Record(C.Structure):
    _fields_ = [("gate_index", C.c_uint64), ("stride_count", C.c_uint64),
                ("min_ratio", C.c_double), ("mean_ratio", C.c_double),
                ("max_chosen_delta", C.c_double), ("bytes_before", C.c_uint64),
                ("bytes_after", C.c_uint64), ("elapsed_ns", C.c_uint64),
                ("norm_after", C.c_double), ("threshold_violations", C.c_uint64),
                ("compressed_in", C.c_uint64)]


# ---------------------------------------------------------------------------
# geometry, ladder, threshold (core.hpp:26-50, aalc.hpp:34-60)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class StateGeometry:
    n_qubits: int
    stride_bits: int

    @staticmethod
    def make(n_qubits: int, stride_bits: int) -> "StateGeometry":
        if n_qubits < 1 or n_qubits > 59:
            raise ValueError(f"n_qubits must be in [1, 59], got {n_qubits}")
        if stride_bits < 0 or stride_bits > n_qubits:
            raise ValueError(f"stride_bits must be in [0, n_qubits], got {stride_bits}")
        return StateGeometry(n_qubits, stride_bits)

    @staticmethod
    def with_default_stride(n_qubits: int) -> "StateGeometry":
        return StateGeometry.make(n_qubits, n_qubits if n_qubits < 20 else 20)

    def n_amplitudes(self) -> int:
        return 1 << self.n_qubits

    def stride_len(self) -> int:
        return 1 << self.stride_bits

    def n_strides(self) -> int:
        return 1 << (self.n_qubits - self.stride_bits)


@dataclass(frozen=True)
class ErrorBoundLadder:
    bounds: tuple

    @staticmethod
    def make(bounds: Sequence[float]) -> "ErrorBoundLadder":
        """aalc.cpp:56-72."""
        b = [float(x) for x in bounds]
        if not b:
            raise ValueError("error-bound ladder must not be empty")
        for i, x in enumerate(b):
            if not (x >= 0.0) or not math.isfinite(x):
                raise ValueError("error bounds must be finite and >= 0")
            if i > 0 and not (x > b[i - 1]):
                raise ValueError("error bounds must be strictly increasing")
        return ErrorBoundLadder(tuple(b))

    @staticmethod
    def lossless_only() -> "ErrorBoundLadder":
        return ErrorBoundLadder.make([0.0])

    @staticmethod
    def default_ladder() -> "ErrorBoundLadder":
        return ErrorBoundLadder.make([0.0, 1e-7, 1e-6, 1e-5, 1e-4, 1e-3])

    @staticmethod
    def parse(text: str) -> "ErrorBoundLadder":
        out = []
        for item in text.split(","):
            try:
                out.append(float(item))
            except ValueError:
                raise ValueError(f"malformed error bound '{item}'") from None
        return ErrorBoundLadder.make(out)

    def fingerprint(self) -> int:
        """FNV-1a over the bound bytes (aalc.cpp:103-115)."""
        h = 0xCBF29CE484222325
        for b in self.bounds:
            for byte in struct.pack("<d", b):
                h ^= byte
                h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
        return h

    def c_array(self):
        return (C.c_double * len(self.bounds))(*self.bounds)


@dataclass(frozen=True)
class RatioThreshold:
    theta: float = 1.0

    def __post_init__(self):
        if not (self.theta >= 1.0):
            raise ValueError("ratio threshold must be >= 1")


@dataclass
class StrideCompressReport:
    stride_index: int
    chosen_delta: float
    ratio: float
    bytes_in: int
    bytes_out: int
    threshold_met: bool

    def as_tuple(self):
        return (self.stride_index, self.chosen_delta, self.ratio, self.bytes_in, self.bytes_out,
                self.threshold_met)


@dataclass
class GateResult:
    reports: List[StrideCompressReport] = field(default_factory=list)
    norm_after: float = 0.0


# ---------------------------------------------------------------------------
# codec plugin (codec.hpp:80-105)
# ---------------------------------------------------------------------------
def compress(x: np.ndarray, delta: float) -> bytes:
    """serialize_block(compress(x, ErrorBound(delta))) computed on the GPU."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    n = C.c_uint64()
    _check(lib().qcs_codec_compress(x.ctypes.data, x.size, float(delta), None, 0, C.byref(n)))
    buf = C.create_string_buffer(max(1, n.value))
    _check(lib().qcs_codec_compress(x.ctypes.data, x.size, float(delta), buf, n.value, C.byref(n)))
    return buf.raw[: n.value]


def decompress(block: bytes, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    _check(lib().qcs_codec_decompress(block, len(block), out.ctypes.data, n))
    return out


# ---------------------------------------------------------------------------
# CompressedState (aalc.hpp:104-175)
# ---------------------------------------------------------------------------
class CompressedState:
    def __init__(self, handle: C.c_void_p, geom: StateGeometry):
        self._h = handle
        self._geom = geom

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib_handle is not None:
            _lib_handle.qcs_state_destroy(h)
            self._h = None

    @staticmethod
    def basis_state(geom: StateGeometry, basis_index: int, device: int = 0) -> "CompressedState":
        if basis_index >= geom.n_amplitudes() or basis_index < 0:
            raise IndexError("basis index out of range")
        h = C.c_void_p()
        _check(lib().qcs_state_create(geom.n_qubits, geom.stride_bits, basis_index, device,
                                      C.byref(h)))
        return CompressedState(h, geom)

    def geometry(self) -> StateGeometry:
        return self._geom

    def apply_gate(self, gate: GateOp, ladder: ErrorBoundLadder,
                   theta: RatioThreshold = RatioThreshold(), workers: int = 0) -> GateResult:
        """Full decompress-normalize-compute-compress cycle (aalc.cpp:261-420).
        ``workers`` is accepted for signature parity; results never depend on it."""
        gate.validate(self._geom.n_qubits)
        desc = pack_gates([gate])
        reps = (Report * self._geom.n_strides())()
        nr = C.c_uint64()
        norm = C.c_double()
        _check(lib().qcs_apply_gate(self._h, desc, ladder.c_array(), len(ladder.bounds),
                                    theta.theta, reps, C.byref(nr), C.byref(norm)))
        out = [StrideCompressReport(r.stride_index, r.chosen_delta, r.ratio, r.bytes_in,
                                    r.bytes_out, bool(r.threshold_met))
               for r in reps[: nr.value]]
        return GateResult(out, norm.value)

    def _stride(self, j: int, scale: bool):
        L = self._geom.stride_len()
        re = np.empty(L, dtype=np.float64)
        im = np.empty(L, dtype=np.float64)
        _check(lib().qcs_read_stride(self._h, j, 1 if scale else 0, re.ctypes.data,
                                     im.ctypes.data))
        return re, im

    def stored_stride(self, j: int):
        return self._stride(j, False)

    def decompress_stride(self, j: int):
        return self._stride(j, True)

    def read_strides_device(self, first: int, count: int, out_ptr: int, apply_scale: bool = True):
        """Decode strides [first, first+count) into a device buffer (e.g. a
        torch.float64 CUDA tensor's data_ptr()) laid out [stride][re|im][L]."""
        _check(lib().qcs_read_strides_device(self._h, first, count, int(apply_scale), out_ptr))

    def load_strides_device(self, first: int, count: int, planes_ptr: int, ladder: ErrorBoundLadder,
                            theta: RatioThreshold = RatioThreshold()) -> None:
        """Replace strides [first, first+count) by the compression of device
        planes [stride][re|im][L] (snapped in place first, like
        compress_stride_adaptive, aalc.cpp:117-138)."""
        _check(lib().qcs_load_strides_device(self._h, first, count, planes_ptr, ladder.c_array(),
                                             len(ladder.bounds), theta.theta))

    def to_amplitudes(self) -> np.ndarray:
        a = np.empty(2 * self._geom.n_amplitudes(), dtype=np.float64)
        _check(lib().qcs_to_amplitudes(self._h, a.ctypes.data))
        return a.view(np.complex128)

    def _stats(self):
        b, r, q = C.c_uint64(), C.c_double(), C.c_double()
        _check(lib().qcs_state_stats(self._h, C.byref(b), C.byref(r), C.byref(q)))
        return b.value, r.value, q.value

    def compressed_bytes(self) -> int:
        return self._stats()[0]

    def min_stride_ratio(self) -> float:
        return self._stats()[1]

    def norm_sq_tracked(self) -> float:
        return self._stats()[2]

    def stride_info(self, j: int):
        sc, ss, a, b = C.c_double(), C.c_double(), C.c_uint64(), C.c_uint64()
        _check(lib().qcs_stride_info(self._h, j, C.byref(sc), C.byref(ss), C.byref(a), C.byref(b)))
        return sc.value, ss.value, a.value, b.value

    def stride_scale(self, j: int) -> float:
        if j < 0 or j >= self._geom.n_strides():
            raise IndexError("stride index out of range")
        return self.stride_info(j)[0]

    def export_blocks(self, j: int):
        n, sc, ss = C.c_uint64(), C.c_double(), C.c_double()
        _check(lib().qcs_export_blocks(self._h, j, None, 0, C.byref(n), C.byref(sc), C.byref(ss)))
        buf = C.create_string_buffer(n.value)
        _check(lib().qcs_export_blocks(self._h, j, buf, n.value, C.byref(n), C.byref(sc),
                                       C.byref(ss)))
        return buf.raw[: n.value], sc.value, ss.value

    KERNEL_CLASSES = ("decode", "serial_chain", "fused", "commit", "mean", "bookkeeping")

    def profile(self, enable) -> None:
        """False/0 off, True/1 every kernel class, 2 the encoder class only."""
        _check(lib().qcs_state_profile(self._h, 2 if enable == 2 else (1 if enable else 0)))

    def kernel_times(self) -> dict:
        out = {}
        for i, name in enumerate(self.KERNEL_CLASSES):
            t, n = C.c_double(), C.c_uint64()
            _check(lib().qcs_state_kernel_time(self._h, i, C.byref(t), C.byref(n)))
            out[name] = (t.value, n.value)
        return out

    def counters(self) -> dict:
        buf = (C.c_uint64 * 24)()
        _check(lib().qcs_state_counters(self._h, buf, 24))
        return {"repaired_lanes": buf[0], "sum_passes": buf[1], "slid_bytes": buf[2],
                "serial_fallback_lanes": buf[3], "compactions": buf[4], "wave_slots": buf[5],
                "sum_tie_events": buf[6], "sum_crossing_events": buf[7], "ladder_exits": buf[15],
                "compaction_ns": buf[14], "stream_left_slots": buf[17], "stream_slots": buf[18],
                "stream_left_why": {k: buf[19 + i] for i, k in enumerate(
                    ("input_not_staged", "unproven_step", "first_element", "sum_head", "sum_event"))},
                "phase_cycles": {k: buf[8 + i] for i, k in enumerate(
                    ("input", "rounds", "final", "sum", "tokcount", "write"))}}

    def launches(self) -> int:
        return lib().qcs_state_launches(self._h)

    def memory(self):
        a, s, x = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(lib().qcs_state_memory(self._h, C.byref(a), C.byref(s), C.byref(x)))
        return a.value, s.value, x.value

    # ---- QCKP v1 checkpoints (aalc.cpp:422-586), byte-compatible ----------
    def save(self, path: str, ladder_fingerprint: int) -> None:
        g = self._geom
        out = bytearray(b"QCKP")
        out += struct.pack("<BIIQQ", 1, g.n_qubits, g.stride_bits, ladder_fingerprint,
                           g.n_strides())
        for j in range(g.n_strides()):
            blocks, sc, ss = self.export_blocks(j)
            out += struct.pack("<dd", sc, ss)
            out += blocks
        try:
            with open(path, "wb") as f:
                f.write(out)
        except OSError as e:
            raise CheckpointError("io", f"cannot open '{path}' for writing") from e

    @staticmethod
    def load(path: str, expected: Optional[StateGeometry] = None, device: int = 0):
        """Returns (state, ladder_fingerprint) (LoadedState, aalc.hpp:177-180)."""
        try:
            with open(path, "rb") as f:
                data = f.read()
        except OSError as e:
            raise CheckpointError("io", f"cannot open '{path}' for reading") from e
        if len(data) < 4 or data[:4] != b"QCKP":
            raise CheckpointError("bad_magic", "not a checkpoint file")
        if len(data) < 29:
            raise CheckpointError("truncated", "checkpoint shorter than its header")
        if data[4] != 1:
            raise CheckpointError("version_mismatch", f"unsupported checkpoint version {data[4]}")
        n, s, fp, ns = struct.unpack_from("<IIQQ", data, 5)
        try:
            geom = StateGeometry.make(n, s)
        except ValueError as e:
            raise CheckpointError("geometry_mismatch", str(e)) from None
        if ns != geom.n_strides():
            raise CheckpointError("geometry_mismatch", "stride count disagrees with geometry")
        if expected is not None and (expected.n_qubits != n or expected.stride_bits != s):
            raise CheckpointError("geometry_mismatch",
                                  f"checkpoint holds {n} qubits at {s} stride bits, expected "
                                  f"{expected.n_qubits}/{expected.stride_bits}")
        st = CompressedState.basis_state(geom, 0, device)
        off = 29
        for j in range(ns):
            if off + 16 > len(data):
                raise CheckpointError("truncated", "checkpoint ends inside stride header")
            sc, ss = struct.unpack_from("<dd", data, off)
            off += 16
            start = off
            for _ in range(2):
                if off + HEADER_BYTES > len(data):
                    raise CheckpointError("truncated", "corrupt checkpoint: block header extends past end of data")
                if data[off:off + 4] != b"QCS1":
                    raise CheckpointError("bad_magic", "corrupt checkpoint: bad block magic")
                plen = struct.unpack_from("<Q", data, off + 21)[0]
                cnt = struct.unpack_from("<Q", data, off + 13)[0]
                if data[off + 4] not in (0, 1):
                    raise CheckpointError("bad_magic", "corrupt checkpoint: unknown codec id")
                off += HEADER_BYTES
                if off + plen > len(data):
                    raise CheckpointError("truncated", "corrupt checkpoint: block payload extends past end of data")
                if cnt != geom.stride_len():
                    raise CheckpointError("geometry_mismatch", "block length disagrees with geometry")
                off += plen
            rc = lib().qcs_import_blocks(st._h, j, data[start:off], off - start, sc, ss)
            if rc:
                msg = lib().qcs_last_error().decode()
                kind = "truncated" if rc == 11 else "bad_magic"
                raise CheckpointError(kind, "corrupt checkpoint: " + msg)
        if off != len(data):
            raise CheckpointError("truncated", "trailing bytes after final stride")
        return st, fp


@dataclass
class RunOptions:
    basis: int = 0
    workers: int = 0
    first_gate: int = 0
    stop_after: Optional[int] = None
    device: int = 0


@dataclass
class RunResult:
    state: CompressedState
    metrics: RunMetrics


def apply_program_range(state: CompressedState, program: CircuitProgram, first: int, last: int,
                        ladder: ErrorBoundLadder, theta: RatioThreshold = RatioThreshold(),
                        workers: int = 0) -> RunMetrics:
    """aalc.cpp:588-634, batched: one device round trip for the whole range."""
    if last > len(program.gates) or first > last:
        raise IndexError("gate range outside program")
    metrics = RunMetrics()
    gates = program.gates[first:last]
    if not gates:
        return metrics
    n = state.geometry().n_qubits
    for i, g in enumerate(gates):
        try:
            g.validate(n)
        except (ValueError, IndexError) as e:
            if i:
                sub = apply_program_range(state, program, first, first + i, ladder, theta)
                metrics.records += sub.records
            raise RuntimeError(f"gate {first + i} ({g.label}) failed: {e}") from e
    desc = pack_gates(gates)
    recs = (Record * len(gates))()
    done = C.c_uint64()
    rc = lib().qcs_run_program(state._h, desc, len(gates), first, ladder.c_array(),
                               len(ladder.bounds), theta.theta, recs, C.byref(done))
    for i in range(done.value):
        r = recs[i]
        metrics.records.append(GateRecord(
            gate_index=first + i, gate_label=gates[i].label, stride_count=r.stride_count,
            min_ratio=r.min_ratio, mean_ratio=r.mean_ratio, max_chosen_delta=r.max_chosen_delta,
            bytes_before=r.bytes_before, bytes_after=r.bytes_after, elapsed_ns=r.elapsed_ns,
            norm_after=r.norm_after))
        metrics.records[-1].compressed_in = r.compressed_in
        metrics.threshold_violations += r.threshold_violations
        metrics.total_elapsed_ns += r.elapsed_ns
    if rc:
        msg = lib().qcs_last_error().decode()
        raise RuntimeError(msg)
    return metrics


def run_program_on(state: CompressedState, program: CircuitProgram, ladder: ErrorBoundLadder,
                   theta: RatioThreshold = RatioThreshold(),
                   options: RunOptions = RunOptions()) -> RunResult:
    """aalc.cpp:653-676."""
    if program.n_qubits != state.geometry().n_qubits:
        raise ValueError("program and state disagree on qubits")
    last = len(program.gates) if options.stop_after is None else min(options.stop_after,
                                                                        len(program.gates))
    m = RunMetrics()
    m.init_min_ratio = state.min_stride_ratio()
    m.init_bytes = state.compressed_bytes()
    gm = apply_program_range(state, program, options.first_gate, last, ladder, theta)
    m.records = gm.records
    m.threshold_violations = gm.threshold_violations
    m.total_elapsed_ns += gm.total_elapsed_ns
    return RunResult(state, m)


def run_program(program: CircuitProgram, ladder: ErrorBoundLadder, theta: RatioThreshold,
                geom: StateGeometry, options: RunOptions = RunOptions()) -> RunResult:
    """aalc.cpp:636-651."""
    if program.n_qubits != geom.n_qubits:
        raise ValueError("program and geometry disagree on qubits")
    t0 = time.perf_counter_ns()
    st = CompressedState.basis_state(geom, options.basis, options.device)
    init_ns = time.perf_counter_ns() - t0
    r = run_program_on(st, program, ladder, theta, options)
    r.metrics.total_elapsed_ns += init_ns
    return r


# ---------------------------------------------------------------------------
# sharded state driven by the C++ cluster driver (qcs_cluster_*, include/qcs_b200.h)
# ---------------------------------------------------------------------------
class Cluster:
    """n qubits sharded over 2^rank_bits engine states (rank = top qubits),
    exchanges by NCCL send/recv (backend "nccl": one device per rank) or device
    copies (backend "loopback": ranks may share a GPU); renormalisation,
    reflect_mean's mean and the GateRecords are folded on the device in the
    reference's global order (bit-identical to one state)."""

    BACKENDS = {"loopback": 0, "nccl": 1}

    def __init__(self, geom: StateGeometry, rank_bits: int, basis: int, devices: Sequence[int],
                 backend: str = "loopback"):
        L = lib()
        L.qcs_cluster_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.POINTER(C.c_int), C.c_int,
                                         C.c_int, C.POINTER(C.c_void_p)]
        L.qcs_cluster_destroy.argtypes = [C.c_void_p]
        L.qcs_cluster_set_schedule.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
        L.qcs_cluster_run_program.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                              C.POINTER(C.c_double), C.c_int, C.c_double, C.c_void_p,
                                              C.POINTER(C.c_uint64)]
        L.qcs_cluster_to_amplitudes.argtypes = [C.c_void_p, C.c_void_p]
        L.qcs_cluster_stats.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                        C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.qcs_cluster_shard.argtypes = [C.c_void_p, C.c_int]
        L.qcs_cluster_shard.restype = C.c_void_p
        self._geom = geom
        self.rank_bits = rank_bits
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        _check(L.qcs_cluster_create(geom.n_qubits, geom.stride_bits, rank_bits, basis, devs, len(devices),
                                    self.BACKENDS[backend], C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib_handle is not None:
            _lib_handle.qcs_cluster_destroy(h)
            self._h = None

    def set_schedule(self, program: CircuitProgram) -> None:
        desc = pack_gates(program.gates)
        _check(lib().qcs_cluster_set_schedule(self._h, desc, len(program.gates)))

    def apply_program_range(self, program: CircuitProgram, first: int, last: int, ladder: ErrorBoundLadder,
                            theta: RatioThreshold = RatioThreshold()) -> RunMetrics:
        gates = program.gates[first:last]
        metrics = RunMetrics()
        if not gates:
            return metrics
        desc = pack_gates(gates)
        recs = (Record * len(gates))()
        done = C.c_uint64()
        rc = lib().qcs_cluster_run_program(self._h, desc, len(gates), first, ladder.c_array(),
                                           len(ladder.bounds), theta.theta, recs, C.byref(done))
        for i in range(done.value):
            r = recs[i]
            metrics.records.append(GateRecord(
                gate_index=first + i, gate_label=gates[i].label, stride_count=r.stride_count,
                min_ratio=r.min_ratio, mean_ratio=r.mean_ratio, max_chosen_delta=r.max_chosen_delta,
                bytes_before=r.bytes_before, bytes_after=r.bytes_after, elapsed_ns=r.elapsed_ns,
                norm_after=r.norm_after))
            metrics.records[-1].compressed_in = r.compressed_in
            metrics.threshold_violations += r.threshold_violations
            metrics.total_elapsed_ns += r.elapsed_ns
        if rc:
            _raise(rc)
        return metrics

    def to_amplitudes(self) -> np.ndarray:
        a = np.empty(2 << self._geom.n_qubits, dtype=np.float64)
        _check(lib().qcs_cluster_to_amplitudes(self._h, a.ctypes.data))
        return a.view(np.complex128)

    def stats(self) -> dict:
        x, b, t, nsq = C.c_uint64(), C.c_uint64(), C.c_double(), C.c_double()
        _check(lib().qcs_cluster_stats(self._h, C.byref(x), C.byref(b), C.byref(t), C.byref(nsq)))
        return {"exchanges": x.value, "exchange_bytes": b.value, "exchange_s": t.value, "norm_sq": nsq.value}
