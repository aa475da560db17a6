"""ctypes bindings for the CPU checkers.  TEST INFRASTRUCTURE ONLY.

* ``Oracle``    — oracle/_build/libqcs_oracle.so, our plain-C restatement of
                  the reference path (oracle/qcs_oracle.c).
* ``Reference`` — oracle/_ref/libqcsref.so, the unmodified reference built
                  from /root/reference by oracle/Makefile (present in this
                  container; on the GPU box only if the prebuilt file travelled).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libqcs_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libqcsref.so")


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Gate(C.Structure):
    _fields_ = [("kind", C.c_int32), ("target", C.c_int32), ("control", C.c_int32),
                ("pad_", C.c_int32), ("flip_index", C.c_uint64), ("u", C.c_double * 8)]


class Report(C.Structure):
    _fields_ = [("stride_index", C.c_uint64), ("bytes_in", C.c_uint64),
                ("bytes_out", C.c_uint64), ("chosen_delta", C.c_double),
                ("ratio", C.c_double), ("threshold_met", C.c_int32), ("pad_", C.c_int32)]


def gate_struct(g) -> Gate:
    k, t, c, f, u = g.desc()
    s = Gate()
    s.kind, s.target, s.control, s.flip_index = k, t, c, f
    for i in range(8):
        s.u[i] = u[i]
    return s


def gate_array(gates) -> C.Array:
    arr = (Gate * max(1, len(gates)))()
    for i, g in enumerate(gates):
        arr[i] = gate_struct(g)
    return arr


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _u8ptr(a):
    return C.cast(C.c_char_p(a) if isinstance(a, bytes) else a.ctypes.data, C.POINTER(C.c_uint8))


def build_oracle() -> str:
    if not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-C", HERE, "oracle"], check=True, capture_output=True)
    return ORACLE_SO


class Oracle:
    """Our C restatement of the reference algorithm."""

    def __init__(self):
        lib = C.CDLL(build_oracle())
        self.lib = lib
        lib.qo_last_error.restype = C.c_char_p
        lib.qo_fidelity.restype = C.c_double
        lib.qo_state_create.argtypes = [C.c_int, C.c_int, C.c_uint64, C.POINTER(C.c_void_p)]
        lib.qo_state_destroy.argtypes = [C.c_void_p]
        lib.qo_apply_gate.argtypes = [C.c_void_p, C.POINTER(Gate), C.POINTER(C.c_double), C.c_int,
                                      C.c_double, C.POINTER(Report), C.POINTER(C.c_uint64),
                                      C.POINTER(C.c_double)]
        lib.qo_to_amplitudes.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
        lib.qo_stats.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_double),
                                 C.POINTER(C.c_double)]
        lib.qo_stride_info.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_double),
                                       C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                                       C.POINTER(C.c_uint64)]
        lib.qo_export_blocks.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_uint8), C.c_uint64,
                                         C.POINTER(C.c_uint64)]
        lib.qo_stored_stride.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.POINTER(C.c_double),
                                         C.POINTER(C.c_double)]
        lib.qo_apply_gate_ex.argtypes = [C.c_void_p, C.POINTER(Gate), C.POINTER(C.c_double),
                                         C.c_int, C.c_double, C.c_int, C.POINTER(C.c_double),
                                         C.POINTER(Report),
                                         C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
        lib.qo_stride_sums.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
        lib.qo_stride_norms.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        lib.qo_scale_all.argtypes = [C.c_void_p, C.c_double]
        lib.qo_import_blocks.argtypes = [C.c_void_p, C.c_uint64, C.c_char_p, C.c_uint64,
                                         C.c_double, C.c_double]

    def _check(self, rc: int):
        if rc:
            raise OracleError(rc, self.lib.qo_last_error().decode())

    # ---- codec ----
    def compress(self, x: np.ndarray, delta: float) -> bytes:
        x = np.ascontiguousarray(x, dtype=np.float64)
        n = C.c_uint64()
        self._check(self.lib.qo_compress(_dptr(x), C.c_uint64(x.size), C.c_double(delta), None,
                                         C.c_uint64(0), C.byref(n)))
        buf = (C.c_uint8 * max(1, n.value))()
        self._check(self.lib.qo_compress(_dptr(x), C.c_uint64(x.size), C.c_double(delta), buf,
                                         C.c_uint64(n.value), C.byref(n)))
        return bytes(buf)[: n.value]

    def decompress(self, blob: bytes, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        self._check(self.lib.qo_decompress(C.c_char_p(blob), C.c_uint64(len(blob)), _dptr(out),
                                           C.c_uint64(n)))
        return out

    # ---- dense ----
    def dense(self, n_qubits: int, gates, basis: int) -> np.ndarray:
        amps = np.empty(2 << n_qubits, dtype=np.float64)
        arr = gate_array(gates)
        self._check(self.lib.qo_dense_run(C.c_int(n_qubits), arr, C.c_uint64(len(gates)),
                                          C.c_uint64(basis), _dptr(amps)))
        return amps.view(np.complex128)

    def fidelity(self, a: np.ndarray, b: np.ndarray) -> float:
        a = np.ascontiguousarray(a, dtype=np.complex128)
        b = np.ascontiguousarray(b, dtype=np.complex128)
        return self.lib.qo_fidelity(_dptr(a.view(np.float64)), _dptr(b.view(np.float64)),
                                    C.c_uint64(a.size))

    # ---- engine ----
    def state(self, n_qubits: int, stride_bits: int, basis: int = 0) -> "OracleState":
        return OracleState(self, n_qubits, stride_bits, basis)


class OracleState:
    def __init__(self, o: Oracle, n: int, s: int, basis: int):
        self.o, self.n, self.s = o, n, s
        self.h = C.c_void_p()
        o._check(o.lib.qo_state_create(n, s, C.c_uint64(basis), C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None):
            self.o.lib.qo_state_destroy(self.h)
            self.h = None

    def apply_gate(self, g, ladder: Sequence[float], theta: float):
        lad = (C.c_double * len(ladder))(*ladder)
        reps = (Report * (1 << (self.n - self.s)))()
        nr = C.c_uint64()
        norm = C.c_double()
        gs = gate_struct(g)
        self.o._check(self.o.lib.qo_apply_gate(self.h, C.byref(gs), lad, len(ladder),
                                               C.c_double(theta), reps, C.byref(nr),
                                               C.byref(norm)))
        return [(r.stride_index, r.chosen_delta, r.ratio, r.bytes_in, r.bytes_out,
                 bool(r.threshold_met)) for r in reps[: nr.value]], norm.value

    def amplitudes(self) -> np.ndarray:
        a = np.empty(2 << self.n, dtype=np.float64)
        self.o._check(self.o.lib.qo_to_amplitudes(self.h, _dptr(a)))
        return a.view(np.complex128)

    def stats(self):
        b, r, q = C.c_uint64(), C.c_double(), C.c_double()
        self.o._check(self.o.lib.qo_stats(self.h, C.byref(b), C.byref(r), C.byref(q)))
        return b.value, r.value, q.value

    def stride_info(self, j: int):
        sc, ss, pr, pi = C.c_double(), C.c_double(), C.c_uint64(), C.c_uint64()
        self.o._check(self.o.lib.qo_stride_info(self.h, C.c_uint64(j), C.byref(sc), C.byref(ss),
                                                C.byref(pr), C.byref(pi)))
        return sc.value, ss.value, pr.value, pi.value

    def export_blocks(self, j: int) -> bytes:
        n = C.c_uint64()
        self.o._check(self.o.lib.qo_export_blocks(self.h, C.c_uint64(j), None, 0, C.byref(n)))
        buf = (C.c_uint8 * n.value)()
        self.o._check(self.o.lib.qo_export_blocks(self.h, C.c_uint64(j), buf, n.value, C.byref(n)))
        return bytes(buf)

    # ---- sharded-run hooks (shard interface of paper_1811_05140_b200.distributed) ----
    def apply(self, g, ladder: Sequence[float], theta: float, mean=None):
        lad = (C.c_double * len(ladder))(*ladder)
        reps = (Report * (1 << (self.n - self.s)))()
        nr = C.c_uint64()
        norm = C.c_double()
        gs = gate_struct(g)
        m = (C.c_double * 2)(*(mean or (0.0, 0.0)))
        self.o._check(self.o.lib.qo_apply_gate_ex(self.h, C.byref(gs), lad, len(ladder),
                                                  C.c_double(theta), 1 | (2 if mean else 0), m,
                                                  reps, C.byref(nr), C.byref(norm)))
        return [(r.stride_index, r.chosen_delta, r.ratio, r.bytes_in, r.bytes_out,
                 bool(r.threshold_met)) for r in reps[: nr.value]]

    def stride_sums(self) -> np.ndarray:
        p = np.empty(2 << (self.n - self.s))
        self.o._check(self.o.lib.qo_stride_sums(self.h, _dptr(p)))
        return p

    def stride_norms(self):
        ns = 1 << (self.n - self.s)
        sc, sm = np.empty(ns), np.empty(ns)
        self.o._check(self.o.lib.qo_stride_norms(self.h, _dptr(sc), _dptr(sm)))
        return sc, sm

    def scale_all(self, f: float):
        self.o._check(self.o.lib.qo_scale_all(self.h, C.c_double(f)))

    def export(self, j: int):
        sc, ss, _, _ = self.stride_info(j)
        return self.export_blocks(j), sc, ss

    def pack(self, bit: int, value: int, first: int = 0, count: int = 1 << 62):
        sel = [j for j in range(1 << (self.n - self.s)) if ((j >> bit) & 1) == value][first:first + count]
        return [(j, *self.export(j)) for j in sel]

    def image_bytes(self, bit: int, value: int) -> int:
        return sum(len(b) + 16 for _, b, _, _ in self.pack(bit, value))

    def unpack(self, payload, xor_mask: int):
        for (j, blob, sc, ss) in payload:
            self.import_(j ^ xor_mask, blob, sc, ss)

    def import_(self, j: int, blob: bytes, scale: float, ssq: float):
        self.o._check(self.o.lib.qo_import_blocks(self.h, C.c_uint64(j), blob, len(blob),
                                                  C.c_double(scale), C.c_double(ssq)))


class OracleBackend:
    """Local-shard factory for distributed.ShardedState on the CPU oracle."""

    def __init__(self, oracle: Optional[Oracle] = None):
        self.o = oracle or Oracle()

    def create(self, n: int, s: int, basis: Optional[int]):
        return OracleState(self.o, n, s, (1 << 64) - 1 if basis is None else basis)


class Reference:
    """The unmodified reference (oracle/_ref/libqcsref.so)."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self):
        lib = C.CDLL(REF_SO)
        self.lib = lib
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_run.argtypes = [C.c_char_p, C.c_int, C.c_uint64, C.POINTER(C.c_double), C.c_int,
                                C.c_double, C.c_int, C.c_int64, C.c_char_p, C.c_uint64,
                                C.POINTER(C.c_uint64), C.POINTER(C.c_double),
                                C.POINTER(C.c_double)]
        lib.ref_dense.argtypes = [C.c_char_p, C.c_uint64, C.POINTER(C.c_double)]
        lib.ref_builtin_circuit.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_char_p,
                                            C.c_uint64, C.POINTER(C.c_uint64)]

    def _check(self, rc: int):
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def _state_api(self):
        L = self.lib
        L.ref_state_create.restype = C.c_void_p
        L.ref_state_create.argtypes = [C.c_char_p, C.c_int, C.c_uint64]
        L.ref_state_from_tables.restype = C.c_void_p
        L.ref_state_from_tables.argtypes = [C.c_char_p, C.c_int] + [C.c_void_p] * 4 + [
            C.c_double, C.c_uint64, C.c_uint64, C.POINTER(C.c_double), C.c_int, C.c_double,
            C.c_char_p, C.c_int]
        L.ref_state_apply.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.POINTER(C.c_double),
                                      C.c_int, C.c_double, C.c_int, C.POINTER(C.c_double)]
        L.ref_state_apply_csv.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.POINTER(C.c_double),
                                          C.c_int, C.c_double, C.c_int, C.c_char_p, C.c_uint64,
                                          C.POINTER(C.c_uint64)]
        L.ref_state_amplitudes.argtypes = [C.c_void_p, C.c_void_p]
        L.ref_state_stats.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
        L.ref_state_destroy.argtypes = [C.c_void_p]

    def state(self, text: str, stride_bits: int, basis: int) -> "RefState":
        """CompressedState::basis_state of the circuit's geometry."""
        self._state_api()
        h = self.lib.ref_state_create(text.encode(), stride_bits, C.c_uint64(basis))
        if not h:
            raise OracleError(1, self.lib.ref_last_error().decode())
        return RefState(self, h)

    def state_from_tables(self, text: str, stride_bits: int, tables: dict, ladder: Sequence[float],
                          theta: float, path: str, workers: int = 0) -> "RefState":
        """A closed-form intermediate state (circuit.stage_tables) compressed by
        the reference's compress_stride_adaptive, written as a QCKP checkpoint
        at `path` and read back by CompressedState::load (oracle/ref_capi.cpp)."""
        self._state_api()
        arrs = [np.ascontiguousarray(tables[k], dtype=np.float64) for k in ("lo_re", "lo_im", "hi_re", "hi_im")]
        lad = (C.c_double * len(ladder))(*ladder)
        h = self.lib.ref_state_from_tables(text.encode(), stride_bits, *[a.ctypes.data for a in arrs],
                                           C.c_double(tables["amp"]), C.c_uint64(tables["zmask"]),
                                           C.c_uint64(tables["zval"]), lad, len(ladder), C.c_double(theta),
                                           path.encode(), workers)
        if not h:
            raise OracleError(1, self.lib.ref_last_error().decode())
        return RefState(self, h)

    def max_threads(self) -> int:
        return self.lib.ref_max_threads()

    def compress(self, x: np.ndarray, delta: float) -> bytes:
        x = np.ascontiguousarray(x, dtype=np.float64)
        n = C.c_uint64()
        self._check(self.lib.ref_codec_compress(_dptr(x), C.c_uint64(x.size), C.c_double(delta),
                                                None, C.c_uint64(0), C.byref(n)))
        buf = (C.c_uint8 * max(1, n.value))()
        self._check(self.lib.ref_codec_compress(_dptr(x), C.c_uint64(x.size), C.c_double(delta),
                                                buf, C.c_uint64(n.value), C.byref(n)))
        return bytes(buf)[: n.value]

    def decompress(self, blob: bytes, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        self._check(self.lib.ref_codec_decompress(C.c_char_p(blob), C.c_uint64(len(blob)),
                                                  _dptr(out), C.c_uint64(n)))
        return out

    def builtin(self, kind: int, n: int, arg: int = 0, iters: int = -1) -> str:
        ln = C.c_uint64()
        self._check(self.lib.ref_builtin_circuit(kind, n, C.c_uint64(arg), iters, None, 0,
                                                 C.byref(ln)))
        buf = C.create_string_buffer(ln.value + 1)
        self._check(self.lib.ref_builtin_circuit(kind, n, C.c_uint64(arg), iters, buf,
                                                 ln.value + 1, C.byref(ln)))
        return buf.value.decode()

    def run(self, text: str, stride_bits: int, basis: int, ladder: Sequence[float],
            theta: float, workers: int = 0, stop_after: int = -1, want_amps: bool = True,
            n_qubits: Optional[int] = None):
        if n_qubits is None:
            n_qubits = int(text.split()[1])
        lad = (C.c_double * len(ladder))(*ladder)
        summ = (C.c_double * 10)()
        amps = np.empty(2 << n_qubits, dtype=np.float64) if want_amps else None
        ln = C.c_uint64()
        cap = 256 * (text.count("\n") + 4) + 4096
        csv = C.create_string_buffer(cap)
        self._check(self.lib.ref_run(text.encode(), stride_bits, C.c_uint64(basis), lad,
                                     len(ladder), C.c_double(theta), workers,
                                     C.c_int64(stop_after), csv, cap, C.byref(ln),
                                     _dptr(amps) if amps is not None else None, summ))
        keys = ["loop_ns", "amp_updates", "init_min_ratio", "threshold_violations",
                "compressed_bytes", "min_stride_ratio", "norm_sq_tracked", "overall_min_ratio",
                "n_records", "wall_ns"]
        return (csv.value.decode(), amps.view(np.complex128) if amps is not None else None,
                dict(zip(keys, list(summ))))

    def dense(self, text: str, basis: int, n_qubits: int) -> np.ndarray:
        amps = np.empty(2 << n_qubits, dtype=np.float64)
        self._check(self.lib.ref_dense(text.encode(), C.c_uint64(basis), _dptr(amps)))
        return amps.view(np.complex128)


class RefState:
    """A persistent reference CompressedState (oracle/ref_capi.cpp)."""

    def __init__(self, ref: Reference, h):
        self.ref, self.h = ref, h

    def apply(self, first, last, ladder, theta, workers=0):
        """apply_program_range over gates [first, last): summed GateRecord
        elapsed_ns, amplitude updates, min ratio, last norm."""
        lad = (C.c_double * len(ladder))(*ladder)
        out = (C.c_double * 4)()
        self.ref._check(self.ref.lib.ref_state_apply(self.h, first, last, lad, len(ladder),
                                                     C.c_double(theta), workers, out))
        return dict(gate_ns=out[0], amp_updates=out[1], min_ratio=out[2], norm=out[3])

    def apply_csv(self, first, last, ladder, theta, workers=0) -> str:
        """apply_program_range, returning emit_csv of the records."""
        lad = (C.c_double * len(ladder))(*ladder)
        cap = 256 * (last - first) + 4096
        buf = C.create_string_buffer(cap)
        n = C.c_uint64()
        self.ref._check(self.ref.lib.ref_state_apply_csv(self.h, first, last, lad, len(ladder),
                                                         C.c_double(theta), workers, buf, cap, C.byref(n)))
        return buf.value.decode()

    def amplitudes(self, n_qubits: int) -> np.ndarray:
        a = np.empty(2 << n_qubits, dtype=np.float64)
        self.ref._check(self.ref.lib.ref_state_amplitudes(self.h, a.ctypes.data))
        return a.view(np.complex128)

    def stats(self):
        out = (C.c_double * 3)()
        self.ref.lib.ref_state_stats(self.h, out)
        return dict(compressed_bytes=out[0], min_ratio=out[1], norm_sq=out[2])

    def __del__(self):
        if self.h:
            self.ref.lib.ref_state_destroy(self.h)
            self.h = None
