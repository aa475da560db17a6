"""Circuit front end: gate alphabet, text format and builders.

Host-side mirror of the reference's circuit/gate front end, which SURVEY.md
§2 marks as reused host code that feeds ``GateOp`` into the boundary:

* ``Unitary2x2`` factories           — gate.cpp:29-56 (same libm calls, so
  the matrices are bit-identical to the reference's)
* ``GateOp`` + ``validate``          — gate.hpp:36-63, gate.cpp:58-137
* ``parse_circuit`` / ``print_circuit`` — circuit.cpp:101-272
* ``build_qft`` / ``build_grover``   — circuit.cpp:274-325
* ``build_grover_gate_form``         — BASELINE config 2 written with the
  primitives the reference text format has:
  H^n; iters x [flip m; H^n; flip 0; H^n].  X^n·MCZ·X^n = diag(-1,1,..,1)
  = ``flip 0`` exactly, so this is BASELINE's diffusion operator.
* ``build_grid``                     — seeded stand-in for BASELINE config 4
  (6x6 grid, CZ on nearest-neighbour pairs + {sqrt X, sqrt Y, T}); emitted
  in the reference text format so both engines parse the same file.  It is
  our own generator (SplitMix64), not any published circuit instance.

Qubit k is bit k of the amplitude index (core.hpp:13-15).
"""
from __future__ import annotations

import math
import struct
from dataclasses import dataclass, field
from typing import List, Optional

KIND_SINGLE, KIND_CONTROLLED, KIND_FLIP, KIND_REFLECT = 0, 1, 2, 3
_PI = math.acos(-1.0)          # circuit.cpp:13 (kPi = std::acos(-1.0))
_UNITARY_TOL = 1e-12           # gate.cpp:11


class ParseError(ValueError):
    """circuit.hpp:33-45: carries the 1-based offending line."""

    def __init__(self, line: int, msg: str):
        super().__init__(f"line {line}: {msg}")
        self.line = line


@dataclass(frozen=True)
class Unitary2x2:
    """2x2 unitary, checked U†U = I to 1e-12 elementwise (gate.cpp:13-33)."""
    u11: complex
    u12: complex
    u21: complex
    u22: complex

    def __post_init__(self):
        a11, a12, a21, a22 = self.u11, self.u12, self.u21, self.u22
        c11 = a11.conjugate() * a11 + a21.conjugate() * a21
        c12 = a11.conjugate() * a12 + a21.conjugate() * a22
        c21 = a12.conjugate() * a11 + a22.conjugate() * a21
        c22 = a12.conjugate() * a12 + a22.conjugate() * a22
        if (abs(c11 - 1.0) > _UNITARY_TOL or abs(c12) > _UNITARY_TOL
                or abs(c21) > _UNITARY_TOL or abs(c22 - 1.0) > _UNITARY_TOL):
            raise ValueError("matrix is not unitary within 1e-12")

    def parts(self) -> List[float]:
        """UnitaryParts order (gate.cpp:141-151)."""
        return [self.u11.real, self.u11.imag, self.u12.real, self.u12.imag,
                self.u21.real, self.u21.imag, self.u22.real, self.u22.imag]

    @staticmethod
    def identity():
        return Unitary2x2(1 + 0j, 0j, 0j, 1 + 0j)

    @staticmethod
    def hadamard():
        h = 1.0 / math.sqrt(2.0)
        return Unitary2x2(complex(h, 0), complex(h, 0), complex(h, 0), complex(-h, 0))

    @staticmethod
    def pauli_x():
        return Unitary2x2(0j, 1 + 0j, 1 + 0j, 0j)

    @staticmethod
    def pauli_y():
        return Unitary2x2(0j, complex(0, -1), complex(0, 1), 0j)

    @staticmethod
    def pauli_z():
        return Unitary2x2(1 + 0j, 0j, 0j, complex(-1, 0))

    @staticmethod
    def phase(theta: float):
        return Unitary2x2(1 + 0j, 0j, 0j, complex(math.cos(theta), math.sin(theta)))

    @staticmethod
    def s_gate():
        return Unitary2x2.phase(_PI / 2.0)

    @staticmethod
    def t_gate():
        return Unitary2x2.phase(_PI / 4.0)

    @staticmethod
    def sqrt_x():
        return Unitary2x2(complex(0.5, 0.5), complex(0.5, -0.5),
                          complex(0.5, -0.5), complex(0.5, 0.5))

    @staticmethod
    def sqrt_y():
        return Unitary2x2(complex(0.5, 0.5), complex(-0.5, -0.5),
                          complex(0.5, 0.5), complex(0.5, 0.5))


@dataclass
class GateOp:
    """gate.hpp:43-63."""
    kind: int = KIND_SINGLE
    unitary: Optional[Unitary2x2] = None
    target: int = 0
    control: Optional[int] = None
    flip_index: int = 0
    phase_theta: Optional[float] = None
    label: str = ""

    @staticmethod
    def single(u: Unitary2x2, target: int, label: str = "") -> "GateOp":
        return GateOp(KIND_SINGLE, u, target, None, 0, None, label)

    @staticmethod
    def controlled(u: Unitary2x2, control: int, target: int, label: str = "") -> "GateOp":
        if control == target:
            raise ValueError("control qubit equals target qubit")
        return GateOp(KIND_CONTROLLED, u, target, control, 0, None, label)

    @staticmethod
    def controlled_phase(theta: float, control: int, target: int, label: str = "") -> "GateOp":
        g = GateOp.controlled(Unitary2x2.phase(theta), control, target, label)
        g.phase_theta = theta
        return g

    @staticmethod
    def phase_flip(flip_index: int) -> "GateOp":
        return GateOp(KIND_FLIP, None, 0, None, int(flip_index), None, f"flip {flip_index}")

    @staticmethod
    def reflect_mean() -> "GateOp":
        return GateOp(KIND_REFLECT, None, 0, None, 0, None, "diffuse")

    def validate(self, n_qubits: int) -> None:
        """GateOp::validate (gate.cpp:109-137): IndexError = std::out_of_range,
        ValueError = std::invalid_argument."""
        if self.kind in (KIND_SINGLE, KIND_CONTROLLED):
            if self.target < 0 or self.target >= n_qubits:
                raise IndexError("target qubit out of range")
            if self.kind == KIND_CONTROLLED:
                if self.control is None or self.control < 0 or self.control >= n_qubits:
                    raise IndexError("control qubit out of range")
                if self.control == self.target:
                    raise ValueError("control qubit equals target qubit")
            if self.unitary is None:
                raise ValueError("gate is missing its unitary")
        elif self.kind == KIND_FLIP:
            if self.flip_index >= (1 << n_qubits):
                raise IndexError("flip index out of range")

    def desc(self) -> tuple:
        """Fields of qcs_gate_desc (include/qcs_b200.h)."""
        u = self.unitary.parts() if self.unitary is not None else [0.0] * 8
        c = self.control if self.control is not None else -1
        return (self.kind, self.target, c, self.flip_index, u)


_GATE_DESC = struct.Struct("<iiiiQ8d")


def pack_gates(gates: List[GateOp]) -> bytes:
    """Array of qcs_gate_desc (72 bytes each), as the C-ABI takes it."""
    out = bytearray()
    for g in gates:
        k, t, c, f, u = g.desc()
        out += _GATE_DESC.pack(k, t, c, 0, f, *u)
    return bytes(out)


@dataclass
class CircuitProgram:
    n_qubits: int = 0
    gates: List[GateOp] = field(default_factory=list)
    name: str = "circuit"


def _append_swap(p: CircuitProgram, a: int, b: int) -> None:
    """circuit.cpp:79-87: swap as three CX."""
    X = Unitary2x2.pauli_x()
    p.gates.append(GateOp.controlled(X, a, b, f"cx {a} {b}"))
    p.gates.append(GateOp.controlled(X, b, a, f"cx {b} {a}"))
    p.gates.append(GateOp.controlled(X, a, b, f"cx {a} {b}"))


def _parse_real(tok: str, line: int) -> float:
    try:
        return float(tok)
    except ValueError:
        raise ParseError(line, f"malformed number '{tok}'") from None


def _parse_qubit(tok: str, n: int, line: int, role: str) -> int:
    try:
        v = int(tok, 10)
    except ValueError:
        raise ParseError(line, f"malformed {role} '{tok}'") from None
    if v < 0 or v >= n:
        raise ParseError(line, f"{role} {tok} out of range for {n} qubits")
    return v


def parse_circuit(text: str, name: str = "circuit") -> CircuitProgram:
    """circuit.cpp:101-211."""
    prog = CircuitProgram(name=name)
    have_header = False
    line_no = 0
    for raw in text.splitlines():
        line_no += 1
        toks = []
        for t in raw.split():
            if t.startswith("#"):
                break
            toks.append(t)
        if not toks:
            continue
        op = toks[0]

        def arity(k):
            if len(toks) != k + 1:
                raise ParseError(line_no, f"'{op}' expects {k} argument(s), got {len(toks) - 1}")

        if not have_header:
            if op != "qubits":
                raise ParseError(line_no, "expected 'qubits <n>' before any instruction")
            arity(1)
            v = _parse_real(toks[1], line_no)
            if v < 1 or v > 59 or v != math.floor(v):
                raise ParseError(line_no, "qubit count must be an integer in [1, 59]")
            prog.n_qubits = int(v)
            have_header = True
            continue
        n = prog.n_qubits
        if op == "qubits":
            raise ParseError(line_no, "duplicate 'qubits' directive")
        if op in ("h", "x", "y", "z", "s", "t"):
            arity(1)
            q = _parse_qubit(toks[1], n, line_no, "qubit")
            u = {"h": Unitary2x2.hadamard, "x": Unitary2x2.pauli_x, "y": Unitary2x2.pauli_y,
                 "z": Unitary2x2.pauli_z, "s": Unitary2x2.s_gate, "t": Unitary2x2.t_gate}[op]()
            prog.gates.append(GateOp.single(u, q, " ".join(toks[:2])))
        elif op in ("cx", "cz"):
            arity(2)
            c = _parse_qubit(toks[1], n, line_no, "control")
            t = _parse_qubit(toks[2], n, line_no, "target")
            if c == t:
                raise ParseError(line_no, "control equals target")
            u = Unitary2x2.pauli_x() if op == "cx" else Unitary2x2.pauli_z()
            prog.gates.append(GateOp.controlled(u, c, t, " ".join(toks[:3])))
        elif op == "cp":
            arity(3)
            c = _parse_qubit(toks[1], n, line_no, "control")
            t = _parse_qubit(toks[2], n, line_no, "target")
            if c == t:
                raise ParseError(line_no, "control equals target")
            theta = _parse_real(toks[3], line_no)
            prog.gates.append(GateOp.controlled_phase(theta, c, t, " ".join(toks[:3])))
        elif op == "swap":
            arity(2)
            a = _parse_qubit(toks[1], n, line_no, "qubit")
            b = _parse_qubit(toks[2], n, line_no, "qubit")
            if a == b:
                raise ParseError(line_no, "swap qubits must differ")
            _append_swap(prog, a, b)
        elif op == "u":
            arity(9)
            q = _parse_qubit(toks[1], n, line_no, "qubit")
            v = [_parse_real(x, line_no) for x in toks[2:]]
            try:
                u = Unitary2x2(complex(v[0], v[1]), complex(v[2], v[3]),
                               complex(v[4], v[5]), complex(v[6], v[7]))
            except ValueError as e:
                raise ParseError(line_no, str(e)) from None
            prog.gates.append(GateOp.single(u, q, f"u {q}"))
        elif op == "flip":
            arity(1)
            v = _parse_real(toks[1], line_no)
            if v < 0 or v >= math.ldexp(1.0, n) or v != math.floor(v):
                raise ParseError(line_no, "basis index out of range")
            prog.gates.append(GateOp.phase_flip(int(v)))
        elif op == "diffuse":
            arity(0)
            prog.gates.append(GateOp.reflect_mean())
        else:
            raise ParseError(line_no, f"unknown instruction '{op}'")
    if not have_header:
        raise ParseError(1 if line_no == 0 else line_no, "missing 'qubits' header")
    return prog


def _fmt(v: float) -> str:
    return "%.17g" % v


def print_circuit(p: CircuitProgram) -> str:
    """circuit.cpp:213-272 (inverse of parse_circuit)."""
    out = [f"qubits {p.n_qubits}"]
    for g in p.gates:
        if g.kind == KIND_SINGLE:
            if g.label and g.label[0] != "u":
                out.append(g.label)
            else:
                u = g.unitary
                out.append(f"u {g.target} " + " ".join(
                    f"{_fmt(a.real)} {_fmt(a.imag)}" for a in (u.u11, u.u12, u.u21, u.u22)))
        elif g.kind == KIND_CONTROLLED:
            u = g.unitary
            is_x = abs(u.u11) < 1e-15 and abs(u.u12 - 1) < 1e-15 and abs(u.u21 - 1) < 1e-15 and abs(u.u22) < 1e-15
            is_z = abs(u.u12) == 0 and abs(u.u21) == 0 and abs(u.u11 - 1) == 0 and u.u22 == complex(-1, 0)
            is_diag = abs(u.u12) == 0 and abs(u.u21) == 0 and abs(u.u11 - 1) == 0
            if is_x:
                out.append(f"cx {g.control} {g.target}")
            elif is_z and g.phase_theta is None:
                out.append(f"cz {g.control} {g.target}")
            elif g.phase_theta is not None:
                out.append(f"cp {g.control} {g.target} {_fmt(g.phase_theta)}")
            elif is_diag:
                out.append(f"cp {g.control} {g.target} {_fmt(math.atan2(u.u22.imag, u.u22.real))}")
            else:
                raise ValueError("controlled gate has no text form: " + g.label)
        elif g.kind == KIND_FLIP:
            out.append(f"flip {g.flip_index}")
        else:
            out.append("diffuse")
    return "\n".join(out) + "\n"


def build_qft(n: int) -> CircuitProgram:
    """circuit.cpp:274-297: swap network first, then per target j its CP ladder
    and a Hadamard.  QFT-n has 3*floor(n/2) + n(n-1)/2 + n gates (F6)."""
    if n < 1:
        raise ValueError("qft needs at least one qubit")
    p = CircuitProgram(n, [], f"qft-{n}")
    for i in range(n // 2):
        _append_swap(p, i, n - 1 - i)
    for j in range(n):
        for k in range(j):
            theta = _PI / math.ldexp(1.0, j - k)
            p.gates.append(GateOp.controlled_phase(theta, k, j, f"cp {k} {j}"))
        p.gates.append(GateOp.single(Unitary2x2.hadamard(), j, f"h {j}"))
    return p


def build_grover(n: int, marked: int, iterations: int = -1) -> CircuitProgram:
    """circuit.cpp:299-325 (flip + diffuse primitives)."""
    if n < 1 or n > 59:
        raise ValueError("grover needs 1 to 59 qubits")
    if marked >= (1 << n):
        raise IndexError("marked index out of range")
    if iterations < 0:
        iterations = int(round(_PI / 4.0 * math.sqrt(math.ldexp(1.0, n))))
    p = CircuitProgram(n, [], f"grover-{n}")
    for q in range(n):
        p.gates.append(GateOp.single(Unitary2x2.hadamard(), q, f"h {q}"))
    for _ in range(iterations):
        p.gates.append(GateOp.phase_flip(marked))
        p.gates.append(GateOp.reflect_mean())
    return p


def build_grover_gate_form(n: int, marked: int, iterations: int) -> CircuitProgram:
    """BASELINE config 2: H^n, then iterations x [oracle flip(marked);
    diffusion H^n X^n MCZ X^n H^n == H^n flip(0) H^n]."""
    if marked >= (1 << n):
        raise IndexError("marked index out of range")
    p = CircuitProgram(n, [], f"grover-gates-{n}")
    H = Unitary2x2.hadamard()
    for q in range(n):
        p.gates.append(GateOp.single(H, q, f"h {q}"))
    for _ in range(iterations):
        p.gates.append(GateOp.phase_flip(marked))
        for q in range(n):
            p.gates.append(GateOp.single(H, q, f"h {q}"))
        p.gates.append(GateOp.phase_flip(0))
        for q in range(n):
            p.gates.append(GateOp.single(H, q, f"h {q}"))
    return p


def splitmix64(seed: int):
    """SplitMix64 stream (public-domain generator), used for our own seeded
    stand-in inputs (basis indices, grid circuits)."""
    x = seed & 0xFFFFFFFFFFFFFFFF
    while True:
        x = (x + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = x
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        yield z ^ (z >> 31)


def build_grid(rows: int, cols: int, depth: int, seed: int) -> CircuitProgram:
    """Seeded random grid circuit (stand-in for BASELINE config 4).

    Cycle c applies CZ on one of four nearest-neighbour edge patterns
    (horizontal even/odd, vertical even/odd, rotating with c) and then a
    single-qubit gate drawn from {sqrt X, sqrt Y, T} on every qubit, never
    repeating the qubit's previous draw.  Qubit (r, c) is index r*cols + c.
    """
    n = rows * cols
    rng = splitmix64(seed)
    p = CircuitProgram(n, [], f"grid-{rows}x{cols}-d{depth}")
    Z = Unitary2x2.pauli_z()
    last = [-1] * n
    gates1 = [Unitary2x2.sqrt_x(), Unitary2x2.sqrt_y(), Unitary2x2.t_gate()]
    for cyc in range(depth):
        pat = cyc % 4
        for r in range(rows):
            for c in range(cols):
                q = r * cols + c
                if pat < 2 and c + 1 < cols and c % 2 == pat:
                    p.gates.append(GateOp.controlled(Z, q, q + 1, f"cz {q} {q + 1}"))
                if pat >= 2 and r + 1 < rows and r % 2 == pat - 2:
                    p.gates.append(GateOp.controlled(Z, q, q + cols, f"cz {q} {q + cols}"))
        for q in range(n):
            k = next(rng) % 3
            if k == last[q]:
                k = (k + 1 + next(rng) % 2) % 3
            last[q] = k
            if k == 2:
                p.gates.append(GateOp.single(gates1[2], q, f"t {q}"))
            else:
                p.gates.append(GateOp.single(gates1[k], q, f"u {q}"))
    return p


def seeded_basis(n: int, seed: int) -> int:
    """Seeded basis index for the QFT configs (our SplitMix64 stream)."""
    return next(splitmix64(seed)) & ((1 << n) - 1)


def pow2_bound(eps: float, n: int) -> float:
    """Parity mapping of BASELINE's point-wise relative bound eps to the
    reference's absolute bound: the largest power of two not above
    eps * 2^-ceil(n/2) (SURVEY.md F2 gives eps*2^-ceil(n/2); rounding down to a
    power of two keeps the bound at least as tight and makes 2*delta*q exact
    in binary64)."""
    d = eps * math.ldexp(1.0, -((n + 1) // 2))
    return math.ldexp(1.0, math.frexp(d)[1] - 1)


def survey_bound(eps: float, n: int) -> float:
    """SURVEY.md §8(d)'s mapping itself: delta = eps * 2^-ceil(n/2) (not a
    power of two for eps = 1e-3 / 1e-4 / 1e-2)."""
    return eps * math.ldexp(1.0, -((n + 1) // 2))


def qft_stage(n: int, x: int, g: int):
    """Exact state that build_qft(n) (circuit.cpp:274-297) produces from the
    basis state x after its first g gates.  QFT keeps a product state: a qubit
    whose Hadamard has run holds (|0> + e^{i phi}|1>)/sqrt2, every other qubit a
    basis bit, and CP(k, j) only moves phi_k (qubit j is still a basis bit when
    its ladder runs).  So
        a_y = 2^(-m/2) exp(2 pi i R(y) / 2^n)  if (y & zmask) == zval, else 0,
        R(y) = sum_k y_k r[k]  (mod 2^n),
    with m the number of processed qubits.  Returns (m, r, zmask, zval)."""
    if not 0 <= g <= len(build_qft(n).gates):
        raise IndexError("gate index outside the program")
    b = x
    done = 0
    for i in range(n // 2):                 # swap network: CX permutes basis states
        a, c = i, n - 1 - i
        for ctl, tgt in ((a, c), (c, a), (a, c)):
            if done == g:
                return 0, [0] * n, (1 << n) - 1, b
            if (b >> ctl) & 1:
                b ^= 1 << tgt
            done += 1
    r = [0] * n
    processed = 0
    mod = (1 << n) - 1
    for j in range(n):
        for k in range(j):
            if done == g:
                break
            if (b >> j) & 1:                # CP(k, j), theta = pi / 2^(j-k)
                r[k] = (r[k] + (1 << (n - 1 - (j - k)))) & mod
            done += 1
        if done == g:
            break
        processed |= 1 << j                 # H(j)
        r[j] = (r[j] + (((b >> j) & 1) << (n - 1))) & mod
        done += 1
    zmask = ((1 << n) - 1) & ~processed
    return bin(processed).count("1"), r, zmask, b & zmask


def stage_tables(n: int, s: int, m: int, r, zmask: int, zval: int):
    """Factor tables of a qft_stage state for generation stride by stride:
    a_y = amp * lo[y mod 2^s] * hi[y >> s] (complex), zero where
    (y & zmask) != zval.  Both benchmark arms (GPU: torch; reference: the C++
    generator in oracle/ref_capi.cpp) form t = hr*lr - hi*li, u = hr*li + hi*lr,
    then amp*t, amp*u with the same IEEE operations, so they start from
    bit-identical amplitudes."""
    import numpy as np
    L, NS = 1 << s, 1 << (n - s)
    mod = np.uint64((1 << n) - 1)
    w = 2.0 * math.pi / float(1 << n)

    def table(bits0, count):
        idx = np.arange(count, dtype=np.uint64)
        R = np.zeros(count, dtype=np.uint64)
        for k in range(bits0, bits0 + (count.bit_length() - 1)):
            R = (R + ((idx >> np.uint64(k - bits0)) & np.uint64(1)) * np.uint64(r[k])) & mod
        ang = R.astype(np.float64) * w
        return np.cos(ang), np.sin(ang)

    lo_re, lo_im = table(0, L)
    hi_re, hi_im = table(s, NS)
    amp = math.ldexp(math.sqrt(0.5) if m & 1 else 1.0, -(m // 2))
    return dict(lo_re=lo_re, lo_im=lo_im, hi_re=hi_re, hi_im=hi_im, amp=amp, zmask=zmask, zval=zval)


class _MT19937_64:
    """std::mt19937_64 (the standard's parameters), for build_random."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            prev = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.i = 312

    def __call__(self) -> int:
        if self.i >= 312:
            mt = self.mt
            for k in range(312):
                y = (mt[k] & 0xFFFFFFFF80000000) | (mt[(k + 1) % 312] & 0x7FFFFFFF)
                v = mt[(k + 156) % 312] ^ (y >> 1)
                if y & 1:
                    v ^= 0xB5026F5AA96619E9
                mt[k] = v
            self.i = 0
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF


def _uniform_int(rng, a: int, b: int) -> int:
    """libstdc++ uniform_int_distribution over a 64-bit engine (GCC >= 11:
    Lemire's nearly divisionless method with a 128-bit product)."""
    urange = (b - a) & 0xFFFFFFFFFFFFFFFF
    if urange == 0xFFFFFFFFFFFFFFFF:
        return a + rng()
    uerange = urange + 1
    product = rng() * uerange
    low = product & 0xFFFFFFFFFFFFFFFF
    if low < uerange:
        threshold = ((1 << 64) - uerange) % uerange
        while low < threshold:
            product = rng() * uerange
            low = product & 0xFFFFFFFFFFFFFFFF
    return a + (product >> 64)


def _uniform_real(rng, a: float, b: float) -> float:
    """libstdc++ uniform_real_distribution: generate_canonical<double, 53> over a
    64-bit engine (one draw / 2^64, clamped below 1), then x * (b - a) + a."""
    r = float(rng()) / 18446744073709551616.0
    if r >= 1.0:
        r = math.nextafter(1.0, 0.0)
    return r * (b - a) + a


def build_random(n: int, gate_count: int, seed: int) -> CircuitProgram:
    """circuit.cpp:327-387, draw for draw: std::mt19937_64(seed), angles
    uniform in [0, 2 pi), qubits uniform in [0, n-1], kind uniform in [0, 9]."""
    if n < 1:
        raise ValueError("random circuit needs at least one qubit")
    if gate_count < 0:
        raise ValueError("gate count must be non-negative")
    p = CircuitProgram(n, [], f"random-{n}")
    rng = _MT19937_64(seed)
    angle = lambda: _uniform_real(rng, 0.0, 2.0 * _PI)  # noqa: E731
    qubit = lambda: _uniform_int(rng, 0, n - 1)  # noqa: E731

    def random_unitary():
        th = angle() / 2.0
        p1 = angle()
        p2 = angle()
        c, s = math.cos(th), math.sin(th)
        return Unitary2x2(complex(c * math.cos(p1), c * math.sin(p1)),
                          complex(s * math.cos(p2), s * math.sin(p2)),
                          complex(-s * math.cos(-p2), -s * math.sin(-p2)),
                          complex(c * math.cos(-p1), c * math.sin(-p1)))

    for i in range(gate_count):
        kind = _uniform_int(rng, 0, 9)
        if kind < 4:
            # GCC evaluates GateOp::single(random_unitary(), qubit(rng), ...)'s
            # arguments right to left: the target is drawn first
            t = qubit()
            p.gates.append(GateOp.single(random_unitary(), t, f"u {i}"))
        elif kind < 6 and n >= 2:
            c = qubit()
            t = qubit()
            while t == c:
                t = qubit()
            p.gates.append(GateOp.controlled(Unitary2x2.pauli_x(), c, t, f"cx {c} {t}"))
        elif kind < 8 and n >= 2:
            c = qubit()
            t = qubit()
            while t == c:
                t = qubit()
            p.gates.append(GateOp.controlled_phase(angle(), c, t, f"cp {c} {t}"))
        elif kind == 8:
            p.gates.append(GateOp.phase_flip(_uniform_int(rng, 0, (1 << n) - 1)))
        else:
            q = qubit()
            p.gates.append(GateOp.single(Unitary2x2.hadamard(), q, f"h {q}"))
    return p
