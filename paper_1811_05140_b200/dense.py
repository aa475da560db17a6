"""Uncompressed complex128 state vector on the GPU (torch): the desk-scale
checker behind the CLI's `compare` / `bench` and the bench's fidelity, after
the reference's dense simulator (dense.hpp, dense.cpp:30-108): the same gate
semantics, fidelity |<a|b>| / (|a| |b|), zero norm -> 0.  Not the hot path
(which is the compressed engine); torch complex arithmetic agrees with the
reference's serial loop to rounding, not bit for bit."""
from __future__ import annotations

from . import circuit as cc

DENSE_QUBIT_GUARD = 26  # dense.hpp:14


def dense_apply(psi, n: int, g) -> None:
    """One gate on a dense state (dense_apply, dense.cpp:30-76)."""
    if g.kind == cc.KIND_FLIP:
        psi[g.flip_index] = -psi[g.flip_index]
        return
    if g.kind == cc.KIND_REFLECT:
        psi.copy_(2.0 * psi.mean() - psi)
        return
    u, t = g.unitary, g.target
    if g.kind == cc.KIND_SINGLE:
        v = psi.view(1 << (n - t - 1), 2, 1 << t)
        a0, a1 = v[:, 0, :].clone(), v[:, 1, :].clone()
        v[:, 0, :] = u.u11 * a0 + u.u12 * a1
        v[:, 1, :] = u.u21 * a0 + u.u22 * a1
        return
    c = g.control
    hi, lo = max(c, t), min(c, t)
    v = psi.view(1 << (n - hi - 1), 2, 1 << (hi - lo - 1), 2, 1 << lo)
    sel = (lambda b: v[:, 1, :, b, :]) if c == hi else (lambda b: v[:, b, :, 1, :])
    a0, a1 = sel(0).clone(), sel(1).clone()
    sel(0).copy_(u.u11 * a0 + u.u12 * a1)
    sel(1).copy_(u.u21 * a0 + u.u22 * a1)


def run_dense(prog, basis: int = 0, max_qubits: int = DENSE_QUBIT_GUARD, device=0, n_gates=None):
    """run_dense (dense.cpp:78-92): the program from |basis> (complex128 tensor)."""
    import torch
    n = prog.n_qubits
    if n > max_qubits:
        raise ValueError(f"dense reference guard exceeded: {n} qubits > {max_qubits}")
    if basis >= (1 << n):
        raise IndexError("basis index out of range")
    psi = torch.zeros(1 << n, dtype=torch.complex128, device=device)
    psi[basis] = 1.0
    for g in prog.gates[: len(prog.gates) if n_gates is None else n_gates]:
        dense_apply(psi, n, g)
    return psi


def fidelity(a, b) -> float:
    """dense.cpp:94-108: |<a|b>| after normalising both; zero norm -> 0."""
    import torch
    na, nb = torch.linalg.vector_norm(a), torch.linalg.vector_norm(b)
    if float(na) == 0.0 or float(nb) == 0.0:
        return 0.0
    return float(torch.abs(torch.vdot(a, b)) / (na * nb))
