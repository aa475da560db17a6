"""Shared test helpers: run a circuit through the oracle or the GPU engine
and compare everything the reference exposes."""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np

from paper_1811_05140_b200 import circuit as cc
from paper_1811_05140_b200 import metrics as mm

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden_runs():
    with open(os.path.join(GOLD, "runs.json")) as f:
        return json.load(f)


def golden_program(entry):
    with open(os.path.join(GOLD, entry["circuit"])) as f:
        return cc.parse_circuit(f.read())


def golden_codec():
    z = np.load(os.path.join(GOLD, "codec.npz"))
    for name in z["names"]:
        name = str(name)
        yield name, z[f"{name}__x"], float(z[f"{name}__delta"][0]), z[f"{name}__blk"].tobytes()


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def oracle_run(oracle, prog, s, basis, ladder, theta):
    st = oracle.state(prog.n_qubits, s, basis)
    recs = []
    for i, g in enumerate(prog.gates):
        reps, norm = st.apply_gate(g, ladder, theta)
        recs.append(mm.gate_record(i, g.label, reps, norm)[0])
    return st, mm.emit_csv(recs, with_elapsed=False)


def gpu_run(prog, s, basis, ladder, theta):
    import paper_1811_05140_b200 as q
    res = q.run_program(prog, q.ErrorBoundLadder.make(ladder), q.RatioThreshold(theta),
                        q.StateGeometry.make(prog.n_qubits, s), q.RunOptions(basis=basis))
    return res, mm.emit_csv(res.metrics.records, with_elapsed=False)


def first_diff(a: str, b: str) -> str:
    for i, (x, y) in enumerate(zip(a.splitlines(), b.splitlines())):
        if x != y:
            return f"line {i}:\n  want {x}\n  got  {y}"
    return "length differs"
