"""The command-line front end (paper_1811_05140_b200/cli.py), after the
reference's tests/test_cli.cpp: exit codes 0/1/2, artifact shapes (QFT-10 =
70 CSV rows), compare / bench / codec outputs, seed determinism, checkpoint
resume -- plus the random-circuit builder against the reference's own
build_random (circuit.cpp:327-387) text for text."""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1811_05140_b200 import circuit as cc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, cwd):
    p = subprocess.run([sys.executable, "-m", "paper_1811_05140_b200"] + args, cwd=cwd,
                       capture_output=True, text=True, env=dict(os.environ, PYTHONPATH=ROOT))
    return p.returncode, p.stdout + p.stderr


@pytest.mark.parametrize("args", [["simulate"], ["frobnicate"], ["simulate", "--circuit", "builtin:qft"],
                                  ["bench", "--circuit", "builtin:qft", "--qubits", "4", "--thetas", ""],
                                  ["simulate", "--circuit", "builtin:qft", "--qubits", "8", "--ladder", "1e-3,1e-7"],
                                  ["simulate", "--circuit", "builtin:nope", "--qubits", "3"]])
def test_usage_errors_exit_2(tmp_path, args):
    """test_cli.cpp:84-95."""
    assert run(args, tmp_path)[0] == 2


def test_help_exits_0(tmp_path):
    assert run(["--help"], tmp_path)[0] == 0


def test_missing_circuit_file_names_path_exit_2(tmp_path):
    """test_cli.cpp:97-103."""
    rc, out = run(["simulate", "--circuit", "./no_such_circuit.txt"], tmp_path)
    assert rc == 2 and "no_such_circuit.txt" in out


def test_corrupt_checkpoint_exit_1(tmp_path):
    """test_cli.cpp:105-116."""
    (tmp_path / "g.qckp").write_bytes(b"QCKPgarbage garbage garbage garbage")
    rc, _ = run(["simulate", "--circuit", "builtin:qft", "--qubits", "8", "--load-state", "g.qckp"], tmp_path)
    assert rc == 1


def test_codec_missing_input_exit_2(tmp_path):
    assert run(["codec", "--input", "nothing.bin"], tmp_path)[0] == 2


@pytest.mark.parametrize("n,g,seed", [(7, 40, 1), (7, 40, 2), (12, 300, 12345), (1, 20, 5), (30, 200, 99), (2, 500, 3)])
def test_build_random_matches_reference(reference, n, g, seed):
    assert cc.print_circuit(cc.build_random(n, g, seed)) == reference.builtin(2, n, seed, g)


@pytest.mark.gpu
def test_simulate_artifacts(tmp_path):
    """test_cli.cpp:118-141: 70 gates of QFT-10 plus the header; summary JSON."""
    rc, out = run(["simulate", "--circuit", "builtin:qft", "--qubits", "10", "--basis", "1", "--theta", "16",
                   "--ladder", "0,1e-7,1e-6,1e-5,1e-4,1e-3", "--out-csv", "r.csv", "--out-json", "r.json"], tmp_path)
    assert rc == 0, out
    assert "overall min ratio" in out
    lines = (tmp_path / "r.csv").read_text().splitlines()
    assert lines[0].startswith("gate_index,") and len(lines) == 71
    js = (tmp_path / "r.json").read_text()
    assert '"overall_min_ratio"' in js and '"qubit_gain"' in js and '"fidelity"' not in js


@pytest.mark.gpu
def test_simulate_csv_matches_reference(reference, tmp_path):
    """The CLI's records are the reference's (default ladder, theta 16)."""
    from paper_1811_05140_b200 import metrics as mm
    rc, out = run(["simulate", "--circuit", "builtin:qft", "--qubits", "10", "--basis", "1", "--out-csv", "r.csv"],
                  tmp_path)
    assert rc == 0, out
    ref_csv, _, _ = reference.run(cc.print_circuit(cc.build_qft(10)), 10, 1, [0, 1e-7, 1e-6, 1e-5, 1e-4, 1e-3], 16.0)
    assert mm.strip_elapsed((tmp_path / "r.csv").read_text()) == mm.strip_elapsed(ref_csv)


@pytest.mark.gpu
def test_circuit_file_and_compare_lossless(tmp_path):
    """test_cli.cpp:143-169: fidelity 1 under a lossless ladder."""
    (tmp_path / "c.txt").write_text(cc.print_circuit(cc.build_qft(6)))
    rc, out = run(["compare", "--circuit", "c.txt", "--ladder", "0", "--theta", "1"], tmp_path)
    assert rc == 0, out
    assert "fidelity:             1.0000" in out and "reference norm" in out and "compressed norm" in out


@pytest.mark.gpu
def test_compare_refuses_above_dense_guard(tmp_path):
    assert run(["compare", "--circuit", "builtin:qft", "--qubits", "12", "--max-dense", "10"], tmp_path)[0] == 2


@pytest.mark.gpu
def test_bench_rows(tmp_path):
    """test_cli.cpp:178-191."""
    rc, out = run(["bench", "--circuit", "builtin:qft", "--qubits", "8", "--thetas", "4,16", "--out-csv", "b.csv"],
                  tmp_path)
    assert rc == 0, out
    lines = (tmp_path / "b.csv").read_text().splitlines()
    assert lines[0] == "theta,min_ratio,fidelity,time_ns" and len(lines) == 3
    assert lines[1].startswith("4,") and lines[2].startswith("16,")


@pytest.mark.gpu
def test_codec_round_trip(tmp_path):
    """test_cli.cpp:193-227."""
    x = np.random.default_rng(3).standard_normal(1000)
    (tmp_path / "d.bin").write_bytes(x.astype("<f8").tobytes())
    rc, out = run(["codec", "--input", "d.bin", "--output", "rt.bin"], tmp_path)
    assert rc == 0 and "max error:        0" in out
    assert (tmp_path / "rt.bin").read_bytes() == (tmp_path / "d.bin").read_bytes()
    rc, out = run(["codec", "--input", "d.bin", "--delta", "1e-3"], tmp_path)
    assert rc == 0 and "ratio:" in out


@pytest.mark.gpu
def test_seed_determinism_and_checkpoint_resume(tmp_path):
    """test_cli.cpp:229-290."""
    from paper_1811_05140_b200 import metrics as mm
    base = ["simulate", "--circuit", "builtin:random", "--qubits", "7", "--gates", "40", "--stride-bits", "3"]
    assert run(base + ["--seed", "5", "--out-csv", "s1.csv"], tmp_path)[0] == 0
    assert run(base + ["--seed", "5", "--out-csv", "s2.csv"], tmp_path)[0] == 0
    assert run(base + ["--seed", "6", "--out-csv", "s3.csv"], tmp_path)[0] == 0
    s = [mm.strip_elapsed((tmp_path / f"s{i}.csv").read_text()) for i in (1, 2, 3)]
    assert s[0] == s[1] and s[0] != s[2]
    common = ["simulate", "--circuit", "builtin:qft", "--qubits", "9", "--stride-bits", "5"]
    assert run(common + ["--out-csv", "full.csv"], tmp_path)[0] == 0
    assert run(common + ["--stop-after", "22", "--save-state", "mid.qckp"], tmp_path)[0] == 0
    assert run(common + ["--load-state", "mid.qckp", "--start-gate", "22", "--out-csv", "tail.csv"], tmp_path)[0] == 0
    full = (tmp_path / "full.csv").read_text().splitlines()
    tail = (tmp_path / "tail.csv").read_text().splitlines()
    assert tail[1].startswith("22,") and len(full) - 1 == (len(tail) - 1) + 22
    assert mm.strip_elapsed("\n".join([full[0]] + full[23:]) + "\n") == mm.strip_elapsed("\n".join(tail) + "\n")
