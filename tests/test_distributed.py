"""Sharded state: every world size reproduces the single-process
bits — per-gate CSV (minus wall time) and the final amplitudes.

CPU: ranks as threads (ThreadComm) and as gloo processes (TorchComm,
world_size 2) over the oracle backend.  GPU: two ranks on one GPU through the
C-ABI, host-staged exchange (no rank waits on another's kernel).
"""
import os
import socket

import numpy as np
import pytest

import paper_1811_05140_b200 as q
from paper_1811_05140_b200 import metrics as mm
from paper_1811_05140_b200 import circuit as cc
from paper_1811_05140_b200.distributed import (GpuBackend, ShardGeometry, run_thread_cluster)

from helpers import golden_program, golden_runs, oracle_run, sha


def _cases():
    lad = [q.pow2_bound(1e-3, 10)]
    return [
        ("qft10", q.build_qft(10), 4, 397, lad, 1.0),
        ("grover_gates10", q.build_grover_gate_form(10, 0x2d3, 3), 4, 0, lad, 1.0),
        ("grover10_reflect", q.build_grover(10, 0x155, 2), 4, 0, lad, 1.0),
        ("grid3x3", q.build_grid(3, 3, 8, 11), 3, 5, [2.0 ** -16, 2.0 ** -12], 2.0),
        ("qft10_lossless", q.build_qft(10), 3, 17, [0.0], 1.0),
    ]


def _single(oracle, prog, s, basis, lad, theta):
    st, csv = oracle_run(oracle, prog, s, basis, lad, theta)
    return st.amplitudes(), csv


@pytest.mark.parametrize("chunk", [None, "1"])
@pytest.mark.parametrize("ranks", [2, 4])
@pytest.mark.parametrize("case", _cases(), ids=lambda c: c[0])
def test_thread_cluster_oracle(oracle, monkeypatch, case, ranks, chunk):
    """chunk="1": every exchange streamed one stride per chunk
    (QCS_EXCHANGE_CHUNK_BYTES), same bits."""
    if chunk:
        monkeypatch.setenv("QCS_EXCHANGE_CHUNK_BYTES", chunk)
    from oracle import OracleBackend
    name, prog, s, basis, lad, theta = case
    rb = ranks.bit_length() - 1
    if prog.n_qubits - rb < s + 2:
        pytest.skip("too few local strides")
    want_amp, want_csv = _single(oracle, prog, s, basis, lad, theta)
    geom = ShardGeometry(prog.n_qubits, s, rb)
    amp, recs = run_thread_cluster(prog, geom, lambda r: OracleBackend(oracle), basis, lad, theta)
    got_csv = mm.emit_csv(recs, with_elapsed=False)
    assert got_csv == want_csv
    assert amp.tobytes() == want_amp.tobytes()


def _golden_sharded():
    out = []
    for name, e in sorted(golden_runs().items()):
        n = golden_program(e).n_qubits
        for ranks in (2, 4):
            if n - (ranks.bit_length() - 1) >= e["stride_bits"] + 2:
                out.append((name, ranks))
    return out


@pytest.mark.parametrize("name,ranks", _golden_sharded())
def test_thread_cluster_matches_reference_golden(oracle, name, ranks):
    """Sharded run vs the reference's own outputs (tests/golden/runs.json)."""
    from oracle import OracleBackend
    e = golden_runs()[name]
    prog = golden_program(e)
    geom = ShardGeometry(prog.n_qubits, e["stride_bits"], ranks.bit_length() - 1)
    amp, recs = run_thread_cluster(prog, geom, lambda r: OracleBackend(oracle), e["basis"],
                                   e["ladder"], e["theta"])
    assert mm.emit_csv(recs, with_elapsed=False) == e["csv"]
    assert sha(amp) == e["amps_sha256"]


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _gloo_worker(rank, world, port, outdir):
    import torch.distributed as dist
    from oracle import OracleBackend
    from paper_1811_05140_b200.distributed import TorchComm, run_sharded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for name, prog, s, basis, lad, theta in _cases():
            st, recs, _ = run_sharded(prog, ShardGeometry(prog.n_qubits, s, 1), TorchComm(),
                                      OracleBackend(), basis, lad, theta)
            amp = st.amplitudes()
            if rank == 0:
                with open(os.path.join(outdir, name + ".csv"), "w") as f:
                    f.write(mm.emit_csv(recs, with_elapsed=False))
                np.save(os.path.join(outdir, name + ".npy"), amp)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_oracle(oracle, tmp_path):
    import torch.multiprocessing as tmp
    tmp.spawn(_gloo_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    for name, prog, s, basis, lad, theta in _cases():
        want_amp, want_csv = _single(oracle, prog, s, basis, lad, theta)
        assert (tmp_path / (name + ".csv")).read_text() == want_csv, name
        assert np.load(tmp_path / (name + ".npy")).tobytes() == want_amp.tobytes(), name


def test_rank_geometry_errors(oracle):
    from oracle import OracleBackend
    from paper_1811_05140_b200.distributed import ShardedState, ThreadComm, ThreadGroup
    with pytest.raises(ValueError):
        ShardedState(ShardGeometry(8, 7, 1), ThreadComm(ThreadGroup(2), 0), OracleBackend(oracle), 0)
    with pytest.raises(ValueError):
        ShardedState(ShardGeometry(8, 4, 2), ThreadComm(ThreadGroup(2), 0), OracleBackend(oracle), 0)


@pytest.mark.gpu
@pytest.mark.parametrize("ranks", [2, 4])
@pytest.mark.parametrize("case", _cases(), ids=lambda c: c[0])
def test_thread_cluster_gpu(oracle, monkeypatch, case, ranks):
    monkeypatch.setenv("QCS_EXCHANGE_CHUNK_BYTES", "4096")  # several chunks per exchange
    name, prog, s, basis, lad, theta = case
    rb = ranks.bit_length() - 1
    if prog.n_qubits - rb < s + 2:
        pytest.skip("too few local strides")
    want_amp, want_csv = _single(oracle, prog, s, basis, lad, theta)
    amp, recs = run_thread_cluster(prog, ShardGeometry(prog.n_qubits, s, rb),
                                   lambda r: GpuBackend(0), basis, lad, theta)
    assert mm.emit_csv(recs, with_elapsed=False) == want_csv
    assert amp.tobytes() == want_amp.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("force_big", [0, 1])
def test_stride_images_round_trip_gpu(oracle, monkeypatch, force_big):
    """qcs_pack_strides / qcs_unpack_strides move strides verbatim (blocks,
    side index, scale, sum) through the commit path of either layout."""
    import torch
    from oracle import OracleBackend
    if force_big:
        monkeypatch.setenv("QCS_FORCE_BIG", "1")
        monkeypatch.setenv("QCS_WAVE_SLOTS", "2")
    prog = q.build_qft(11)
    lad = [q.pow2_bound(1e-3, 11)]
    a = GpuBackend(0).create(11, 6, 5)
    o = OracleBackend(oracle).create(11, 6, 5)
    for g in prog.gates[:40]:
        a.apply(g, lad, 1.0)
        o.apply(g, lad, 1.0)
    # swap stride bit 3 = 1 half into a fresh zero state's bit 3 = 0 half
    b = GpuBackend(0).create(11, 6, None)
    img = a.pack(3, 1)
    assert img.is_cuda and img.dtype == torch.uint8
    b.unpack(img, 1 << 3)
    ob = OracleBackend(oracle).create(11, 6, None)
    ob.unpack(o.pack(3, 1), 1 << 3)
    for j in range(32):
        assert b.export(j) == ob.export(j), j
    # and back onto the source: a no-op on its content
    a.unpack(b.pack(3, 0), 1 << 3)
    for j in range(32):
        assert a.export(j) == o.export(j), j


@pytest.mark.gpu
def test_sharded_bench_functional(tmp_path):
    """bench.py's N > 1 path (sharded C2 weak scaling) end to end with two
    ranks.  One GPU here: both ranks share it and exchange through gloo, so no
    rank waits on another's kernel; the numbers are not a measurement."""
    import json
    import subprocess
    import sys
    env = dict(os.environ, QCS_DIST_BACKEND="gloo", QCS_SAME_DEVICE="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
                        os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, timeout=900, env=env, cwd=str(tmp_path))
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["config"]["n_qubits"] == 25


def _gloo_gpu_worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    from paper_1811_05140_b200.distributed import TorchComm, run_sharded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    try:
        for name, prog, s, basis, lad, theta in _cases()[:3]:
            st, recs, _ = run_sharded(prog, ShardGeometry(prog.n_qubits, s, 1), TorchComm(),
                                      GpuBackend(0), basis, lad, theta)
            amp = st.amplitudes()
            if rank == 0:
                with open(os.path.join(outdir, name + ".csv"), "w") as f:
                    f.write(mm.emit_csv(recs, with_elapsed=False))
                np.save(os.path.join(outdir, name + ".npy"), amp)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_gloo_world2_gpu_shards(oracle, tmp_path):
    """Two processes (one GPU shared; images staged through gloo) running QFT
    (controlled phases with rank-qubit controls and targets), Grover gate form
    and reflect_mean: equal to the single-process oracle."""
    import torch.multiprocessing as tmp
    tmp.spawn(_gloo_gpu_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    for name, prog, s, basis, lad, theta in _cases()[:3]:
        want_amp, want_csv = _single(oracle, prog, s, basis, lad, theta)
        assert (tmp_path / (name + ".csv")).read_text() == want_csv, name
        assert np.load(tmp_path / (name + ".npy")).tobytes() == want_amp.tobytes(), name


def test_lazy_permutation_one_exchange_per_rank_qubit_gate(oracle):
    """Rank-qubit targets swap in once and stay (no swap back, furthest-next-use
    eviction): one exchange per gate that finds its target on a rank bit, and
    fewer exchanges than the swap-in / swap-out scheme (two per rank-qubit
    target)."""
    from oracle import OracleBackend
    from paper_1811_05140_b200.distributed import ShardedState, ThreadComm, ThreadGroup
    import threading
    for prog, s in ((q.build_qft(10), 4), (q.build_grover_gate_form(10, 0x2d3, 3), 4)):
        geom = ShardGeometry(prog.n_qubits, s, 2)
        grp = ThreadGroup(4)
        res = [None] * 4

        def worker(r):
            st = ShardedState(geom, ThreadComm(grp, r), OracleBackend(oracle), 0)
            st.set_schedule(prog.gates)
            rank_gates = 0
            for i, g in enumerate(prog.gates):
                if g.kind in (0, 1) and g.target >= s and st.pi[g.target - s] >= geom.local_qubits - s:
                    rank_gates += 1
                st.apply_gate(g, [q.pow2_bound(1e-3, 10)], 1.0, i)
            res[r] = (st.exchanges, rank_gates)

        ts = [threading.Thread(target=worker, args=(r,)) for r in range(4)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        ex, rg = res[0]
        assert ex == rg  # exactly one exchange per gate that found its target on a rank bit
        from paper_1811_05140_b200.distributed import plan_exchanges
        assert len(plan_exchanges(prog, geom)) == ex  # the data-free planner makes the same decisions
        naive = sum(1 for g in prog.gates if g.kind in (0, 1) and g.target >= geom.local_qubits)
        assert ex <= 2 * naive // 2 + naive // 2, (ex, naive)  # at most 1.5 per rank-qubit gate
        assert ex < 2 * naive


def test_control_on_the_only_local_stride_bit(oracle):
    """One local stride bit (n - g = s + 1) and a controlled gate whose control
    holds it while the target is a rank qubit: the control is evicted to a rank
    bit (then the rank-level skip applies) -- same bits as one process."""
    from oracle import OracleBackend
    n, s, rb = 6, 4, 1
    U = cc.Unitary2x2
    prog = cc.CircuitProgram(n, [cc.GateOp.single(U.hadamard(), q, f"h {q}") for q in range(n)] +
                             [cc.GateOp.controlled(U.sqrt_x(), 4, 5, "c4t5"), cc.GateOp.controlled(U.t_gate(), 5, 4, "c5t4"),
                              cc.GateOp.controlled(U.pauli_y(), 4, 5, "c4t5y")], "ctl-local")
    lad, theta = [2.0 ** -14], 1.0
    want_amp, want_csv = _single(oracle, prog, s, 3, lad, theta)
    amp, recs = run_thread_cluster(prog, ShardGeometry(n, s, rb), lambda r: OracleBackend(oracle), 3, lad, theta)
    assert mm.emit_csv(recs, with_elapsed=False) == want_csv
    assert amp.tobytes() == want_amp.tobytes()
