"""C5 one-shard rehearsal on one B200 (BASELINE configs[4]: QFT-37, 2^21-amp
strides, 8 GPUs, the 3 top qubits index the GPU).  Rank 0's shard -- 34 local
qubits, 8192 strides of 2^21 amplitudes -- runs rank 0's part of every one of
the 757 gates through the sharded layer (paper_1811_05140_b200/distributed.py:
lazy qubit permutation, Belady eviction, control-on-rank-qubit skips), and at
each planned exchange sends half of its strides as device stride images
(qcs_pack_strides_range), moves them through a device copy standing in for the
NVLink transfer, and installs them (qcs_unpack_strides) -- against itself as a
loopback partner: the same bytes move as between two ranks, the data differ
from the real 8-GPU run (rank 0 receives its own strides), and the global
renormalisation folds 8 copies of rank 0's tables.  Reports the per-GPU device
time, the exchange count, bytes and time.
usage: python tools/c5_rehearsal.py [gates] > profiles/r2_c5_rehearsal.json"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1811_05140_b200 import circuit as cc  # noqa: E402
from paper_1811_05140_b200.distributed import GpuBackend, ShardedState, ShardGeometry, plan_exchanges  # noqa: E402


class LoopbackComm:
    """Rank 0 of `size` ranks whose partners mirror it: gathers return 8 copies
    of rank 0's data, an exchange returns a device copy of what was sent."""

    def __init__(self, size):
        self.rank, self.size = 0, size
        self.bytes = 0
        self.copy_s = 0.0

    def allgather(self, obj):
        return [obj] * self.size

    def allgather_array(self, arr):
        return [np.array(arr, copy=True) for _ in range(self.size)]

    def exchange(self, peer, obj, device=False):
        if peer is None:
            return None
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        got = obj.clone()                       # the NVLink transfer's stand-in
        torch.cuda.synchronize()
        self.copy_s += time.perf_counter() - t0
        self.bytes += obj.numel()
        return got


n, s, g = 37, 21, 3
prog = cc.build_qft(n)
# the seeded basis with its low three bits cleared: after the swap network
# they are the rank bits, so rank 0 holds the state's non-zero part through
# the late stages -- the busiest rank, which sets C5's time (the others hold
# all-zero strides until the rank qubits' Hadamards spread the state)
x = next(cc.splitmix64(n)) & ((1 << n) - 1) & ~7
delta = cc.pow2_bound(1e-3, n)
# dense part of the run: the last four stages (targets 33..36; the three rank
# qubits 34..36 need the exchanges), from the exact state at their start
g0 = len(prog.gates) - (n + (n - 1) + (n - 2) + (n - 3))
n_gates = int(sys.argv[1]) if len(sys.argv) > 1 else len(prog.gates) - g0
geom = ShardGeometry(n, s, g)
comm = LoopbackComm(1 << g)
os.environ.setdefault("QCS_RESERVE_BYTES", str(12 << 30))  # exchange images (pack + copy) live outside the arena
os.environ.setdefault("QCS_EXCHANGE_CHUNK_BYTES", str(1 << 30))
st = ShardedState(geom, comm, GpuBackend(0), 0)
# rank 0's strides of the exact state at gate g0 (global strides [0, 2^(n-g-s)),
# identity permutation), compressed through qcs_load_strides_device
from paper_1811_05140_b200.stage import StageGen  # noqa: E402
from paper_1811_05140_b200.engine import ErrorBoundLadder, _check, lib  # noqa: E402
gen = StageGen(cc.stage_tables(n, s, *cc.qft_stage(n, x, g0)), n, s, 0)
L, nsl = 1 << s, geom.local_strides
lad = ErrorBoundLadder.make([delta])
buf = torch.empty(32 * 2 * L, dtype=torch.float64, device=0)
for j0 in range(0, nsl, 32):
    m = min(32, nsl - j0)
    gen.fill(buf[: m * 2 * L].view(m, 2, L), j0, m)
    torch.cuda.synchronize()
    _check(lib().qcs_load_strides_device(st.local.h, j0, m, buf.data_ptr(), lad.c_array(), 1, 1.0))
del buf, gen
torch.cuda.empty_cache()
sub = cc.CircuitProgram(n, prog.gates[g0:], prog.name)
st.set_schedule(sub.gates)
planned = [g0 + i for i in plan_exchanges(sub, geom)]
dev_ns = 0
t0 = time.perf_counter()
for i, gate in enumerate(sub.gates[:n_gates]):
    torch.cuda.synchronize()
    a = time.perf_counter()
    st.apply_gate(gate, [delta], 1.0, i)
    torch.cuda.synchronize()
    dev_ns += (time.perf_counter() - a) * 1e9
    if i % 16 == 0:
        print(f"gate {g0 + i}: {dev_ns * 1e-9:.1f} s, exchanges {st.exchanges}", file=sys.stderr, flush=True)
wall = time.perf_counter() - t0
import ctypes as C  # noqa: E402

b, r, q = C.c_uint64(), C.c_double(), C.c_double()
lib().qcs_state_stats(st.local.h, C.byref(b), C.byref(r), C.byref(q))
amp_updates = 0  # per gate: rewritten strides of rank 0
print(json.dumps({
    "what": "C5 one-shard rehearsal: rank 0 of QFT-37 on 8 GPUs (34 local qubits, 2^21-amp strides) on one B200, "
            "the last four stages (targets 33..36, dense) from the exact state at their start; the exchanges "
            "for the rank-qubit targets move half the shard through a device copy (loopback partner standing "
            "in for NVLink: rank 0 receives its own strides, so the bytes moved are real, the data not)",
    "n_qubits": n, "stride_bits": s, "rank_bits": g, "local_qubits": n - g, "delta": delta, "basis": x,
    "first_gate": g0, "gates": n_gates, "planned_exchanges": [i for i in planned if i < g0 + n_gates],
    "exchanges": st.exchanges, "exchange_bytes_sent": comm.bytes, "exchange_copy_s": comm.copy_s,
    "exchange_at_770GBps_s": comm.bytes / 770e9,
    "wall_s_per_gpu": wall, "gate_loop_s": dev_ns * 1e-9, "s_per_gate": dev_ns * 1e-9 / max(1, n_gates),
    "final_shard_compressed_bytes": b.value, "final_shard_min_ratio": r.value,
    "note": "host wall time around each gate (the Python sharded layer folds on the host per gate; the C++ "
            "driver qcs_cluster_* folds on the device).  Exchange cost at NVLink speed = bytes / 770 GB/s "
            "(measured peer bandwidth, B200_PROFILING.md)",
}))
