import sys, time, os
sys.path.insert(0, os.getcwd())
import torch
import paper_1811_05140_b200 as q
from paper_1811_05140_b200 import circuit as cc
from paper_1811_05140_b200.distributed import GpuBackend, ShardedState, ShardGeometry, ThreadComm, ThreadGroup
n, s = 24, 16
marked = next(cc.splitmix64(7)) & ((1 << n) - 1)
prog = cc.build_grover_gate_form(n, marked, 64)
lad = [cc.pow2_bound(1e-4, n)]
st = ShardedState(ShardGeometry(n, s, 0), ThreadComm(ThreadGroup(1), 0), GpuBackend(0), 0)
for i in range(n + 100): st.apply_gate(prog.gates[i], lad, 1.0, i)
torch.cuda.synchronize(); t0 = time.perf_counter()
for i in range(n + 100, n + 200): st.apply_gate(prog.gates[i], lad, 1.0, i)
torch.cuda.synchronize(); t1 = time.perf_counter()
print("sharded(1 rank) per gate ms", (t1 - t0) * 10)
eng = q.CompressedState.basis_state(q.StateGeometry.make(n, s), 0)
L, T = q.ErrorBoundLadder.make(lad), q.RatioThreshold(1.0)
q.apply_program_range(eng, prog, 0, n + 100, L, T)
torch.cuda.synchronize(); t0 = time.perf_counter()
q.apply_program_range(eng, prog, n + 100, n + 200, L, T)
torch.cuda.synchronize(); t1 = time.perf_counter()
print("engine run_program per gate ms", (t1 - t0) * 10)
t0 = time.perf_counter()
for i in range(n + 200, n + 300): eng.apply_gate(prog.gates[i], L, T)
torch.cuda.synchronize(); t1 = time.perf_counter()
print("engine apply_gate per gate ms", (t1 - t0) * 10)
