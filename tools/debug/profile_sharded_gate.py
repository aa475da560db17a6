import sys, os, cProfile, pstats
sys.path.insert(0, os.getcwd())
import torch
from paper_1811_05140_b200 import circuit as cc
from paper_1811_05140_b200.distributed import GpuBackend, ShardedState, ShardGeometry, ThreadComm, ThreadGroup
n, s = 24, 16
marked = next(cc.splitmix64(7)) & ((1 << n) - 1)
prog = cc.build_grover_gate_form(n, marked, 64)
lad = [cc.pow2_bound(1e-4, n)]
st = ShardedState(ShardGeometry(n, s, 0), ThreadComm(ThreadGroup(1), 0), GpuBackend(0), 0)
for i in range(n + 100): st.apply_gate(prog.gates[i], lad, 1.0, i)
pr = cProfile.Profile(); pr.enable()
for i in range(n + 100, n + 300): st.apply_gate(prog.gates[i], lad, 1.0, i)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
