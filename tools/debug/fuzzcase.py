"""Replay one tests/test_gpu_fuzz.py case gate by gate against the oracle."""
import random
import sys

sys.path.insert(0, '.'); sys.path.insert(0, 'tests'); sys.path.insert(0, 'oracle')
import paper_1811_05140_b200 as q
from paper_1811_05140_b200 import metrics as mm
from oracle import Oracle
from test_gpu_fuzz import _random_ladder, _random_program

seed = int(sys.argv[1])
rng = random.Random(1000 + seed)
n = rng.randrange(3, 14)
s = rng.randrange(0, n + 1)
prog = _random_program(rng, n)
ladder, theta = _random_ladder(rng, n)
basis = rng.randrange(1 << n)
print(n, s, ladder, theta, basis, flush=True)
o = Oracle()
ost = o.state(n, s, basis)
st = q.CompressedState.basis_state(q.StateGeometry.make(n, s), basis)
lad = q.ErrorBoundLadder.make(ladder)
for i, g in enumerate(prog.gates):
    print("gate", i, g.label, g.kind, g.target, g.control, flush=True)
    reps, norm = ost.apply_gate(g, ladder, theta)
    want = mm.emit_csv([mm.gate_record(i, g.label, reps, norm)[0]], with_elapsed=False)
    m = q.apply_program_range(st, prog, i, i + 1, lad, q.RatioThreshold(theta))
    got = mm.emit_csv(m.records, with_elapsed=False)
    if got.split("\n")[1].split(",")[2:] != want.split("\n")[1].split(",")[2:]:
        print("DIFF", got, want)
        break
    bad = [j for j in range(1 << (n - s)) if st.export_blocks(j)[0] != ost.export_blocks(j)]
    if bad:
        j = bad[0]
        print("BLOCK DIFF after gate", i, "strides", bad[:8], len(bad))
        print(" gpu", st.export_blocks(j)[0].hex())
        print(" ora", ost.export_blocks(j).hex())
        break
    if st.to_amplitudes().tobytes() != ost.amplitudes().tobytes():
        print("AMP DIFF after gate", i)
        break
print("done")
