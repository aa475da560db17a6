"""Dev tool: the reference's default configuration (QFT-n, stride bits
min(n, 20), ladder 0,1e-7..1e-3, theta 16, basis 1) on one GPU — kernel-class
times, codec counters and the slowest gates.  QCS_SERIAL_CHAIN selects the
non-power-of-two path."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_05140_b200 as q  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
prog = q.build_qft(n)
geom = q.StateGeometry.make(n, min(n, 20))
st = q.CompressedState.basis_state(geom, 1)
st.profile(True)
t = time.perf_counter()
m = q.apply_program_range(st, prog, 0, len(prog.gates), q.ErrorBoundLadder.default_ladder(), q.RatioThreshold(16.0))
w = time.perf_counter() - t
print("QCS_SERIAL_CHAIN =", os.environ.get("QCS_SERIAL_CHAIN", "1"), f"qft-{n}", "wall %.3f s" % w,
      "device %.3f s" % (m.total_elapsed_ns / 1e9))
print({k: (round(v[0] / 1e6, 1), v[1]) for k, v in st.kernel_times().items()})
c = st.counters()
c.pop("phase_cycles")
print(c)
worst = sorted(m.records, key=lambda r: -r.elapsed_ns)[:5]
print("slowest gates (ms):", [(r.gate_label, round(r.elapsed_ns / 1e6, 2), round(r.max_chosen_delta, 8)) for r in worst])
