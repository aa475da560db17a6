"""Dev tool: QFT-20 (s=14) through three ladders on one GPU — device time per
kernel class, codec counters and the last gates' times.  QCS_SERIAL_CHAIN
selects the non-power-of-two path (0 rounds, 1 policy, 2 serial chain)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_05140_b200 as q  # noqa: E402

prog = q.build_qft(20)
geom = q.StateGeometry.make(20, 14)
print("QCS_SERIAL_CHAIN =", os.environ.get("QCS_SERIAL_CHAIN", "1 (default)"))
for lad in ([0.0], [q.pow2_bound(1e-3, 20)], [0.0, 1e-7, 1e-6, 1e-5, 1e-4, 1e-3]):
    st = q.CompressedState.basis_state(geom, 1)
    st.profile(True)
    t = time.perf_counter()
    m = q.apply_program_range(st, prog, 0, len(prog.gates), q.ErrorBoundLadder.make(lad),
                              q.RatioThreshold(16.0 if len(lad) > 1 else 1.0))
    w = time.perf_counter() - t
    kt = st.kernel_times()
    print(lad[:2], "wall %.3f s" % w, "device %.3f s" % (m.total_elapsed_ns / 1e9),
          {k: (round(v[0] / 1e6, 2), v[1]) for k, v in kt.items()})
    print("  ", st.counters())
    print("   last gates (us):", [(r.gate_label, r.elapsed_ns // 1000) for r in m.records[-6:]])
